for v in cur f0 f2 f6; do lib=paper_2605_04263_b200/libparse_$v.so; [ $v = cur ] && lib=paper_2605_04263_b200/libparse.so
for cfg in qwen3_235b qwen3_8b; do PARSE_LIB=$PWD/$lib bash tools/ncu_cycles.sh $cfg gpurun_out/fp8_${v}_$cfg --fp8 > /dev/null 2>&1
echo "== fp8 $v $cfg $(grep -h '"sm__cycles_elapsed.avg"' gpurun_out/fp8_${v}_$cfg.csv | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')"; done; done
bash tools/ab.sh cur
