timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_varlen.py tests/test_gpu_parity_full.py tests/test_gpu_plan.py -m gpu -x -q 2>&1 | tail -3
bash tools/ab.sh cur prev
for v in cur prev; do lib=paper_2605_04263_b200/libparse_$v.so; [ $v = cur ] && lib=paper_2605_04263_b200/libparse.so
for cfg in qwen3_235b qwen3_8b; do PARSE_LIB=$PWD/$lib bash tools/ncu_cycles.sh $cfg gpurun_out/fp8_${v}_$cfg --fp8 > /dev/null 2>&1
echo "== fp8 $v $cfg $(grep -h '"sm__cycles_elapsed.avg"' gpurun_out/fp8_${v}_$cfg.csv | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')"; done; done
