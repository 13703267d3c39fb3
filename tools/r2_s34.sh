for v in cur nocl; do
  lib=paper_2605_04263_b200/libparse_$v.so; [ "$v" = cur ] && lib=paper_2605_04263_b200/libparse.so
  PARSE_LIB=$PWD/$lib timeout 600 ncu --clock-control none -k regex:attn_ -s 2 -c 1 --csv --metrics lts__t_sectors_srcunit_tex_op_read.sum,l1tex__m_xbar2l1tex_read_bytes.sum,sm__cycles_elapsed.avg,dram__bytes_read.sum python tools/prof_attn.py --config qwen3_235b > gpurun_out/l2_$v.csv 2>&1
  echo "== $v"; grep -E "lts__t_sectors|xbar2l1tex|cycles_elapsed|dram__bytes" gpurun_out/l2_$v.csv | awk -F'","' '{print $(NF-2), $NF}'
done
