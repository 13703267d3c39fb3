mkdir -p gpurun_out
for v in tracenosm trace; do
  for c in long qwen3_235b; do
  TRACE_SAVE=gpurun_out/tr_${v}_$c.npy PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_$v.so python tools/trace_attn.py --config $c --batch 2 --show 0 > /dev/null 2>&1
  done
done
ls gpurun_out/*.npy
