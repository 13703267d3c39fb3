mkdir -p gpurun_out
: > gpurun_out/trace_ep.txt
for c in qwen3_8b qwen3_235b; do
  echo "== $c" >> gpurun_out/trace_ep.txt
  PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace.so python tools/trace_attn.py --config $c --show 0 2>&1 | grep -i "item transitions\|period\|steps recorded\|Error\|error" >> gpurun_out/trace_ep.txt
done
