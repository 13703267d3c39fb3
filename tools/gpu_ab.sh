# usage: bash tools/gpu_ab.sh <variants...>: parity tests of the current build, then ncu cycles per variant
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_varlen.py tests/test_gpu_fp8.py -x -q > gpurun_out/ab_test.log 2>&1; echo test $? > gpurun_out/ab.txt
bash tools/ab.sh "$@" >> gpurun_out/ab.txt 2>&1
bash tools/ncu_cycles.sh qwen3_235b gpurun_out/ab_cur_fp8 --fp8 > /dev/null 2>&1
echo "== cur fp8 $(grep -h '"sm__cycles_elapsed.avg"' gpurun_out/ab_cur_fp8.csv | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')" >> gpurun_out/ab.txt
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace.so timeout 300 python tools/trace_attn.py --config qwen3_235b --show 4 > gpurun_out/tr_ab.txt 2>&1
