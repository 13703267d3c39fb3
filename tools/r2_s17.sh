timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_varlen.py tests/test_gpu_parity_full.py tests/test_gpu_plan.py -m gpu -x -q 2>&1 | tail -4
bash tools/ab.sh cur two
timeout 300 python tools/time_attn.py qwen3_235b qwen3_8b tree long --batch 4
TRACE_SAVE=gpurun_out/trace_si.npy PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace1.so timeout 300 python tools/trace_attn.py --config qwen3_235b --batch 4 --show 4 > gpurun_out/trace_si.txt 2>&1
