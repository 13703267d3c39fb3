timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_varlen.py tests/test_gpu_parity_full.py tests/test_gpu_plan.py -m gpu -x -q 2>&1 | tail -4
bash tools/ab.sh cur prev
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace1.so timeout 300 python tools/trace_attn.py --config qwen3_8b --show 4 2>&1 | grep -E "item transitions"
