timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_varlen.py tests/test_gpu_parity_full.py tests/test_gpu_plan.py -m gpu -x -q 2>&1 | tail -2
bash tools/ab.sh cur
