python -m paper_2605_04263_b200.build
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_varlen.py tests/test_gpu_fp8.py tests/test_gpu_parity_full.py tests/test_gpu_fullsize.py tests/test_gpu_plan.py tests/test_gpu_shards.py -x -q 2>&1 | tail -2
bash tools/ab.sh cur
bash tools/time_ab.sh qwen3_235b 2 cur clalt nocl
bash tools/time_ab.sh qwen3_8b 2 cur nocl
