python -m paper_2605_04263_b200.build
timeout 300 python -m pytest tests/test_gpu_select.py tests/test_gpu_attn.py -x -q 2>&1 | tail -1
bash tools/time_ab.sh tiny 2 cur nopdl nocl
bash tools/time_ab.sh qwen3_8b 2 cur nopdl
