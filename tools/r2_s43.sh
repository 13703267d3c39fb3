python -m paper_2605_04263_b200.build
timeout 1500 python -m pytest tests/test_gpu_attn.py tests/test_gpu_varlen.py tests/test_gpu_fp8.py tests/test_gpu_plan.py tests/test_gpu_2sm.py tests/test_gpu_cluster_fuzz.py tests/test_gpu_select.py -q 2>&1 | tail -2
bash tools/ab.sh cur
