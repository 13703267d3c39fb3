PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_polym.so timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_varlen.py tests/test_gpu_fp8.py tests/test_gpu_parity_full.py tests/test_gpu_fullsize.py -x -q 2>&1 | tail -3
bash tools/ab.sh polym
bash tools/time_ab.sh qwen3_235b 2 cur polym
bash tools/time_ab.sh qwen3_8b 2 cur polym
bash tools/time_ab.sh tree 2 cur polym
