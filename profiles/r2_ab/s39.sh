PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_polym2.so timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_cluster_fuzz.py -x -q 2>&1 | tail -1
bash tools/ab.sh cur polym2
bash tools/time_ab.sh qwen3_8b 2 cur polym2
bash tools/time_ab.sh qwen3_235b 2 cur polym2
