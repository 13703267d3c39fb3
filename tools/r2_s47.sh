PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_pfs.so timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_parity_full.py -m gpu -x -q -k "not fp8" 2>&1 | tail -2
bash tools/ab.sh cur pfs
