PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_cllocal.so timeout 300 python -m pytest tests/test_gpu_attn.py -x -q -k "small_dense and bf16" 2>&1 | tail -1
bash tools/ab.sh cur clnomc cllocal
