timeout 600 python -m pytest tests/test_gpu_varlen.py -m gpu -x -q 2>&1 | tail -2
for r in 1 2; do for v in cur prev; do lib=paper_2605_04263_b200/libparse_$v.so; [ $v = cur ] && lib=paper_2605_04263_b200/libparse.so
PARSE_LIB=$PWD/$lib timeout 300 python tools/time_ragged.py qwen3_235b qwen3_8b; done; done
