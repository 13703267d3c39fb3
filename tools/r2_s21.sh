timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_varlen.py tests/test_gpu_parity_full.py tests/test_gpu_plan.py -m gpu -x -q 2>&1 | tail -3
bash tools/ab.sh cur prev
for c in tree long; do for v in cur prev; do lib=paper_2605_04263_b200/libparse_$v.so; [ $v = cur ] && lib=paper_2605_04263_b200/libparse.so; PARSE_LIB=$PWD/$lib timeout 300 python tools/time_attn.py $c --batch 4; done; done
