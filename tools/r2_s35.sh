timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_varlen.py tests/test_gpu_parity_full.py tests/test_gpu_plan.py tests/test_gpu_shards.py tests/test_gpu_fullsize.py -m gpu -x -q 2>&1 | tail -3
bash tools/ab.sh cur prev
for r in 1 2; do for v in cur prev; do lib=paper_2605_04263_b200/libparse_$v.so; [ $v = cur ] && lib=paper_2605_04263_b200/libparse.so
PARSE_LIB=$PWD/$lib timeout 300 python tools/time_attn.py qwen3_235b --batch 16 --iters 20; PARSE_LIB=$PWD/$lib timeout 300 python tools/time_attn.py qwen3_8b tree --iters 20; done; done
