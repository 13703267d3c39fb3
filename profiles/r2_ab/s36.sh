python -m paper_2605_04263_b200.build
timeout 900 python -m pytest tests/test_gpu_varlen.py tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_plan.py -x -q 2>&1 | tail -2
for r in 1 2; do
for v in cur nocl; do
  lib=paper_2605_04263_b200/libparse_$v.so; [ "$v" = cur ] && lib=paper_2605_04263_b200/libparse.so
  PARSE_LIB=$PWD/$lib timeout 600 python tools/time_ragged.py qwen3_235b --iters 10 2>&1 | tail -1
done
done
