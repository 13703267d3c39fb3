# one-S-buffer kernel: parity first, then A/B timing against the previous build (libparse_base.so)
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_fp8.py tests/test_gpu_varlen.py -m gpu -x -q 2>&1 | tail -8
for i in 1 2; do
timeout 300 python tools/time_attn.py qwen3_235b qwen3_8b tree long --batch 4
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_base.so timeout 300 python tools/time_attn.py qwen3_235b qwen3_8b tree long --batch 4
done
bash tools/ab.sh cur base
