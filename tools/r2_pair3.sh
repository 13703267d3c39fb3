python -m paper_2605_04263_b200.build
python -c "from paper_2605_04263_b200 import build; build.build(out='paper_2605_04263_b200/libparse_trace.so', defines=['PARSE_TRACE=1'])"
timeout 300 python -m pytest tests/test_gpu_attn.py -q -x -k "bf16" 2>&1 | tail -3
timeout 300 python tools/time_attn.py qwen3_235b qwen3_8b tree long --batch 4
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace.so timeout 300 python tools/trace_pair.py --config qwen3_235b --batch 2
timeout 600 python -m pytest tests/test_gpu_parity_full.py -q -x -k "not fp8" 2>&1 | tail -3
