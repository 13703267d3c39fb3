PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace.so timeout 300 python tools/trace_attn.py --config qwen3_235b --batch 4 --show 4 2>&1 | head -32
