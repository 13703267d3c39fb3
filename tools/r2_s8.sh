bash tools/ab.sh r200 r192 r184
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace.so timeout 300 python tools/trace_attn.py --config qwen3_235b --batch 4 --show 4 2>&1 | grep -E "item transitions"
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_trace.so timeout 300 python tools/trace_attn.py --config qwen3_8b --show 4 2>&1 | grep -E "item transitions|period|busy"
