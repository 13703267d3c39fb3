PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_cs.so timeout 300 python tools/cta_stat.py --config qwen3_8b 2>&1 | tail -12
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_cs.so timeout 300 python tools/cta_stat.py --config qwen3_235b 2>&1 | tail -12
