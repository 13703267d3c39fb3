timeout 1200 python -m pytest tests/test_gpu_2sm.py -q 2>&1 | tail -2
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_clalt.so timeout 300 python -m pytest tests/test_gpu_attn.py -x -q -k "bf16" 2>&1 | tail -1
bash tools/ab.sh clalt
bash tools/time_ab.sh qwen3_235b 2 cur clalt nocl
