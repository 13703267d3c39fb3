python -m paper_2605_04263_b200.build
python -c "from paper_2605_04263_b200 import build; build.build(out='paper_2605_04263_b200/libparse_notma.so', defines=['PARSE_NO_O_TMA=1'])"
for i in 1 2; do
timeout 300 python tools/time_attn.py qwen3_235b qwen3_8b tree --batch 4
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_notma.so timeout 300 python tools/time_attn.py qwen3_235b qwen3_8b tree --batch 4
done
timeout 300 python tools/time_attn.py qwen3_8b
PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_notma.so timeout 300 python tools/time_attn.py qwen3_8b
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
