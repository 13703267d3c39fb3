python -m paper_2605_04263_b200.build
python -c "from paper_2605_04263_b200 import build; build.build(out='paper_2605_04263_b200/libparse_notma.so', defines=['PARSE_NO_O_TMA=1'])"
bash tools/ab.sh cur notma cur notma
