python -m paper_2605_04263_b200.build
B="from paper_2605_04263_b200 import build; build.build"
python -c "$B(out='paper_2605_04263_b200/libparse_shf.so', defines=['PARSE_EXP_SHF=1'])" &
python -c "$B(out='paper_2605_04263_b200/libparse_shf8.so', defines=['PARSE_EXP_SHF=1','PARSE_POLY16=8'])" &
python -c "$B(out='paper_2605_04263_b200/libparse_shf10.so', defines=['PARSE_EXP_SHF=1','PARSE_POLY16=10'])" &
wait
bash tools/ab.sh cur shf shf8 shf10 cur shf
