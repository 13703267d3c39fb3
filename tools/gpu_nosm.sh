mkdir -p gpurun_out
: > gpurun_out/ctastat2.txt
for c in tree qwen3_8b qwen3_235b; do
  PARSE_LIB=$PWD/paper_2605_04263_b200/libparse_ctastat.so python tools/cta_stat.py --config $c >> gpurun_out/ctastat2.txt 2>&1
done
