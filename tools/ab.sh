# usage: bash tools/ab.sh <variant>... — ncu cycles of each libparse_<variant>.so ("cur" = libparse.so), config 3 and 2
for v in "$@"; do
  lib=paper_2605_04263_b200/libparse_$v.so; [ "$v" = cur ] && lib=paper_2605_04263_b200/libparse.so
    [ -f "$lib" ] || python tools/variant.py "$v" > /dev/null
  for cfg in qwen3_235b qwen3_8b; do
    PARSE_LIB=$PWD/$lib bash tools/ncu_cycles.sh $cfg gpurun_out/ab_${v}_$cfg > /dev/null 2>&1
    c=$(grep -h '"sm__cycles_elapsed.avg"' gpurun_out/ab_${v}_$cfg.csv | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')
    echo "== $v $cfg $c"
  done
done
