#!/bin/bash
# usage: bash tools/time_ab.sh <config> <rounds> <variant>...  — wall time per step of
# each libparse_<variant>.so ("cur" = libparse.so), interleaved on one box so
# power-cap clock behaviour (not just cycles) enters the comparison
cfg=$1; rounds=$2; shift 2
for r in $(seq 1 $rounds); do
  for v in "$@"; do
    lib=paper_2605_04263_b200/libparse_$v.so; [ "$v" = cur ] && lib=paper_2605_04263_b200/libparse.so
    [ -f "$lib" ] || python tools/variant.py "$v" > /dev/null
    PARSE_LIB=$PWD/$lib timeout 300 python bench.py --config $cfg --steps 40 --warmup 10 --no-cpu-baseline \
      --no-e2e --no-readout --no-naive --no-ragged --no-fp8 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']
print('== $v r$r', '%.4f ms' % d['ms_per_step'], 'frac %.4f' % d['roofline']['frac'], 'mhz', c['sm_mhz'], 'W', c.get('power_w'), c['reasons'])"
  done
done
