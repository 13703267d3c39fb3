#!/bin/bash
# usage: tools/ncu_cycles.sh <config> [out-prefix]  — one attention launch, key counters
cfg=${1:-qwen3_235b}; out=${2:-gpurun_out/cyc_$cfg}; extra=${3:-}
ncu --clock-control none -k regex:attn_ -s 2 -c 1 --csv \
  --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__issue_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
  python tools/prof_attn.py --config $cfg $extra > $out.csv 2>&1
python - "$out.csv" << 'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ni, vi, ui = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
for r in rows[1:]:
    print(f"{r[ni]:70s} {r[vi]:>20s} {r[ui]}")
PY
