mkdir -p gpurun_out
: > gpurun_out/tw.txt
for v in "" _tw148 _tw296 _tw592; do
  for c in qwen3_8b qwen3_235b tree; do
  lib=paper_2605_04263_b200/libparse$v.so
  PARSE_LIB=$PWD/$lib ncu --clock-control none -k regex:attn_ -s 2 -c 1 --csv --metrics sm__cycles_elapsed.avg,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed python tools/prof_attn.py --config $c > gpurun_out/tw_x.csv 2>&1
  echo "$v $c $(grep -h 'cycles_elapsed.avg"' gpurun_out/tw_x.csv | awk -F'","' '{print $NF}' | tr -d '"') $(grep -h 'tensor' gpurun_out/tw_x.csv | awk -F'","' '{print $NF}' | tr -d '"')" >> gpurun_out/tw.txt
  done
done
