bash tools/ab.sh nokv nmnokv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/r2full235 python tools/prof_attn.py --config qwen3_235b > gpurun_out/r2full235.log 2>&1; echo "ncu rc=$?"
