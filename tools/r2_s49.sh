timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/r2g_full235 python tools/prof_attn.py --config qwen3_235b > /dev/null 2>&1; echo "ncu235 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/r2g_full8b python tools/prof_attn.py --config qwen3_8b > /dev/null 2>&1; echo "ncu8b rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/r2g_fullfp8 python tools/prof_attn.py --config qwen3_235b --fp8 > /dev/null 2>&1; echo "ncufp8 rc=$?"
timeout 900 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
