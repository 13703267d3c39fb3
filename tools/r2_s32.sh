# round-2 final validation of the cluster (K/V multicast) build
python -m paper_2605_04263_b200.build
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "tests $(( $(date +%s)-t0 ))s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 300 python -m pytest tests/test_gpu_parity_full.py -q -s 2>&1 | grep -iE "max|passed" > gpurun_out/s32_parity_full.txt
bash tools/gpu_benches.sh
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.err; echo ref $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s32_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/s32_full235 python tools/prof_attn.py --config qwen3_235b > /dev/null 2>&1; echo "ncu235 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/s32_full8b python tools/prof_attn.py --config qwen3_8b > /dev/null 2>&1; echo "ncu8b rc=$?"
timeout 900 ncu --set full --clock-control none -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/s32_fullfp8 python tools/prof_attn.py --config qwen3_235b --fp8 > /dev/null 2>&1; echo "ncufp8 rc=$?"
