# round-2 final validation on the committed build
python -m paper_2605_04263_b200.build
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "tests $(( $(date +%s)-t0 ))s"
bash tools/gpu_sanitize.sh
timeout 900 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config qwen3_8b --no-cpu-baseline > gpurun_out/r2f_bench_8b.json 2> gpurun_out/r2f_bench_8b.err; echo "bench8b rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/r2f_full235 python tools/prof_attn.py --config qwen3_235b > /dev/null 2>&1; echo "ncu235 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/r2f_full8b python tools/prof_attn.py --config qwen3_8b > /dev/null 2>&1; echo "ncu8b rc=$?"
