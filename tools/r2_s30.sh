timeout 1500 python bench.py --config long --per-rank-batch 8 --no-cpu-baseline > gpurun_out/r2e_bench_long.json 2> gpurun_out/r2e_bench_long.err; echo "long rc=$?"
