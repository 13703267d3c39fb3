# round-2 bench run: default line, 2-rank plumbing on one GPU (gloo), reference arm, config 2
python -m paper_2605_04263_b200.build
cd $GRAFT_REPO_ROOT
t0=$(date +%s); timeout 900 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$? $(( $(date +%s)-t0 ))s"
t0=$(date +%s); PARSE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-readout --no-naive --no-ragged --no-fp8 > gpurun_out/r2_bench_2rank_gloo.json 2> gpurun_out/r2_bench_2rank_gloo.err; echo "2rank rc=$? $(( $(date +%s)-t0 ))s"
t0=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$? $(( $(date +%s)-t0 ))s"
t0=$(date +%s); timeout 900 python bench.py --config qwen3_8b --no-cpu-baseline > gpurun_out/r2_bench_8b.json 2> gpurun_out/r2_bench_8b.err; echo "8b rc=$? $(( $(date +%s)-t0 ))s"
