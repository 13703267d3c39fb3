# bench lines of every single-GPU workload (no profiler)
mkdir -p gpurun_out
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/b_235b.json 2> gpurun_out/b_235b.err; echo b235 $?
timeout 600 python bench.py --config qwen3_8b --steps 30 --warmup 5 > gpurun_out/b_8b.json 2> gpurun_out/b_8b.err; echo b8b $?
timeout 900 python bench.py --config long --per-rank-batch 8 --steps 3 --warmup 3 --no-naive --no-ragged --no-fp8 > gpurun_out/b_long.json 2> gpurun_out/b_long.err; echo blong $?
timeout 600 python bench.py --config tree --steps 20 --warmup 5 --no-naive --no-ragged > gpurun_out/b_tree.json 2> gpurun_out/b_tree.err; echo btree $?
timeout 600 python bench.py --config tiny --steps 30 --warmup 5 > gpurun_out/b_tiny.json 2> gpurun_out/b_tiny.err; echo btiny $?
