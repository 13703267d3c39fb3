# Bench lines of every single-GPU workload + the launch list of the bench step + ncu summaries
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/b_235b.json 2> gpurun_out/b_235b.err; echo b235 $?
timeout 600 python bench.py --config qwen3_8b --steps 30 --warmup 5 > gpurun_out/b_8b.json 2> gpurun_out/b_8b.err; echo b8b $?
timeout 900 python bench.py --config long --per-rank-batch 8 --steps 3 --warmup 3 --no-naive --no-ragged --no-fp8 > gpurun_out/b_long.json 2> gpurun_out/b_long.err; echo blong $?
timeout 600 python bench.py --config tiny --steps 30 --warmup 5 > gpurun_out/b_tiny.json 2> gpurun_out/b_tiny.err; echo btiny $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-naive --no-ragged --no-fp8 --no-readout > gpurun_out/launches.log 2>&1; echo launches $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/full235fp8 -f python tools/prof_attn.py --config qwen3_235b --fp8 > gpurun_out/full235fp8.log 2>&1; echo full8 $?
