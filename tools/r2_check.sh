# round-2 re-entry check: full GPU suite + default bench line + config 2 line
python -m paper_2605_04263_b200.build
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15; echo "tests $(( $(date +%s)-t0 ))s"
t0=$(date +%s); timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo "bench rc=$? $(( $(date +%s)-t0 ))s"
timeout 300 python tools/time_attn.py qwen3_235b qwen3_8b tree long --batch 4
