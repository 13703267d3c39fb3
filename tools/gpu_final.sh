# Round-end refresh: smoke, GPU tests, bench lines of every single-GPU workload,
# launch list of the bench step, ncu --set full of the attention kernel (bf16, fp8)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f_pytest.log 2>&1; echo pytest $?
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/b_235b.json 2> gpurun_out/b_235b.err; echo b235 $?
timeout 600 python bench.py --config qwen3_8b --steps 30 --warmup 5 > gpurun_out/b_8b.json 2> gpurun_out/b_8b.err; echo b8b $?
timeout 900 python bench.py --config long --per-rank-batch 8 --steps 3 --warmup 3 --no-naive --no-ragged --no-fp8 > gpurun_out/b_long.json 2> gpurun_out/b_long.err; echo blong $?
timeout 600 python bench.py --config tree --steps 20 --warmup 5 --no-naive --no-ragged > gpurun_out/b_tree.json 2> gpurun_out/b_tree.err; echo btree $?
timeout 600 python bench.py --config tiny --steps 30 --warmup 5 > gpurun_out/b_tiny.json 2> gpurun_out/b_tiny.err; echo btiny $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-naive --no-ragged --no-fp8 --no-readout > gpurun_out/launches.log 2>&1; echo launches $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/full235 -f python tools/prof_attn.py --config qwen3_235b > gpurun_out/full235.log 2>&1; echo full235 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/full8b -f python tools/prof_attn.py --config qwen3_8b > gpurun_out/full8b.log 2>&1; echo full8b $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/full235fp8 -f python tools/prof_attn.py --config qwen3_235b --fp8 > gpurun_out/full235fp8.log 2>&1; echo full8 $?
for cfg in long tree; do
  timeout 900 ncu --clock-control none -k regex:attn_sm100 -s 1 -c 1 --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum python tools/prof_attn.py --config $cfg --iters 2 --batch 8 > gpurun_out/dram_$cfg.csv 2>&1; echo dram_$cfg $?
done
