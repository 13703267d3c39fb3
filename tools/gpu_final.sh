set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke $?
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/f_pytest.log 2>&1; echo pytest $?
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench $?
timeout 600 python bench.py --config qwen3_8b --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/f_bench8b.json 2> gpurun_out/f_bench8b.err; echo bench8b $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f_ncu_bench.log 2>&1; echo launches $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/f_attn235 -f python tools/prof_attn.py --config qwen3_235b > gpurun_out/f_full235.log 2>&1; echo full235 $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/f_attn8b -f python tools/prof_attn.py --config qwen3_8b > gpurun_out/f_full8b.log 2>&1; echo full8b $?
