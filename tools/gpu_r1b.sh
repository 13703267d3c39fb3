set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/f_smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/f_pytest.log 2>&1; echo pytest $?
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench $?
timeout 600 python bench.py --config tree --steps 20 --warmup 5 --no-cpu-baseline --no-naive --no-ragged > gpurun_out/f_benchtree.json 2> gpurun_out/f_benchtree.err; echo benchtree $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-naive --no-ragged > gpurun_out/f_ncu_bench.log 2>&1; echo launches $?
