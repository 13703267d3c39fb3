# final build: full GPU suite, smoke, default bench line, launch list
python -m paper_2605_04263_b200.build
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "tests $(( $(date +%s)-t0 ))s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/s37_bench.json 2> gpurun_out/s37_bench.err; echo "bench rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s37_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1; echo "launches rc=$?"
