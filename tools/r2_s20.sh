# session re-entry check on the committed build: GPU tests, default bench, config-2/3 cycles
python -m paper_2605_04263_b200.build
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "tests $(( $(date +%s)-t0 ))s"
timeout 900 python bench.py > gpurun_out/s20_bench.json 2> gpurun_out/s20_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/s20_bench.json
bash tools/ab.sh cur
