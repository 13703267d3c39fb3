python -m paper_2605_04263_b200.build
timeout 1200 python -m pytest tests/test_gpu_cluster_fuzz.py -q -s 2>&1 | grep -E "fuzz|passed|failed|Error" > gpurun_out/s38_fuzz.txt; tail -3 gpurun_out/s38_fuzz.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e --no-readout --no-naive --no-ragged --no-fp8 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['roofline'].get('cluster_units'), d['roofline'].get('l2_read_bytes_ncu'))"
