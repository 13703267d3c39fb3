python -m paper_2605_04263_b200.build
timeout 600 python -m pytest tests/test_gpu_readout.py tests/test_gpu_select.py -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --no-cpu-baseline --no-naive --no-ragged --no-fp8 --no-e2e --steps 5 --warmup 3 > gpurun_out/r2_rd.json 2> gpurun_out/r2_rd.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2_rd.json').read().strip().splitlines()[-1]); print(json.dumps(d['readout'], indent=0))"
