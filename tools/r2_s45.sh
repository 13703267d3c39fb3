timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-readout --no-naive --no-ragged --no-fp8 > gpurun_out/r2_b45.json 2> gpurun_out/r2_b45.err; echo "rc=$?"
tail -3 gpurun_out/r2_b45.err
