PARSE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-readout --no-naive --no-ragged --no-fp8 > gpurun_out/r2_2rank.json 2> gpurun_out/r2_2rank.err; echo "2rank rc=$?"
tail -3 gpurun_out/r2_2rank.err
