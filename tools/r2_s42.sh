PARSE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 5 --warmup 3 --no-readout --no-naive --no-ragged --no-fp8 > gpurun_out/s42_2rank.json 2> gpurun_out/s42_2rank.err; echo "2rank rc=$?"
tail -c 1500 gpurun_out/s42_2rank.json
