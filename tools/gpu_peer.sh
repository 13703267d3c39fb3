mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peer_gather.py tests/test_gpu_select.py -x -q > gpurun_out/peer_test.log 2>&1; echo test $? > gpurun_out/peer.txt
PARSE_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29565 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-naive --no-ragged --no-fp8 --no-readout --no-e2e --gather peer > gpurun_out/mr_peer.json 2> gpurun_out/mr_peer.err; echo peerbench $? >> gpurun_out/peer.txt
