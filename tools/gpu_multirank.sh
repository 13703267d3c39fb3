# N>1 plumbing of bench.py on a 1-GPU box: 2 ranks share cuda:0 over gloo (timings meaningless)
mkdir -p gpurun_out
: > gpurun_out/mr.txt
run() { name=$1; shift; PARSE_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $((29550 + RANDOM % 400)) bench.py --gpus 2 "$@" > gpurun_out/mr_$name.json 2> gpurun_out/mr_$name.err; echo $name $? >> gpurun_out/mr.txt; }
run weak --steps 3 --warmup 3 --no-cpu-baseline --no-naive --no-ragged --no-fp8 --no-readout
run strong --steps 3 --warmup 3 --no-cpu-baseline --no-naive --no-ragged --no-fp8 --no-readout --scaling strong
run peer --steps 3 --warmup 3 --no-cpu-baseline --no-naive --no-ragged --no-fp8 --no-readout --no-e2e --gather peer
run graph --steps 3 --warmup 3 --no-cpu-baseline --no-naive --no-ragged --no-fp8 --no-readout --no-e2e --graph
run ref --impl reference --steps 1 --warmup 1
