# FP8 variant: parity tests, bf16 regression, cycles of both paths on configs 3 and 2
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fp8.py -x -q -s > gpurun_out/fp8_test.log 2>&1; echo fp8test $? > gpurun_out/fp8.txt
timeout 600 python -m pytest tests/test_gpu_attn.py -x -q > gpurun_out/fp8_attn.log 2>&1; echo attntest $? >> gpurun_out/fp8.txt
for cfg in qwen3_235b qwen3_8b; do
  bash tools/ncu_cycles.sh $cfg gpurun_out/cyc_bf16_$cfg >> gpurun_out/fp8.txt 2>&1
  bash tools/ncu_cycles.sh $cfg gpurun_out/cyc_fp8_$cfg --fp8 >> gpurun_out/fp8.txt 2>&1
done
timeout 300 python tools/prof_attn.py --config qwen3_235b --iters 10 >> gpurun_out/fp8.txt 2>&1
timeout 300 python tools/prof_attn.py --config qwen3_235b --iters 10 --fp8 >> gpurun_out/fp8.txt 2>&1
