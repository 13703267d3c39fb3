python -c "from paper_2605_04263_b200 import build; build.build()" > gpurun_out/v_build.log 2>&1
bash tools/ncu_cycles.sh qwen3_235b gpurun_out/cyc_ring_235b > gpurun_out/v_cyc.log 2>&1
bash tools/ncu_cycles.sh qwen3_8b gpurun_out/cyc_ring_8b >> gpurun_out/v_cyc.log 2>&1
timeout 900 python -m pytest tests/test_gpu_varlen.py tests/test_gpu_attn.py -x -q > gpurun_out/v_varlen.log 2>&1; echo varlen $?
