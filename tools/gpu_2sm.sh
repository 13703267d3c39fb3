mkdir -p gpurun_out
: > gpurun_out/2sm.txt
PARSE_2SM=1 timeout 300 python -m pytest tests/test_gpu_attn.py -x -q -k "bf16 and (mha_d128 or gqa4 or gqa16 or delta40 or random_b or k1_full)" > gpurun_out/2sm_test.log 2>&1; echo test $? >> gpurun_out/2sm.txt
for cfg in qwen3_235b qwen3_8b; do
  PARSE_2SM=1 timeout 300 bash tools/ncu_cycles.sh $cfg gpurun_out/cyc2_$cfg > /dev/null 2>&1
  echo "2sm $cfg $(grep -h '"sm__cycles_elapsed.avg"' gpurun_out/cyc2_$cfg.csv | tail -1 | awk -F'","' '{print $NF}' | tr -d '"') tensor $(grep -h 'pipe_tensor_cycles_active' gpurun_out/cyc2_$cfg.csv | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')" >> gpurun_out/2sm.txt
done
