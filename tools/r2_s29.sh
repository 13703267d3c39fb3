# cluster (K/V multicast) kernel as default: full GPU suite, sanitizers, bench, ncu
python -m paper_2605_04263_b200.build
t0=$(date +%s); timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "tests $(( $(date +%s)-t0 ))s"
bash tools/gpu_sanitize.sh
for t in memcheck racecheck synccheck; do tail -2 gpurun_out/san_$t.txt; done
timeout 900 python bench.py > gpurun_out/s29_bench.json 2> gpurun_out/s29_bench.err; echo "bench rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attn_sm100 -s 2 -c 1 -o gpurun_out/s29_full235 python tools/prof_attn.py --config qwen3_235b > /dev/null 2>&1; echo "ncu235 rc=$?"
