python -m paper_2605_04263_b200.build
for c in long tree tiny; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2e_bench_$c.json 2> gpurun_out/r2e_bench_$c.err; echo "$c rc=$?"; done
timeout 600 python bench.py --config tiny --graph --no-cpu-baseline > gpurun_out/r2e_bench_tiny_graph.json 2> gpurun_out/r2e_bench_tiny_graph.err; echo "tinyg rc=$?"
