# final state: full GPU suite + default bench line
python -m paper_2605_04263_b200.build
t0=$(date +%s); timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3; echo "tests $(( $(date +%s)-t0 ))s"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/s40_bench.json 2> gpurun_out/s40_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s40_ref.json 2> gpurun_out/s40_ref.err; echo "ref rc=$?"
