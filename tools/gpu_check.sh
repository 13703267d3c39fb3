# quick round-end check: smoke, every GPU test, the default bench line
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/c_smoke.log 2>&1; echo smoke $? > gpurun_out/c.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/c_pytest.log 2>&1; echo pytest $? >> gpurun_out/c.txt
timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo bench $? >> gpurun_out/c.txt
