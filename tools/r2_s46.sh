timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3; echo "smoke rc=$?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/r2_ref.json
