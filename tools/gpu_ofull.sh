mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/of_pytest.log 2>&1; echo pytest $? > gpurun_out/of.txt
timeout 600 compute-sanitizer --tool synccheck python tools/sanitize_run.py > gpurun_out/san_synccheck.txt 2>&1; echo synccheck $? >> gpurun_out/of.txt
timeout 600 compute-sanitizer --tool racecheck python tools/sanitize_run.py > gpurun_out/san_racecheck.txt 2>&1; echo racecheck $? >> gpurun_out/of.txt
timeout 600 compute-sanitizer --tool memcheck python tools/sanitize_run.py > gpurun_out/san_memcheck.txt 2>&1; echo memcheck $? >> gpurun_out/of.txt
bash tools/ab.sh cur >> gpurun_out/of.txt 2>&1
