set -x
nproc; lscpu | grep -E "Model name|Socket|Core|Thread|NUMA node\(s\)"; free -g | head -2; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2605_04263_b200.build
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
