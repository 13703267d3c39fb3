timeout 900 python -m pytest tests/test_gpu_cluster_fuzz.py -q -s -k ragged 2>&1 | grep -E "fuzz|passed|failed|Error|assert" | tail -14
