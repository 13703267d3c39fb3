timeout 900 python -m pytest tests/test_gpu_parity_full.py -m gpu -q -s -k "mixed" 2>&1 | grep -E "parity|passed|failed|Error|assert" | head -20
