# round-2 parity run: all-element multi-item parity, f3 100 cases, readout -inf
python -m paper_2605_04263_b200.build
timeout 1500 python -m pytest tests/test_gpu_parity_full.py tests/test_model_equivalence.py tests/test_gpu_readout.py -m gpu -q -s --durations=30 2>&1 | grep -v "^$" | tail -80
