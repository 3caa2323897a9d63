timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "converged_mid_graph" 2>&1 | tail -3
