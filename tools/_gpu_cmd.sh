PARITY_OUT_C2=gpurun_out/parity_c2.json timeout 1200 python -m pytest tests/test_c2_subset.py -m gpu -q --durations=5 2>&1 | tail -25 > gpurun_out/pytest_c2.log
