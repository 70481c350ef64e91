timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_regime.py tests/test_c1_end_to_end.py tests/test_edge_cases.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
bash tools/gpu_launches_build.sh r02e
