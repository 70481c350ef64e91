timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_c2_subset.py tests/test_large_regime.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
bash tools/gpu_ab.sh c3 bw7 > gpurun_out/ab14.log 2>&1
