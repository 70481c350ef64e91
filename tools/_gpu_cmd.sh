timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_large_regime.py tests/test_offload.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
bash tools/gpu_ab.sh c3 pmgather > gpurun_out/ab10.log 2>&1
