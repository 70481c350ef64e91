bash tools/gpu_ab.sh c3 gl8 jt8 > gpurun_out/ab20.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_c1_end_to_end.py tests/test_c2_subset.py tests/test_large_regime.py tests/test_offload.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
