free -g > gpurun_out/host_mem.txt
timeout 900 python -m pytest tests/test_offload.py -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_offload.log
