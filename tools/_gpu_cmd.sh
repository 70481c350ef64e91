timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -8 > gpurun_out/pytest_gpu.log
bash tools/gpu_ab.sh c3 > gpurun_out/ab15.log 2>&1
