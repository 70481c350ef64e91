timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
bash tools/gpu_ncu_product.sh prod_camf
bash tools/gpu_ab.sh c3 base > gpurun_out/ab23.log 2>&1
