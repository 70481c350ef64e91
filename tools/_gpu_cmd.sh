timeout 1200 python bench.py > gpurun_out/bench_c3.log 2>&1
bash tools/gpu_ncu_product.sh prod_r02
