NOFULL=1 bash tools/gpu_ncu_product.sh prod_c4 c4
