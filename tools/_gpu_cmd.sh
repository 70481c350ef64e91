bash tools/gpu_ncu_product.sh prod_gm2
