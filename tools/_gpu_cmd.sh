NOFULL=1 SLM_LIB=paper_2409_12892_b200/_variants/nogather/libsplatlm_b200.so bash tools/gpu_ncu_product.sh prod_nog
