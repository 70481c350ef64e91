timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
NOFULL=1 bash tools/gpu_ncu_product.sh prod_tq
NOFULL=1 SLM_LIB=paper_2409_12892_b200/_variants/base/libsplatlm_b200.so bash tools/gpu_ncu_product.sh prod_tqbase
