mkdir -p gpurun_out
SLM_LIB=paper_2409_12892_b200/_variants/j2/libsplatlm_b200.so timeout 240 python -m pytest tests/test_gpu_parity.py tests/test_scale_properties.py tests/test_large_regime.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/ab_tests.log
bash tools/gpu_ab.sh c3 j2 > gpurun_out/ab.log 2>&1
bash tools/gpu_ab.sh c4 j2 > gpurun_out/ab2.log 2>&1
cat gpurun_out/ab_tests.log; grep -h "==\|k_stream_fused\|fused_jtwj\|api_apply_j\"" gpurun_out/ab.log gpurun_out/ab2.log
