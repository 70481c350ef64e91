# round evidence: GPU tests, smoke, bench (C3 default + C2 + C4 + C5 + reference arm),
# launch list and full captures of the hot kernels (C3 subset)
set -x
mkdir -p gpurun_out/ncu
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
bash tools/gpu_launches.sh final
bash tools/gpu_full.sh k_stream 8 stream5_final
bash tools/gpu_full.sh k_pair_m 0 pairm_final
bash tools/gpu_full.sh k_gauss_backward_packed 0 bwd_final
bash tools/gpu_full.sh k_raster 25 count_final
bash tools/gpu_full.sh k_raster 26 fill_final
bash tools/gpu_full.sh k_residuals 0 resid_final
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
