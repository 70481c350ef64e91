# round evidence: GPU tests, smoke, bench (C3 default + C2 + C4 + C5 + reference arm),
# product launch list + full captures (NVTX product range), build launch list, sanitizers
set -x
mkdir -p gpurun_out/ncu
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1
timeout 600 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2.log 2>&1
timeout 900 python bench.py --config c4 --steps 2 --warmup 3 --no-cpu > gpurun_out/bench_c4.log 2>&1
timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_c5.log 2>&1
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout 600 python bench.py --config c1 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --config c1 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c1_ref.log 2>&1
timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu --offload 0.25 > gpurun_out/bench_c5_off.log 2>&1
timeout 600 python tools/profile_subset.py --config c3 --reps 2 > gpurun_out/profile_c3.json 2>&1
bash tools/gpu_launches_build.sh final
bash tools/gpu_ncu_product.sh prod_final
bash tools/gpu_launches.sh final
mkdir -p gpurun_out/sanitizer; bash tools/sanitize.sh > gpurun_out/sanitizer/summary.txt 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log
