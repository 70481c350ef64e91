set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python tools/profile_subset.py --config c3 --reps 2 > gpurun_out/profile_c3.json 2>&1
timeout 1200 python bench.py > gpurun_out/bench_c3.log 2>&1
tail -3 gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench_c3.log
cat gpurun_out/profile_c3.json
