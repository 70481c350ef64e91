mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c3.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; tail -c 1500 gpurun_out/bench_c3.log
