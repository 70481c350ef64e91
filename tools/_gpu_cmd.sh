timeout 1200 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/bench_c5.log 2>&1
timeout 1200 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu --offload 0.25 > gpurun_out/bench_c5_off.log 2>&1
