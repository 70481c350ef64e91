timeout 900 python bench.py --config c1 --steps 5 --warmup 3 > gpurun_out/bench_c1.log 2>&1
timeout 900 python bench.py --config c1 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c1_ref.log 2>&1
