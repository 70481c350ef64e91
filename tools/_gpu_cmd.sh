mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1
timeout 900 python bench.py --config c1 --impl reference --steps 2 --warmup 1 > gpurun_out/bench_c1_ref.log 2>&1
tail -c 400 gpurun_out/bench_ref.log; tail -c 300 gpurun_out/bench_c1_ref.log
