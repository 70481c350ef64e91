timeout 400 python tools/profile_subset.py --config c3 --reps 3 --skip-pcg > gpurun_out/prof_sync2.json 2>&1
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c3_sync.log 2>&1
