timeout 600 python tools/profile_subset.py --config c3 --reps 2 > gpurun_out/profile_c3.json 2>&1
