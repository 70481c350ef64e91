timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
bash tools/gpu_launches_build.sh u32keys
SLM_LIB=paper_2409_12892_b200/_variants/base/libsplatlm_b200.so timeout 400 python tools/profile_subset.py --config c3 --reps 2 --skip-pcg > gpurun_out/ab21_base.log 2>&1
