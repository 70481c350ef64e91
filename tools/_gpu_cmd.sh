mkdir -p gpurun_out
SLM_LIB=paper_2409_12892_b200/_variants/gts/libsplatlm_b200.so timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_solver_oracle.py tests/test_lm_outer.py -m gpu -q -x 2>&1 | tail -2 > gpurun_out/ab_tests.log
for v in "" gts "" gts; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  echo "== ${v:-default}"
  timeout 300 python tools/profile_subset.py --config c3 --reps 2 2>&1 | grep '"pcg_total"\|"k_backward"\|"fused_jtwj'
done > gpurun_out/ab.log 2>&1
cat gpurun_out/ab_tests.log gpurun_out/ab.log
