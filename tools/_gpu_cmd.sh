timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_c1_end_to_end.py tests/test_c2_subset.py tests/test_large_regime.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
for v in "" base "" base; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  echo "== ${v:-default}" >> gpurun_out/ab24.log
  timeout 400 python tools/profile_subset.py --config c3 --reps 2 --skip-pcg 2>&1 | grep '"rhs"' >> gpurun_out/ab24.log
done
