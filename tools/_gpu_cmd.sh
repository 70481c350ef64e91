timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
mkdir -p gpurun_out/ncu
for v in "" bw1_2 bw1_4; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  timeout 600 ncu --kernel-name-base demangled -k regex:'k_gauss_backward_packed<.int.16, .int.1>' --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/bw1_${v:-default}.csv python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > /dev/null 2>&1
done
