# PCG vector kernel launch lists (ncu) for the in-tree library and variants: bash tools/gpu_pcg_ab.sh VARIANT...
mkdir -p gpurun_out/ncu
for v in "" "$@"; do
  if [ -n "$v" ]; then export SLM_LIB=paper_2409_12892_b200/_variants/$v/libsplatlm_b200.so; else unset SLM_LIB; fi
  timeout 1200 ncu --kernel-name-base demangled -k regex:'k_pcg|k_combine' --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu/pcg_vec_${v:-default}.csv python tools/profile_subset.py --config c3 --reps 1 > gpurun_out/ncu/pcg_vec_${v:-default}.log 2>&1
done
