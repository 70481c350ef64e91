# full ncu captures (source-level) of the product tail kernels at C3: the forward
# chain on the padded gaussian-major p (4th k_pair_m launch of profile_subset)
# and the J^T backward chain; $1 = tag
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ncu/clocks_$1.txt
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:'k_pair_m<.int.16>' --launch-skip 3 -c 1 \
  -o gpurun_out/ncu/$1_pm python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/$1_pm.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:'k_gauss_backward_packed<.int.16, .int.0>|k_gm_to_am' --launch-skip 4 -c 2 \
  -o gpurun_out/ncu/$1_bw python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/$1_bw.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/ncu/clocks_$1.txt
