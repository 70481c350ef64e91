# full ncu captures (source-level) of the product tail kernels at C3: backward, pair forward, gm->am
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ncu/clocks_tail.txt
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:'k_gauss_backward_packed|k_pair_m|k_gm_to_am' --launch-skip 3 -c 3 \
  -o gpurun_out/ncu/tail_r02b python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/tail_r02b.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/ncu/clocks_tail.txt
