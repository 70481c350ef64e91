mkdir -p gpurun_out/ncu
timeout 1200 ncu --nvtx --nvtx-include "build/" --kernel-name-base demangled -k regex:'k_raster' --set full --import-source on --clock-control none -c 2 \
  -o gpurun_out/ncu/raster_r02 python tools/profile_subset.py --config c3 --reps 1 --product-only > gpurun_out/ncu/raster_r02.log 2>&1
