set -x
mkdir -p gpurun_out/ncu
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_stream --launch-skip 7 -c 1 \
  -o gpurun_out/ncu/stream_fused_c3 python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/full1.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_raster -c 2 \
  -o gpurun_out/ncu/raster_c3 python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/full3.log 2>&1
ls -la gpurun_out/ncu
