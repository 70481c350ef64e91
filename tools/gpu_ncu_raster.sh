# full ncu captures (source-level) of the COUNT / FILL rasteriser at C3 (one subset); $1 = tag
mkdir -p gpurun_out/ncu
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  --nvtx --nvtx-include "build/" -k regex:k_raster -c 2 \
  -o gpurun_out/ncu/$1_raster python tools/profile_subset.py --config c3 --reps 1 --product-only > gpurun_out/ncu/$1_raster.log 2>&1
