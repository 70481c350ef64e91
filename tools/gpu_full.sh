# full ncu capture of one kernel of the C3 product path: $1 = kernel regex, $2 = launch-skip, $3 = tag
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$1 --launch-skip ${2:-0} -c 1 \
  -o gpurun_out/ncu/$3 python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/$3.log 2>&1
