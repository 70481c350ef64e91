# full ncu capture (source-level) of the fused diag + rhs sweep k_stream<8> at C3 (one subset); $1 = tag
mkdir -p gpurun_out/ncu
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k regex:'k_stream<.int.8>' -c 1 \
  -o gpurun_out/ncu/$1_diag python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/$1_diag.log 2>&1
