# full ncu capture (source-level) of the fused product kernel k_stream<5> at C3; $1 = tag
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ncu/clocks_$1.txt
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:'k_stream<.int.5>' --launch-skip 1 -c 1 \
  -o gpurun_out/ncu/$1 python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/$1.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> gpurun_out/ncu/clocks_$1.txt
