# ncu of the C3 J^T W J p product's launches (NVTX range 'product' of
# tools/profile_subset.py --product-only): $1 = tag.  Writes the launch list
# (times + DRAM bytes) and one --set full capture of every product kernel.
mkdir -p gpurun_out/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/ncu/clocks_$1.txt
timeout 900 ncu --nvtx --nvtx-include "product/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum \
  --clock-control none --csv --log-file gpurun_out/ncu/$1_launches.csv \
  python tools/profile_subset.py --config ${2:-c3} --reps 1 --product-only > gpurun_out/ncu/$1_launches.log 2>&1
[ -n "$NOFULL" ] || timeout 1200 ncu --nvtx --nvtx-include "product/" --set full --import-source on --clock-control none -c 4 \
  -o gpurun_out/ncu/$1_full python tools/profile_subset.py --config c3 --reps 1 --product-only > gpurun_out/ncu/$1_full.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv >> gpurun_out/ncu/clocks_$1.txt
