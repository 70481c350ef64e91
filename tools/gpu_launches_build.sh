# launch list of one subset's cache build only (NVTX range 'build' of tools/profile_subset.py); $1 = tag, $2 = config (c3)
mkdir -p gpurun_out/ncu
timeout 900 ncu --nvtx --nvtx-include "build/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/build_${1:-cur}.csv python tools/profile_subset.py --config ${2:-c3} --reps 1 --product-only > gpurun_out/ncu/build_${1:-cur}.log 2>&1
