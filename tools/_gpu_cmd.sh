mkdir -p gpurun_out/ncu
timeout 900 ncu --nvtx --nvtx-include "build/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/ncu/build_c4.csv python tools/profile_subset.py --config c4 --reps 1 --product-only > gpurun_out/ncu/build_c4.log 2>&1
