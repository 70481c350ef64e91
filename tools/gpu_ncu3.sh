set -x
mkdir -p gpurun_out/ncu
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/launches_v2.csv python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_stream --launch-skip 7 -c 1 \
  -o gpurun_out/ncu/stream_v2 python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > /dev/null 2>&1
ls gpurun_out/ncu
