# round-1 evidence: GPU tests, launch list and full captures of the product kernels (C3 subset)
set -x
mkdir -p gpurun_out/ncu
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 python tools/profile_subset.py --config c3 --reps 2 > gpurun_out/profile_c3.json 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/ncu/launches_c3_subset.csv python tools/profile_subset.py --config c3 --reps 1 > gpurun_out/ncu/launches.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:k_stream<5>' -c 1 \
  -o gpurun_out/ncu/stream_fused_c3 python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/full1.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k 'regex:k_pair_backward|k_run_params|k_pair_forward|k_diag_tile' -c 6 \
  -o gpurun_out/ncu/chain_c3 python tools/profile_subset.py --config c3 --reps 1 --skip-pcg > gpurun_out/ncu/full2.log 2>&1
tail -3 gpurun_out/ncu/*.log
cat gpurun_out/pytest_gpu.log
