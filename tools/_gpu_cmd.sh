mkdir -p gpurun_out/ncu
timeout 1200 ncu --kernel-name-base demangled -k regex:'k_pcg|k_combine' --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ncu/pcg_vec.csv python tools/profile_subset.py --config c3 --reps 1 > gpurun_out/ncu/pcg_vec.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_c1_end_to_end.py tests/test_c2_subset.py tests/test_large_regime.py tests/test_offload.py -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest_quick.log
