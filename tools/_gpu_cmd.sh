bash tools/gpu_ab.sh c3 bw1m3 bw1m4 > gpurun_out/ab8.log 2>&1
