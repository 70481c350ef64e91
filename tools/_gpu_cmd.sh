bash tools/gpu_ab.sh c3 pmd5 pmd6 > gpurun_out/ab16.log 2>&1
