bash tools/gpu_evidence.sh > gpurun_out/evidence.log 2>&1
