bash tools/gpu_launches.sh build_r02
