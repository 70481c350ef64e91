# 2-rank bench on one GPU over gloo (the N>1 launch path of bench.py), then the 1-rank C2 line
set -x
BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c2_2rank_gloo.log 2>&1
tail -2 gpurun_out/bench_c2_2rank_gloo.log
timeout 600 python bench.py --config c2 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c2.log 2>&1; tail -1 gpurun_out/bench_c2.log
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_ref.log 2>&1; tail -1 gpurun_out/bench_ref.log
bash tools/gpu_full.sh k_stream 8 stream5_v6
