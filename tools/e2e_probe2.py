import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
import bench
from paper_2409_12892_b200.engine import LossConfig
from paper_2409_12892_b200.scene import GaussianScene
from paper_2409_12892_b200.solver import BatchSchedule, lm_direction
cfg = bench.CONFIGS[sys.argv[1]]
dev = torch.device("cuda", 0)
init, cams, gts = bench.make_workload(cfg, dev)
scene = init.to_device(dev)
sched = BatchSchedule(cfg["subsets"])
for _ in range(3):
    lm_direction(scene, cams, gts, sched, 1e-4, 8, None, LossConfig())
torch.cuda.synchronize()
x_host = scene.x.detach().cpu().pin_memory()
gts_host = [g.cpu().pin_memory() for g in gts]
out_host = torch.empty(scene.param_count, dtype=torch.float32).pin_memory()
for rep in range(4):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    xs = x_host.to(dev, non_blocking=True)
    sc = GaussianScene(xs, scene.sh_degree, scene.background)
    r = lm_direction(sc, cams, gts_host, sched, 1e-4, 8, None, LossConfig())
    out_host.copy_(r.delta, non_blocking=True)
    e1.record()
    torch.cuda.synchronize()
    print("e2e rep", rep, e0.elapsed_time(e1), "wall", time.perf_counter() - t0, flush=True)
