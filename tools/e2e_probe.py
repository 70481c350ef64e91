"""Where does the e2e time go?  Times the C3 LM step with device inputs, with
host inputs, and the raw H2D copies alone (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_12892_b200.engine import LossConfig  # noqa: E402
from paper_2409_12892_b200.scene import GaussianScene  # noqa: E402
from paper_2409_12892_b200.solver import BatchSchedule, lm_direction  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
dev = torch.device("cuda", 0)
init, cams, gts = bench.make_workload(cfg, dev)
scene = init.to_device(dev)
sched = BatchSchedule(cfg["subsets"])
x_host = scene.x.cpu().pin_memory()
g_host = [g.cpu().pin_memory() for g in gts]


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


for _ in range(2):
    lm_direction(scene, cams, gts, sched, 1e-4, 8, None, LossConfig())
torch.cuda.synchronize()
a = ev(); lm_direction(scene, cams, gts, sched, 1e-4, 8, None, LossConfig()); b = ev()
torch.cuda.synchronize()
print("device inputs ms", a.elapsed_time(b))
a = ev()
xs = x_host.to(dev, non_blocking=True)
gd = [g.to(dev, non_blocking=True) for g in g_host]
b = ev()
torch.cuda.synchronize()
print("h2d only ms", a.elapsed_time(b))
t0 = time.perf_counter()
a = ev()
xs = x_host.to(dev, non_blocking=True)
gd = [g.to(dev, non_blocking=True) for g in g_host]
sc = GaussianScene(xs, scene.sh_degree, scene.background)
r = lm_direction(sc, cams, gd, sched, 1e-4, 8, None, LossConfig())
b = ev()
torch.cuda.synchronize()
print("host inputs ms", a.elapsed_time(b), "wall", time.perf_counter() - t0)
for rep in range(3):
    a = ev()
    xs = x_host.to(dev, non_blocking=True)
    sc = GaussianScene(xs, scene.sh_degree, scene.background)
    r = lm_direction(sc, cams, g_host, sched, 1e-4, 8, None, LossConfig())
    b = ev()
    torch.cuda.synchronize()
    print("host images streamed per subset ms", a.elapsed_time(b))
    a = ev()
    xs = x_host.to(dev, non_blocking=True)
    gd = [g.to(dev, non_blocking=True) for g in g_host]
    sc = GaussianScene(xs, scene.sh_degree, scene.background)
    r = lm_direction(sc, cams, gd, sched, 1e-4, 8, None, LossConfig())
    b = ev()
    torch.cuda.synchronize()
    print("host inputs copied up front ms", a.elapsed_time(b))
    a = ev(); lm_direction(scene, cams, gts, sched, 1e-4, 8, None, LossConfig()); b = ev()
    torch.cuda.synchronize()
    print("device inputs ms", a.elapsed_time(b))
