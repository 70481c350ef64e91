"""Per-phase ms of one LM direction (lm_direction with a PhaseTimer) after a
warm-up step, plus the caching allocator's device-allocation counters.

    [PYTORCH_CUDA_ALLOC_CONF=...] python tools/phase_probe.py [--config c3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_12892_b200.engine import PhaseTimer  # noqa: E402
from paper_2409_12892_b200.solver import BatchSchedule, lm_direction  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    dev = torch.device("cuda", 0)
    init, cams, gts = bench.make_workload(cfg, dev)
    scene = init.to_device(dev)
    sched = BatchSchedule(cfg["subsets"])
    lm_direction(scene, cams, gts, sched, 1e-4, cfg["iters"])
    torch.cuda.synchronize()
    s0 = torch.cuda.memory_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pt = PhaseTimer()
    e0.record()
    rep = lm_direction(scene, cams, gts, sched, 1e-4, cfg["iters"], phase_timer=pt)
    e1.record()
    torch.cuda.synchronize()
    s1 = torch.cuda.memory_stats()
    out = {k: round(v, 2) for k, v in rep.phases.items()}
    out["step_ms"] = e0.elapsed_time(e1)
    for k in ("num_device_alloc", "num_device_free", "num_alloc_retries"):
        out[k] = s1.get(k, 0) - s0.get(k, 0)
    out["alloc_conf"] = os.environ.get("PYTORCH_CUDA_ALLOC_CONF")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
