"""One full LM iteration (lm_step: batched direction, line search, rho,
trust-region decision) on a bench configuration; prints the energies, gamma,
rho, the decision, the PCG statistics and the observed fraction.

    python tools/lm_step_probe.py [--config c3] [--perturb 0.02] [--lam 1e-4] [--iters 8] [--subsets N]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_12892_b200 import lm as L  # noqa: E402
from paper_2409_12892_b200 import synthetic as S  # noqa: E402
from paper_2409_12892_b200.solver import BatchSchedule  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--perturb", type=float, default=None)
    ap.add_argument("--lam", type=float, default=1e-4)
    ap.add_argument("--iters", type=int, default=None)
    ap.add_argument("--subsets", type=int, default=None)
    ap.add_argument("--views", type=int, default=None)
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    if args.iters:
        cfg["iters"] = args.iters
    if args.subsets:
        cfg["subsets"] = args.subsets
    if args.views:
        cfg["views"] = args.views
    if args.perturb is not None:
        cfg["perturb"] = args.perturb
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    init, cams, gts = bench.make_workload(cfg, dev)
    scene = init.to_device(dev)
    t0 = time.time()
    e_all0 = L.energy(scene, cams, gts)
    rep = L.lm_step(scene, cams, gts, BatchSchedule(cfg["subsets"]), lam=args.lam, n_iters=cfg["iters"])
    e_all1 = L.energy(rep.scene, cams, gts) if rep.accepted else e_all0
    torch.cuda.synchronize()
    d = rep.delta.double()
    out = dict(config=args.config, perturb=cfg.get("perturb"), lam=args.lam, iters=cfg["iters"],
               energy_all_before=e_all0, energy_all_after=e_all1, gamma=rep.gamma, rho=rep.rho,
               accepted=rep.accepted, lam_new=rep.lam, batch0_energy_before=rep.energy_before,
               batch0_energy_after=rep.energy_after, observed_fraction=rep.direction.observed_fraction,
               delta_absmax=float(d.abs().max()), delta_median=float(d.abs().median()),
               pcg=rep.direction.pcg[:3], wall_s=round(time.time() - t0, 1))
    print(json.dumps(out, default=float))


if __name__ == "__main__":
    main()
