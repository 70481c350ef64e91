"""Precision breakdown of the GPU path vs the fp64 oracle on the parity-test
problem (diagnostic; prints JSON)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from helpers import ocam, oscene, problem, rel  # noqa: E402
from paper_2409_12892_b200.engine import CacheSet  # noqa: E402
from paper_2409_12892_b200.solver import pcg_run  # noqa: E402


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--G", type=int, default=60)
    ap.add_argument("--views", type=int, default=3)
    ap.add_argument("--W", type=int, default=32)
    ap.add_argument("--H", type=int, default=28)
    ap.add_argument("--degree", type=int, default=3)
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    truth, init, cams, gts = problem(seed=args.seed, G=args.G, n_views=args.views, W=args.W, H=args.H,
                                     degree=args.degree)
    osc = oscene(init)
    ocs = [ocam(c) for c in cams]
    gv, b = [], 0
    for c, gt in zip(ocs, gts):
        rs = O.rasterize(osc, c)
        res = O.residuals(rs["image"], gt)
        bb, v = O.build_cache(osc, c, res, rast=rs)
        gv.append(O.gaussian_order(v))
        b = b + bb
    M = sum(O.diag_jtj(osc, v) for v in gv)
    scene = init.to_device()
    cs = CacheSet(scene, cams, [torch.from_numpy(g).cuda() for g in gts])
    out = {}
    bg = cs.rhs().double().cpu().numpy()
    Mg = cs.diag().double().cpu().numpy()
    out["b"] = rel(bg, b)
    out["M"] = rel(Mg, M)
    out["b_maxrel"] = float(np.max(np.abs(bg - b) / np.maximum(np.abs(b), 1e-30)))
    out["M_maxrel"] = float(np.max(np.abs(Mg - M) / np.maximum(np.abs(M), 1e-30)))
    rng = np.random.default_rng(3)
    for name, p in (("rand", rng.standard_normal(b.size)), ("b_over_M", b / np.maximum(M, 1e-12))):
        ref = O.jtwj(p, osc, gv)
        g = torch.empty(b.size, dtype=torch.float32, device="cuda")
        cs.jtwj(torch.from_numpy(p).float().cuda(), g)
        gg = g.double().cpu().numpy()
        out[f"jtwj_{name}"] = rel(gg, ref)
        out[f"jtwj_{name}_p32"] = rel(O.jtwj(p.astype(np.float32).astype(np.float64), osc, gv), ref)
    for lam in (1.0, 1e-4):
        ref = O.pcg(osc, gv, b, M, lam, 8)
        x = pcg_run(cs, cs.rhs(), cs.diag(), lam, 8).double().cpu().numpy()
        out[f"pcg_{lam}"] = rel(x, ref)
        x2 = O.pcg(osc, gv, bg, Mg, lam, 8)
        out[f"pcg_{lam}_oracle_with_gpu_bM"] = rel(x2, ref)
        x3 = pcg_run(cs, torch.from_numpy(b).float().cuda(), torch.from_numpy(M).float().cuda(), lam,
                     8).double().cpu().numpy()
        out[f"pcg_{lam}_gpu_with_oracle_bM"] = rel(x3, ref)
        x4 = O.pcg(osc, gv, b.astype(np.float32).astype(float), M.astype(np.float32).astype(float), lam, 8)
        out[f"pcg_{lam}_oracle_f32_bM"] = rel(x4, ref)
    # hybrid: fp64 host PCG loop, GPU products; per-iteration product errors
    for lam in (1.0, 1e-4):
        Mf = np.maximum(M, 1e-12)

        def gp(p):
            g = torch.empty(b.size, dtype=torch.float32, device="cuda")
            cs.jtwj(torch.from_numpy(p).float().cuda(), g)
            return g.double().cpu().numpy() + lam * Mf * p

        def op(p):
            return O.jtwj(p, osc, gv) + lam * Mf * p
        errs = []
        x = b / Mf
        r = b - gp(x)
        errs.append(rel(gp(x), op(x)))
        z = r / Mf
        p = z.copy()
        rz = r @ z
        for i in range(8):
            g = gp(p)
            errs.append(rel(g, op(p)))
            a = rz / (p @ g)
            x = x + a * p
            r = r - a * g
            z = r / Mf
            rzn = r @ z
            p = z + (rzn / rz) * p
            rz = rzn
        out[f"hybrid_{lam}"] = rel(x, O.pcg(osc, gv, b, M, lam, 8))
        out[f"hybrid_{lam}_prod_errs"] = errs
    out = {k: v for k, v in out.items() if not k.endswith("prod_errs")}
    out["args"] = vars(args)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
