"""Per-phase CUDA-event breakdown of one subset of a bench config.

    python tools/profile_subset.py [--config c3] [--views 25] [--reps 3]

Prints JSON: build phases, rhs, diag, and the four kernels of one
J^T W J p product (pair forward, applyJ, applyJT pairs, pair backward).
Used to pick ncu targets; not a bench number.
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2409_12892_b200 import _lib  # noqa: E402
from paper_2409_12892_b200.engine import CacheSet, PhaseTimer  # noqa: E402
from paper_2409_12892_b200.solver import BatchSchedule, pcg_run  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--skip-pcg", action="store_true")
    ap.add_argument("--product-only", action="store_true",
                    help="build, rhs, diag, then 2 fused products inside an NVTX range 'product' (ncu --nvtx)")
    args = ap.parse_args()
    cfg = dict(bench.CONFIGS[args.config])
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    views = BatchSchedule(cfg["subsets"]).batches(cfg["views"])[0]
    cfg_one = dict(cfg)
    init, cams, gts = bench.make_workload(cfg_one, dev, only=set(views))
    scene = init.to_device(dev)
    cams = [cams[i] for i in views]
    gts = [gts[i] for i in views]
    out = {}
    cs = None
    for rep in range(args.reps):
        # release the previous rep's cache first: with two 37 GB caches alive
        # the allocator would cudaMalloc inside the timed FILL phase
        cs = None
        torch.cuda.synchronize()
        T = PhaseTimer()
        torch.cuda.nvtx.range_push("build")
        cs = CacheSet(scene, cams, gts, timer=T)
        torch.cuda.nvtx.range_pop()
        T.tick("done")
        phases = T.summary()
        a = ev()
        b = cs.rhs()
        c = ev()
        M = cs.diag()
        d = ev()
        torch.cuda.synchronize()
        phases["rhs"] = a.elapsed_time(c)
        phases["diag"] = c.elapsed_time(d)
        p = torch.randn(scene.param_count, device=dev)
        g = torch.empty_like(p)
        if args.product_only:
            p_gm = cs.gm_pack(p)
            dp = torch.zeros(_lib.load().slm_backward_blocks(cs.G), dtype=torch.float64, device=dev)
            cs.jtwj(p, g, 1e-4, M, dp, False, p_gm=p_gm)      # warm
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_push("product")
            for _ in range(2):
                cs.jtwj(p, g, 1e-4, M, dp, False, p_gm=p_gm)
            torch.cuda.nvtx.range_pop()
            torch.cuda.synchronize()
            print(json.dumps(dict(phases, E=cs.E, N=cs.N, R=cs.R, pairs=cs.n_pairs, G=cs.G)))
            return
        # the padded gaussian-major copy the PCG p kernels hand to the product
        p_gm = cs.gm_pack(p)
        k = []
        for _ in range(3):
            e0 = ev()
            cs.pair_forward(p)
            e1 = ev()
            cs.apply_j_raw(weighted=True)
            e2 = ev()
            cs.apply_jt_raw(cs.u, g, 1.0, p, M, 1e-4, None)
            e3 = ev()
            k.append((e0, e1, e2, e3))
        torch.cuda.synchronize()
        e0, e1, e2, e3 = k[-1]
        phases["api_pair_forward"] = e0.elapsed_time(e1)
        phases["api_apply_j"] = e1.elapsed_time(e2)
        phases["api_apply_jt+backward"] = e2.elapsed_time(e3)
        f = []
        for _ in range(3):
            f0 = ev()
            cs.jtwj(p, g, 1e-4, M, None, p_gm=p_gm)
            f1 = ev()
            f.append((f0, f1))
        torch.cuda.synchronize()
        phases["fused_jtwj_product"] = f[-1][0].elapsed_time(f[-1][1])
        # the fused product's launches timed one by one
        from paper_2409_12892_b200._lib import call, off, ptr, stream_ptr
        dp = torch.zeros(_lib.load().slm_backward_blocks(cs.G), dtype=torch.float64, device=dev)
        ks = []
        for _ in range(3):
            t0 = ev()
            cs.pair_forward(p, p_gm=p_gm)
            t1 = ev()
            a = cs._tile_args(with_m=True)
            a.gradr, a.out, a.out1 = ptr(cs.gradr), ptr(cs.run_acc), off(cs.run_acc, 8 * cs.R)
            call("slm_jtwj_runs", _lib.byref(a), stream_ptr())
            t2 = ev()
            cs._backward(cs.run_acc, g, 0, 1.0, p, M, 1e-4, dp, False)
            t3 = ev()
            ks.append((t0, t1, t2, t3))
        torch.cuda.synchronize()
        t0, t1, t2, t3 = ks[-1]
        phases["k_pair_forward"] = t0.elapsed_time(t1)
        phases["k_stream_fused"] = t1.elapsed_time(t2)
        phases["k_backward"] = t2.elapsed_time(t3)

        if not args.skip_pcg:
            s0 = ev()
            pcg_run(cs, b, M, 1e-4, cfg["iters"])
            s1 = ev()
            torch.cuda.synchronize()
            phases["pcg_total"] = s0.elapsed_time(s1)
        phases.update(E=cs.E, N=cs.N, R=cs.R, pairs=cs.n_pairs, G=cs.G,
                      mem_gb=torch.cuda.max_memory_allocated() / 1e9)
        out = phases
        del cs
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
