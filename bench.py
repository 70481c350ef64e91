"""Benchmark: one full LM iteration (cache build + PCG + Eq. 7 combine) of the
3DGS-LM inner solver on the BASELINE.json headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3|c2|c1]
                    [--impl ours|reference]

Default workload (config C3, BASELINE.json configs[2], the metric's "1M
Gaussians"): 1,000,000 Gaussians (SH degree 3), 200 views at 1024x1024 split
into 8 strided subsets of 25 views, 8 PCG iterations, lambda_reg = 1e-4.
Subsets are sharded round-robin over N ranks (one process per GPU, NCCL);
the only exchange is one all_reduce of the packed Eq. 7 [num; den].

`value` = LM step ms (device-timed with CUDA events, inputs resident, max over
ranks).  `e2e` = the same step through the public API with the scene and the
ground-truth images copied from pinned host memory and the update direction
copied back, every step.  `roofline` = the J^T W J p product (pair forward +
applyJ + applyJT + pair backward) against measured HBM bandwidth, algorithmic
bytes 48 E + 36 N + 16 M per product.  `--impl reference` times
the reference's own numpy implementation (pip-installed into baseline/_ref)
driven through Alg. 1 / Eq. 7 on every host core (one process per core and
view, oracle/ref_parallel.py), on a bounded sample of the same generator, and
projects it to the workload.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LM step ms and JᵀJp HBM GB/s vs peak, 1M Gaussians, at 1/2/4/8 B200"

CONFIGS = {
    # name: gaussians, views, W, H, subsets, pcg iters, generator
    "c1": dict(G=2000, views=8, W=64, H=64, subsets=1, iters=10, gen="reference", degree=3),
    "c2": dict(G=100_000, views=32, W=256, H=256, subsets=4, iters=8, gen="reference", degree=3),
    "c3": dict(G=1_000_000, views=200, W=1024, H=1024, subsets=8, iters=8, gen="footprint", degree=3),
    # BASELINE.json configs[3] (Mip-NeRF360 scale; quoted for 8 GPUs, one subset per GPU)
    "c4": dict(G=3_000_000, views=200, W=1552, H=1032, subsets=8, iters=8, gen="footprint", degree=3),
    # BASELINE.json configs[4] (ScanNet++ scale; 16 subsets, 2 per GPU on 8 GPUs), "gradient cache sized
    # near 180 GB HBM per GPU": with the reference's opacity law the T >= 1e-4 stop saturates the
    # generator near K ~ 50 entries per pixel (2.16e9 entries per subset), i.e. 155 GB per subset in
    # the reference's 72-byte records; here 45 GB at 21 B/entry (150 GB HBM peak with rho's cache)
    "c5": dict(G=2_000_000, views=400, W=1616, H=1080, subsets=16, iters=8, gen="footprint", degree=3,
               k_target=71.0),
}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._p = None
        self._t = None

    def __enter__(self):
        cmd = ["nvidia-smi", "-i", str(self.gpu),
               "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
               "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
               "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
               "--format=csv,noheader,nounits", "-lms", "200"]
        try:
            self._p = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
            # nvidia-smi's NVML start-up stalls the driver for tens of ms: let
            # it finish (first row) before the caller opens the timed region
            t_end = time.time() + 5.0
            while not self.rows and time.time() < t_end:
                time.sleep(0.01)
        except Exception:
            self._p = None
        return self

    def _read(self):
        for line in self._p.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self._p is not None:
            self._p.terminate()
            try:
                self._p.wait(timeout=5)
            except Exception:
                self._p.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4)
                          if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def make_host_workload(cfg):
    """(truth, init, cameras) host scenes of a configuration (the reference's
    generator for C1/C2, the footprint generator for C3-C5)."""
    from paper_2409_12892_b200 import synthetic as S
    G, V, W, H, deg = cfg["G"], cfg["views"], cfg["W"], cfg["H"], cfg["degree"]
    if cfg["gen"] == "reference":
        truth = S.make_synthetic_scene(0, G, deg)
        init = S.perturb(truth, 1, cfg.get("perturb", 0.1))
    else:
        truth = S.make_footprint_scene(0, G, W, H, deg, k_target=cfg.get("k_target", 32.0))
        init = S.perturb(truth, 1, cfg.get("perturb", 0.02))
    return truth, init, S.make_camera_ring(V, W, H)


def make_workload(cfg, device, only=None):
    import torch

    from paper_2409_12892_b200.rasterizer import render
    truth, init, cams = make_host_workload(cfg)
    tscene = truth.to_device(device)
    gts = []
    for i, c in enumerate(cams):
        if only is not None and i not in only:
            gts.append(None)
            continue
        img = render(tscene, c, traversals=False).image
        gts.append(img.float().contiguous())
    del tscene
    torch.cuda.synchronize()
    return init, cams, gts


def run_ours(args, cfg):
    import torch
    import torch.distributed as dist

    from paper_2409_12892_b200 import _lib
    from paper_2409_12892_b200.engine import LossConfig
    from paper_2409_12892_b200.solver import BatchSchedule, lm_direction

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # BENCH_BACKEND=gloo lets the multi-rank path be exercised with several
    # ranks sharing one GPU (functional check only; the bench uses NCCL)
    backend = os.environ.get("BENCH_BACKEND", "nccl")
    local = local % max(torch.cuda.device_count(), 1) if backend != "nccl" else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    _lib.load()
    init_h, cams, gts = make_workload(cfg, dev)
    scene = init_h.to_device(dev)
    sched = BatchSchedule(cfg["subsets"])
    loss = LossConfig()
    lam, iters = 1e-4, cfg["iters"]
    stream = torch.cuda.current_stream()

    class ProdTimer:
        def __init__(self):
            self.ev = []

        def __enter__(self):
            s = torch.cuda.Event(enable_timing=True)
            s.record(stream)
            self.ev.append([s, None])

        def __exit__(self, *a):
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            self.ev[-1][1] = e

    offload = None if args.offload in (None, "none", "0") else (args.offload if args.offload == "auto"
                                                                  else float(args.offload))

    def step(timer=None):
        return lm_direction(scene, cams, gts, sched, lam, iters, None, loss, rank, world, product_timer=timer,
                            offload=offload)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for _ in range(args.warmup):
        rep = step()
    barrier()
    timer = ProdTimer()
    launches0 = _lib.launch_counter["calls"]
    gpu_index = int(os.environ.get("CUDA_VISIBLE_DEVICES", str(local)).split(",")[local]) \
        if os.environ.get("CUDA_VISIBLE_DEVICES") else local
    with ClockSampler(gpu_index) as clk:
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        reps = []
        for _ in range(args.steps):
            reps.append(step(timer))
        t1.record(stream)
        barrier()
    launches = _lib.launch_counter["calls"] - launches0
    ms = t0.elapsed_time(t1) / args.steps
    prod_ms = [a.elapsed_time(b) for a, b in timer.ev]
    rep = reps[-1]
    # e2e through the public API with host buffers
    x_host = scene.x.detach().cpu().pin_memory()
    gts_host = [g.cpu().pin_memory() for g in gts]
    h2d = x_host.numel() * 8 + sum(g.numel() * 4 for g in gts_host)
    d2h = scene.param_count * 4
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    out_host = torch.empty(scene.param_count, dtype=torch.float32).pin_memory()
    from paper_2409_12892_b200.scene import GaussianScene
    n_e2e = max(1, min(args.steps, 3))
    for it in range(1 + n_e2e):  # one untimed warm-up call (first use of the pinned buffers)
        if it == 1:
            barrier()
            e0.record(stream)
        xs = x_host.to(dev, non_blocking=True)
        sc = GaussianScene(xs, scene.sh_degree, scene.background)
        # the images stay in pinned host memory: lm_direction copies each
        # subset's images on a side stream while the previous subset is solved
        r = lm_direction(sc, cams, gts_host, sched, lam, iters, None, loss, rank, world, offload=offload)
        out = out_host.copy_(r.delta, non_blocking=True)
        del sc, xs
    e1.record(stream)
    barrier()
    e2e_ms = e0.elapsed_time(e1) / n_e2e
    _ = out
    # one untimed full LM iteration (direction + line search + rho + trust
    # region) on the same inputs: is the benchmarked direction a descent
    # step, and where does a step's time go (CUDA-event phases)
    from paper_2409_12892_b200 import lm as L
    from paper_2409_12892_b200.engine import PhaseTimer
    pt = PhaseTimer()
    # phases of one plain step (the timed call, with CUDA-event ticks)
    step_phases = lm_direction(scene, cams, gts, sched, lam, iters, None, loss, rank, world,
                                        phase_timer=pt, offload=offload).phases
    e_before = L.energy(scene, cams, gts, rank=rank, world_size=world)
    lr = L.lm_step(scene, cams, gts, sched, lam, iters, rank=rank, world_size=world)
    e_after = L.energy(lr.scene, cams, gts, rank=rank, world_size=world) if lr.accepted else e_before
    lm_info = {"energy_before": e_before, "energy_after": e_after, "gamma": lr.gamma, "rho": lr.rho,
               "accepted": bool(lr.accepted), "lam_new": lr.lam,
               "observed_fraction": lr.direction.observed_fraction,
               "energy_views": "all views; line search on the strided 30 % (SPEC:409-417)"}
    phases = {k: round(v, 2) for k, v in (step_phases or {}).items()}
    del lr
    # max over ranks
    vals = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
    ms, e2e_ms = float(vals[0]), float(vals[1])
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None
    # roofline of the J^T W J p product (per subset: E, N from this rank's caches)
    E_sub = statistics.mean(rep.entries) if rep.entries else 0
    N_sub = (cfg["views"] // cfg["subsets"]) * cfg["W"] * cfg["H"]
    Mp = scene.param_count
    alg_bytes = 48 * E_sub + 36 * N_sub + 16 * Mp
    t_prod = statistics.median(prod_ms) / 1e3 if prod_ms else float("nan")
    achieved = alg_bytes / t_prod / 1e9
    peak, peak_kind = peaks()
    # DRAM bytes per product from the committed ncu launch list of this config
    # (tools/gpu_ncu_product.sh -> tools/traffic_from_ncu.py); null without one
    traffic, traffic_src = None, None
    tf = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tf):
        try:
            tj = json.load(open(tf))
            traffic = tj.get(args.config)
            src = tj.get("_source", {}).get(args.config, {})
            if traffic is not None:
                traffic_src = f"ncu launch list {os.path.basename(src.get('launch_list', '?'))} ({src.get('written', '?')})"
        except Exception:
            traffic = None
    cpu = cpu_baseline(cfg, rep, args) if (world == 1 and not args.no_cpu) else None
    line = {
        "metric": METRIC, "value": round(ms, 3), "unit": "ms", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32 cache/products, f64 rasteriser+residuals", "data": "synthetic",
        "config": {"workload": f"{args.config.upper()}: {cfg['G']} Gaussians (SH{cfg['degree']}), "
                               f"{cfg['views']} views @ {cfg['W']}x{cfg['H']}, {cfg['subsets']} strided subsets, "
                               f"{cfg['iters']} PCG iters, lambda 1e-4",
                   "generator": cfg["gen"], "entries_per_subset": E_sub,
                   "entries_per_pixel": round(E_sub / N_sub, 2) if N_sub else None,
                   "pcg": rep.pcg[:2], "lm_step": lm_info,
                   "offload": {"mode": args.offload, "host_record_bytes_per_step": 21 * sum(rep.offloaded_entries),
                               "peak_hbm_gb": round(torch.cuda.max_memory_allocated(dev) / 1e9, 1)},
                   "phases_ms_per_step": phases,
                   "l2": "inputs larger than L2 (cache >> 126 MB)",
                   "parallelism": f"subsets round-robin over {world} rank(s), one NCCL all_reduce"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_source": traffic_src,
                     "peak_kind": peak_kind,
                     "kernel": "J^T W J p product", "product_ms_median": round(t_prod * 1e3, 4),
                     "algorithmic_bytes": alg_bytes},
        "e2e": {"value": round(e2e_ms, 3), "unit": "ms", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": launches,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return line


# ---------------------------------------------------------------------------
# CPU reference arm: the reference's own numpy code (baseline/_ref) driven
# through Alg. 1 + Eq. 7 (oracle/ref_driver.py); the oracle port only when the
# reference package is absent.
# ---------------------------------------------------------------------------

def cpu_sample(cfg, n_views=2):
    """Bounded sample of the same generator at the same pixels-per-Gaussian
    (hence the same entries-per-pixel): G_s Gaussians, n_views views,
    resolution scaled so that W*H / G matches the workload."""
    import numpy as np

    from paper_2409_12892_b200 import synthetic as S
    G = cfg["G"]
    Gs = min(G, 16000)
    scale = np.sqrt(Gs / G)
    W = max(16, int(round(cfg["W"] * scale)))
    H = max(16, int(round(cfg["H"] * scale)))
    if cfg["gen"] == "reference":
        truth = S.make_synthetic_scene(0, Gs, cfg["degree"])
        init = S.perturb(truth, 1, cfg.get("perturb", 0.1))
    else:
        truth = S.make_footprint_scene(0, Gs, W, H, cfg["degree"], k_target=cfg.get("k_target", 32.0))
        init = S.perturb(truth, 1, cfg.get("perturb", 0.02))
    cams = S.make_camera_ring(n_views, W, H)
    return truth, init, cams, (Gs, W, H)


class CpuArm:
    """The reference's own numpy code (baseline/_ref) driven through Alg. 1 /
    Eq. 7 on the host: one process per host core (oracle/ref_parallel.py; the
    reference's render is GIL-bound, so processes, not threads), one view per
    core of a bounded sample; the oracle port (1 core) only when the reference
    package is absent.  The sample's inputs are prepared once; `run()` times
    one LM direction."""

    def __init__(self, cfg):
        from oracle import ref_driver as RD
        self.cfg = cfg
        self.R = RD.import_reference()
        self.cores = (os.cpu_count() or 1) if self.R is not None else 1
        # a workload small enough for the CPU (BASELINE C1) is run as is:
        # the measurement is then the whole step, not a projection
        self.full = cfg["G"] <= 16000 and cfg["gen"] == "reference"
        if self.full:
            truth, init, cams = make_host_workload(cfg)
            self.shape = (cfg["G"], cfg["W"], cfg["H"])
            self.n_batches = cfg["subsets"]
        else:
            truth, init, cams, self.shape = cpu_sample(cfg, max(2, self.cores) if self.R is not None else 2)
            self.n_batches = 1
        self.n_views = len(cams)
        if self.R is not None:
            self.kind = "reference"
            self.R["parallel"].set_num_threads(1)
            rc = [RD.ref_camera(self.R, c) for c in cams]
            self.gts = [self.R["rasterizer"].render(RD.ref_scene(self.R, truth), c).image.rgb for c in rc]
            self.scene, self.cams = RD.ref_scene(self.R, init), rc
        else:
            import oracle as O
            self.kind = "port"

            def osc(h):
                return O.OScene(h.positions, h.rotations, h.log_scales, h.opacity_logits, h.sh_coeffs,
                                h.sh_degree, h.background)
            self.cams = [O.OCamera(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width, c.height)
                         for c in cams]
            self.gts = [O.rasterize(osc(truth), c)["image"] for c in self.cams]
            self.scene = osc(init)

    def run(self):
        """(seconds, entries, phases) of one LM direction on the sample."""
        iters = self.cfg["iters"]
        t0 = time.perf_counter()
        if self.kind == "reference":
            from oracle import ref_parallel as RP
            ph = {}
            _, E, _ = RP.lm_direction(self.R, self.scene, self.cams, self.gts, n_batches=self.n_batches,
                                      lam=1e-4, n_iters=iters, workers=self.cores, phases=ph)
            return time.perf_counter() - t0, E, ph
        import oracle as O
        O.lm_direction(self.scene, self.cams, self.gts, n_batches=self.n_batches, lam=1e-4, n_iters=iters)
        dt = time.perf_counter() - t0
        E = sum(O.rasterize(self.scene, c)["pixel"].size for c in self.cams)
        return dt, E, {}

    def text(self, E, dt, ph):
        who = ("reference splatlm (baseline/_ref) + Alg. 1/Eq. 7 driver, view-parallel over "
               f"{self.cores} processes" if self.kind == "reference" else "oracle port, 1 core")
        phs = ", ".join(f"{k} {v:.2f}s" for k, v in ph.items())
        what = "the full workload" if self.full else "a bounded sample"
        return (f"{who}, {what}: LM step on {self.shape[0]} Gaussians, {self.n_views} views @ {self.shape[1]}x"
                f"{self.shape[2]}, {E} entries, {self.cfg['iters']} PCG iters = {dt:.2f} s "
                f"({1e9 * dt / max(E, 1):.0f} ns/entry wall; {phs})")


def cpu_baseline(cfg, rep, args):
    arm = CpuArm(cfg)
    dt, E, ph = arm.run()
    E_full = sum(rep.entries) * 1.0
    proj_ms = dt * 1e3 * (1.0 if arm.full else E_full / max(E, 1)) if rep.entries else None
    return {"value": round(proj_ms, 1) if proj_ms else None, "unit": "ms", "cores": arm.cores, "kind": arm.kind,
            "sample": arm.text(E, dt, ph)
            + ("" if arm.full else f"; projected linearly in cache entries to the workload's {int(E_full)} entries/step"),
            "cpu": _cpu_name(), "os_cpu_count": os.cpu_count()}


def _cpu_name():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    arm = CpuArm(cfg)
    times = []
    for i in range(args.warmup + args.steps):
        dt, E, ph = arm.run()
        if i >= args.warmup:
            times.append(dt)
    dt = statistics.median(times)
    # entries of the full workload: K (entries per pixel, from the sample) x pixels
    k = E / (arm.n_views * arm.shape[1] * arm.shape[2])
    E_full = E if arm.full else k * cfg["views"] * cfg["W"] * cfg["H"]
    ms = dt * 1e3 * E_full / E
    line = {"metric": METRIC, "value": round(ms, 1), "unit": "ms", "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 1), "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": f"{args.config.upper()} (same generator), " + (
                           "measured on the full workload" if arm.full else "projected from a bounded sample"),
                       "entries_per_pixel": round(k, 2)},
            "cpu_baseline": {"value": round(ms, 1), "unit": "ms", "cores": arm.cores, "kind": arm.kind,
                             "sample": arm.text(E, dt, ph)
                             + f"; median of {args.steps}" + ("" if arm.full else
                                                               f", x{E_full / E:.0f} entries to the workload")},
            "e2e": {"value": round(ms, 1), "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return line


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--offload", default=None,
                    help="cache offload to host memory: a fraction of the records, or 'auto' (only what "
                         "does not fit in HBM); default none")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
