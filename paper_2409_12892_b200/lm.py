"""LM outer-loop rows on the device (SPEC-only in the
reference): energy, dyadic line search, model reduction and
rho (Eq. 6), trust-region update and one full LM
iteration (SPEC lm_fit body).

Energies are fp64 (rasteriser and residual kernels); the model reduction uses
the frozen caches of the first image batch:
    ||F||^2 - ||F + gamma J Delta||^2 = 2 gamma b.Delta - gamma^2 Delta.(J^T W J Delta)
with b = -J^T color_grad (build_cache) and W = grad_r_sq, i.e. the
"J gamma Delta via apply_j + weight" path of SPEC:431 expanded.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .engine import LossConfig, ViewFrame, project_and_bin, raster_args, rast_cfg_struct, residual_pass
from .scene import GaussianScene
from .solver import BatchSchedule, lm_direction

LAMBDA_MIN, LAMBDA_MAX = 1e-4, 1e4   # SPEC:473 bounds used by trust_region_update


def view_energy(scene: GaussianScene, camera, gt: torch.Tensor, config=None, loss: LossConfig = LossConfig(),
                cfg_s=None, err: torch.Tensor | None = None) -> torch.Tensor:
    """E = sum r^2 of one view as a device fp64 scalar (render COUNT pass +
    residual kernel, no cache).  `gt` may live on the host (it is copied to
    the scene's device); the projection's error flags (non-finite
    parameters, zero quaternion) are OR-ed into `err` when given."""
    from .rasterizer import DEFAULT_CONFIG
    dev = scene.device
    gt = gt.to(dev, non_blocking=True)
    config = config if config is not None else DEFAULT_CONFIG
    cfg_s = cfg_s if cfg_s is not None else rast_cfg_struct(config, scene.background)
    fr = ViewFrame(camera, 0)
    hw = camera.num_pixels
    if scene.num_gaussians == 0:      # the background image
        fr.rgb = torch.tensor(scene.background, dtype=torch.float64, device=dev).repeat(hw)
        g4 = torch.empty(hw * 4, dtype=torch.float32, device=dev)
        return residual_pass(fr, gt, loss, g4, torch.empty_like(g4)).sum()
    if err is None:
        err = torch.zeros(1, dtype=torch.int32, device=dev)
    project_and_bin(scene, fr, cfg_s, err)
    fr.rgb = torch.empty(hw * 3, dtype=torch.float64, device=dev)
    fr.t_final = torch.empty(hw, dtype=torch.float64, device=dev)
    cnt = torch.zeros(hw + 1, dtype=torch.int32, device=dev)
    a = raster_args(fr, cfg_s)
    a.px_count, a.rgb, a.t_final = ptr(cnt), ptr(fr.rgb), ptr(fr.t_final)
    call("slm_raster_count", _lib.byref(a), stream_ptr())
    g4 = torch.empty(hw * 4, dtype=torch.float32, device=dev)
    c4 = torch.empty(hw * 4, dtype=torch.float32, device=dev)
    part = residual_pass(fr, gt, loss, g4, c4)
    return part.sum()


def energy(scene: GaussianScene, cameras, gts, config=None, loss: LossConfig = LossConfig(), rank: int = 0,
           world_size: int = 1, nonfinite: str = "raise") -> float:
    """sum over views of ||F||^2 (ref: residuals.py:241-246 per view); with
    world_size > 1 the views are sharded round-robin and the partial energies
    summed with one scalar all_reduce (the error flags travel in the same
    buffer, one sync).

    A scene with non-finite parameters or a zero quaternion raises ValueError
    like the reference's render (ref rasterizer.py:81-82, 124-125), or gives
    +inf with nonfinite="inf" (line-search candidates)."""
    from .rasterizer import DEFAULT_CONFIG
    from .solver import allreduce_sum_
    config = config if config is not None else DEFAULT_CONFIG
    cfg_s = rast_cfg_struct(config, scene.background)
    err = torch.zeros(1, dtype=torch.int32, device=scene.device)
    tot = torch.zeros(2, dtype=torch.float64, device=scene.device)
    for i, (c, g) in enumerate(zip(cameras, gts)):
        if i % world_size == rank:
            tot[0] += view_energy(scene, c, g, config, loss, cfg_s, err)
    tot[1] = err[0].to(torch.float64)
    if world_size > 1:
        allreduce_sum_(tot)
    e, flags = tot.tolist()
    if flags != 0:
        if nonfinite == "inf":
            return float("inf")
        raise ValueError("scene contains non-finite parameters" if int(flags) & 1
                         else "quaternion with (near-)zero norm")
    return e


def offset_scene(scene: GaussianScene, delta: torch.Tensor, gamma: float) -> GaussianScene:
    """x + gamma * delta (attribute-major fp32 direction, fp64 scene)."""
    out = torch.empty_like(scene.x)
    call("slm_axpy_scene", ptr(scene.x), ptr(delta.contiguous()), float(gamma), ptr(out), out.numel(),
         stream_ptr())
    return GaussianScene(out, scene.sh_degree, scene.background)


def line_search(scene: GaussianScene, delta: torch.Tensor, cameras, gts, depth: int = 8, config=None,
                loss: LossConfig = LossConfig(), e0: float | None = None, rank: int = 0,
                world_size: int = 1) -> tuple[float, float]:
    """gamma from {1, 1/2, ..., 2^-depth} u {0} minimising the
    energy of the given (strided subset) views; ties go to the smaller gamma.
    Returns (gamma, energy at gamma)."""
    best_g = 0.0
    best_e = energy(scene, cameras, gts, config, loss, rank, world_size) if e0 is None else float(e0)
    for gma in sorted(2.0 ** -i for i in range(depth + 1)):
        e = energy(offset_scene(scene, delta, gma), cameras, gts, config, loss, rank, world_size, nonfinite="inf")
        if e < best_e:
            best_g, best_e = gma, e
    return best_g, best_e


def model_reduction(cache, delta: torch.Tensor, gamma: float) -> float:
    """||F||^2 - ||F + gamma J Delta||^2 on one cache (Eq. 6 denominator)."""
    g = torch.empty_like(delta)
    cache.jtwj(delta, g)
    b = cache.rhs()
    bd = torch.dot(b.double(), delta.double())
    q = torch.dot(delta.double(), g.double())
    return float((2.0 * gamma * bd - gamma * gamma * q).item())


def compute_rho(e_old: float, e_new: float, model_red: float) -> float:
    """Eq. 6; |denominator| < 1e-12 -> -inf (rejection sentinel)."""
    if abs(model_red) < 1e-12:
        return -np.inf
    return (e_old - e_new) / model_red


def trust_region_update(lam: float, rho: float, lam_min: float = LAMBDA_MIN, lam_max: float = LAMBDA_MAX):
    """accept iff rho > 1e-5; lam *= 1 - (2 rho - 1)^3 (clamped),
    else lam doubles (clamped).  Returns (accept, new lam)."""
    if rho > 1e-5:
        return True, float(min(max(lam * (1.0 - (2.0 * rho - 1.0) ** 3), lam_min), lam_max))
    return False, float(min(max(2.0 * lam, lam_min), lam_max))


@dataclass
class LMStepReport:
    scene: GaussianScene
    lam: float
    accepted: bool
    gamma: float
    rho: float
    energy_before: float
    energy_after: float
    delta: torch.Tensor
    direction: object = None     # solver.StepReport of the batched direction (PCG stats, entries)


def lm_step(scene: GaussianScene, cameras, gts, schedule: BatchSchedule = BatchSchedule(), lam: float = 1e-4,
            n_iters: int = 8, ls_fraction: float = 0.3, config=None, loss: LossConfig = LossConfig(),
            rank: int = 0, world_size: int = 1, phase_timer=None) -> LMStepReport:
    """One LM iteration (SPEC lm_fit body): batched direction (Eq. 7), line
    search on a strided ls_fraction of the views (PAPER 3.2), rho on the first
    batch's frozen caches, trust-region accept / revert."""
    n = len(cameras)
    rep = lm_direction(scene, cameras, gts, schedule, lam, n_iters, config, loss, rank, world_size,
                       keep_caches=True, phase_timer=phase_timer)
    delta = rep.delta
    step = max(1, int(round(1.0 / ls_fraction))) if ls_fraction > 0 else 1
    ls_views = list(range(0, n, step))
    ls_c, ls_g = [cameras[i] for i in ls_views], [gts[i] for i in ls_views]
    gamma, _ = line_search(scene, delta, ls_c, ls_g, config=config, loss=loss, rank=rank, world_size=world_size)
    # rho on the rank's first accepted batch; with several ranks, rank 0's
    # value (its first batch is the global first batch) is broadcast so every
    # rank takes the same accept / lambda decision
    rho = -np.inf
    e_old = e_new = float("nan")
    if rep.caches and gamma > 0:
        cs = rep.caches[0]
        v0 = cs.view_ids
        e_old = float(sum(cs.energies))
        e_new = energy(offset_scene(scene, delta, gamma), [cameras[i] for i in v0], [gts[i] for i in v0], config,
                       loss)
        rho = compute_rho(e_old, e_new, model_reduction(cs, delta, gamma))
    if world_size > 1:
        import torch.distributed as dist
        t = torch.tensor([rho], dtype=torch.float64, device=scene.device)
        dist.broadcast(t, 0)
        rho = float(t.item())
    accept, lam_new = trust_region_update(lam, rho)
    new_scene = offset_scene(scene, delta, gamma) if accept else scene
    return LMStepReport(new_scene, lam_new, accept, gamma, rho, e_old, e_new, delta, rep)
