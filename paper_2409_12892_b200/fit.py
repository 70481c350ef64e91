"""Stage 1 (ADAM), the LM fit loop and the two-stage driver (SURVEY 8(f) row
4).  The reference ships these as SPEC only (lm_fit, adam_fit,
two_stage_fit; no code under pkg/), so this module restates the SPEC on top
of the device path:

* the loss gradient is the cache build's right-hand side: E = sum r^2 and
  b = -J^T color_grad with color_grad = sum_terms r dr/dc (ref
  jacobian.py:411-413, residuals.py:293-294), so dE/dx = -2 b, formed by the
  same kernels as the LM products ("gradient computed analytically
  via the same chain as the Jacobian module");
* ADAM (beta1 0.9, beta2 0.999, eps 1e-15) with the SPEC's per-class learning
  rates (SPEC DESIGN DECISIONS), one random image per iteration (batch size
  1, PAPER 3.1), seeded;
* lm_fit: lm_step per outer iteration, full-training-set energy
  recorded every iteration, lambda escalation on a failed solve until
  lambda_max (then the error propagates);
* two_stage_fit: adam_fit for K iterations, then lm_fit, history labelled by
  stage.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np
import torch

from .engine import CacheSet, LossConfig
from .errors import NonSPDError
from .lm import LAMBDA_MAX, energy, lm_step
from .scene import GaussianScene
from .solver import BatchSchedule

# SPEC DESIGN DECISIONS: per-class ADAM learning rates (3DGS-style defaults)
ADAM_LR = {"position": 1.6e-4, "rotation": 1e-3, "log_scale": 5e-3, "opacity": 5e-2, "sh": 2.5e-3}
# attribute rows of the attribute-major parameter vector (ref scene.py:17-36)
_CLASS_ROWS = {"position": (0, 3), "rotation": (3, 7), "log_scale": (7, 10), "opacity": (10, 11)}


@dataclass
class FitRecord:
    """One history row (SPEC RunReport / convergence.csv columns)."""
    iteration: int
    stage: str            # "adam" | "lm"
    energy: float         # adam: the sampled image's energy before the step; lm: full training set after it
    accepted: bool
    lam: float
    gamma: float
    time_s: float


def learning_rates(scene: GaussianScene, lr: dict | None = None) -> torch.Tensor:
    """Attribute-major per-parameter learning rates (fp64) from per-class rates."""
    lr = {**ADAM_LR, **(lr or {})}
    G, P = scene.num_gaussians, scene.params_per_gaussian
    rows = torch.full((P,), float(lr["sh"]), dtype=torch.float64)
    for cls, (a, b) in _CLASS_ROWS.items():
        rows[a:b] = float(lr[cls])
    return rows.repeat_interleave(G).to(scene.device)


def loss_gradient(scene: GaussianScene, camera, gt: torch.Tensor, config=None,
                  loss: LossConfig = LossConfig()) -> tuple[torch.Tensor, float]:
    """(dE/dx attribute-major fp64, E) for one image: E = sum r^2 and
    dE/dx = -2 b with b from the cache build (one-view CacheSet + its rhs).
    Raises ValueError on a non-finite gradient."""
    cs = CacheSet(scene, [camera], [gt.to(scene.device)], config, loss)
    g = cs.rhs().double().mul_(-2.0)
    e = float(sum(cs.energies))
    del cs
    if not bool(torch.isfinite(g).all()):
        raise ValueError("non-finite loss gradient")
    return g, e


def adam_fit(scene: GaussianScene, cameras, gts, iters: int = 200, lr: dict | None = None,
             betas=(0.9, 0.999), eps: float = 1e-15, seed: int = 0, config=None,
             loss: LossConfig = LossConfig(), history: list | None = None):
    """ADAM on Eq. 2, one random image per iteration (seeded).
    Returns (scene', history)."""
    history = [] if history is None else history
    b1, b2 = betas
    lrv = learning_rates(scene, lr)
    x = scene.x.clone()
    m = torch.zeros_like(x)
    v = torch.zeros_like(x)
    rng = np.random.RandomState(seed)
    t0 = time.perf_counter()
    for t in range(1, iters + 1):
        i = int(rng.randint(len(cameras)))
        g, e = loss_gradient(GaussianScene(x, scene.sh_degree, scene.background), cameras[i], gts[i], config, loss)
        m.mul_(b1).add_(g, alpha=1.0 - b1)
        v.mul_(b2).addcmul_(g, g, value=1.0 - b2)
        mh = m / (1.0 - b1 ** t)
        vh = v / (1.0 - b2 ** t)
        x.sub_(lrv * mh / (vh.sqrt() + eps))
        history.append(FitRecord(t, "adam", e, True, 0.0, 0.0, time.perf_counter() - t0))
    return GaussianScene(x, scene.sh_degree, scene.background), history


def lm_fit(scene: GaussianScene, cameras, gts, n_iters: int = 5, pcg_iters: int = 8, n_batches: int = 1,
           lam: float = 1e-4, ls_fraction: float = 0.3, config=None, loss: LossConfig = LossConfig(),
           history: list | None = None, rank: int = 0, world_size: int = 1):
    """n_iters LM iterations (batched direction, line search,
    rho, trust region).  A failed solve (every batch non-SPD) doubles lambda
    and retries; past lambda_max the error propagates.  Returns (scene',
    lambda, history); history row 0 is the starting energy."""
    history = [] if history is None else history
    t0 = time.perf_counter()
    sched = BatchSchedule(n_batches)
    e = energy(scene, cameras, gts, config, loss, rank, world_size)
    history.append(FitRecord(0, "lm", e, True, lam, 0.0, 0.0))
    for it in range(1, n_iters + 1):
        while True:
            try:
                st = lm_step(scene, cameras, gts, sched, lam, pcg_iters, ls_fraction, config, loss, rank, world_size)
                break
            except NonSPDError:
                if lam >= LAMBDA_MAX:
                    raise
                lam = min(2.0 * lam, LAMBDA_MAX)
        if st.accepted:
            scene = st.scene
            e = energy(scene, cameras, gts, config, loss, rank, world_size)
        lam = st.lam
        history.append(FitRecord(it, "lm", e, st.accepted, lam, st.gamma, time.perf_counter() - t0))
    return scene, lam, history


def two_stage_fit(scene: GaussianScene, cameras, gts, stage1_iters: int = 200, lm_iters: int = 5,
                  pcg_iters: int = 8, n_batches: int = 1, lam: float = 1e-4, lr: dict | None = None,
                  seed: int = 0, config=None, loss: LossConfig = LossConfig()):
    """adam_fit for stage1_iters (K), then lm_fit; one history
    with stage labels ("adam" rows, then "lm" rows).  Returns (scene', history)."""
    history: list[FitRecord] = []
    if stage1_iters > 0:
        scene, history = adam_fit(scene, cameras, gts, stage1_iters, lr, seed=seed, config=config, loss=loss,
                                  history=history)
    scene, _, history = lm_fit(scene, cameras, gts, lm_iters, pcg_iters, n_batches, lam, config=config, loss=loss,
                               history=history)
    return scene, history
