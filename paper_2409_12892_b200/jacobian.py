"""Gradient cache and matrix-free Jacobian products -- reference API.

Mirrors ref: jacobian.py (CacheOrder 37-39, CacheOrderError 42-43,
GradientCache 46-84, sort_cache_by_gaussians 93-105, sort_cache_by_pixels
108-121, build_cache 360-416, apply_j 419-455, weight_residuals 458-464,
apply_jt 467-483, diag_jtj 486-512, dump_cache / load_cache_dump 618-656).

A GradientCache wraps a device CacheSet (engine.py) that holds BOTH record
orders; the order tag keeps the reference's contract (apply_jt / diag_jtj
require a gaussian-sorted cache) while sorting is a tag flip on already-built
streams.  Multi-view caches (one Eq. 7 batch) are products summed over views
(SPEC:393).
"""

from __future__ import annotations

import enum
import struct
from dataclasses import dataclass, replace

import numpy as np
import torch

from .engine import CacheSet, LossConfig
from .errors import CacheOrderError
from .rasterizer import DEFAULT_CONFIG, RenderConfig
from .residuals import ResidualBundle
from .scene import Camera, GaussianScene, Layout, ParamVector


class CacheOrder(enum.Enum):
    PIXEL_SORTED = "pixel"
    GAUSSIAN_SORTED = "gaussian"


@dataclass(frozen=True, eq=False)
class GradientCache:
    cacheset: CacheSet
    order: CacheOrder
    view_id: int = 0

    @property
    def camera(self) -> Camera:
        return self.cacheset.cameras[0]

    @property
    def n_gaussians(self) -> int:
        return self.cacheset.G

    @property
    def config(self) -> RenderConfig:
        return self.cacheset.config

    @property
    def entry_count(self) -> int:
        return self.cacheset.E

    @property
    def nbytes(self) -> int:
        return self.cacheset.nbytes

    def require_order(self, order: CacheOrder) -> None:
        if self.order is not order:
            raise CacheOrderError(f"expected {order.value}-sorted cache, got {self.order.value}")

    def export(self, v: int = 0) -> dict:
        return self.cacheset.export_view(v)


def build_cache(scene: GaussianScene, camera, bundle: ResidualBundle | list, config: RenderConfig = DEFAULT_CONFIG,
                render_result=None, view_id: int = 0):
    """b = -J^T F and the (pixel-sorted) cache; `camera` may be a list of views
    with a matching list of bundles (one Eq. 7 batch).  `render_result` is
    accepted for signature compatibility (ref: jacobian.py:360-363) and not
    needed: the device build re-runs the fp64 rasteriser (COUNT + FILL), which
    is cheaper than shipping a host Traversals back to the GPU."""
    cams = camera if isinstance(camera, (list, tuple)) else [camera]
    bundles = bundle if isinstance(bundle, (list, tuple)) else [bundle]
    if len(cams) != len(bundles):
        raise ValueError("one residual bundle per camera is required")
    for c, b in zip(cams, bundles):
        if (b.height, b.width) != (c.height, c.width):
            raise ValueError("residual bundle does not match the camera resolution")
    cs = CacheSet(scene, list(cams), None, config, LossConfig(), weights=[(b.gradr4, b.cgrad4) for b in bundles])
    b = ParamVector(cs.rhs().clone(), Layout.ATTRIBUTE_MAJOR, scene.num_gaussians, scene.params_per_gaussian)
    return b, GradientCache(cs, CacheOrder.PIXEL_SORTED, view_id)


def sort_cache_by_gaussians(cache: GradientCache) -> GradientCache:
    cache.require_order(CacheOrder.PIXEL_SORTED)
    return replace(cache, order=CacheOrder.GAUSSIAN_SORTED)


def sort_cache_by_pixels(cache: GradientCache) -> GradientCache:
    cache.require_order(CacheOrder.GAUSSIAN_SORTED)
    return replace(cache, order=CacheOrder.PIXEL_SORTED)


def apply_j(p: ParamVector, scene: GaussianScene, cache: GradientCache) -> torch.Tensor:
    """u_hat = J p (unweighted), 3 slots per pixel, views concatenated; p gaussian-major."""
    p.require_layout(Layout.GAUSSIAN_MAJOR)
    if len(p) != scene.param_count:
        raise ValueError(f"parameter vector length {len(p)} does not match scene ({scene.param_count})")
    cs = cache.cacheset
    cs.pair_forward(p.values.float().contiguous(), gaussian_major=True)
    u = cs.apply_j_raw(weighted=False)
    return u.view(-1, 4)[:, :3].reshape(-1).clone()


def weight_residuals(u_hat: torch.Tensor, bundle: ResidualBundle) -> torch.Tensor:
    w = bundle.grad_r_sq.reshape(-1)
    if tuple(u_hat.shape) != tuple(w.shape):
        raise ValueError(f"length mismatch: {tuple(u_hat.shape)} vs {tuple(w.shape)}")
    return u_hat * w.to(u_hat.dtype)


def apply_jt(u: torch.Tensor, scene: GaussianScene, cache: GradientCache) -> ParamVector:
    cache.require_order(CacheOrder.GAUSSIAN_SORTED)
    cs = cache.cacheset
    if tuple(u.shape) != (cs.N * 3,):
        raise ValueError(f"expected color-space vector of length {cs.N * 3}, got {tuple(u.shape)}")
    u4 = torch.zeros(cs.N, 4, dtype=torch.float32, device=cs.device)
    u4[:, :3] = u.view(-1, 3).float()
    out = torch.empty(scene.param_count, dtype=torch.float32, device=cs.device)
    cs.apply_jt_raw(u4.view(-1), out)
    return ParamVector(out, Layout.ATTRIBUTE_MAJOR, scene.num_gaussians, scene.params_per_gaussian)


def diag_jtj(scene: GaussianScene, cache: GradientCache) -> ParamVector:
    cache.require_order(CacheOrder.GAUSSIAN_SORTED)
    M = cache.cacheset.diag()
    return ParamVector(M.clone(), Layout.ATTRIBUTE_MAJOR, scene.num_gaussians, scene.params_per_gaussian)


# ---------------------------------------------------------------------------
# GCCH debug dump, byte-compatible with ref: jacobian.py:618-656
# ---------------------------------------------------------------------------
_DUMP_MAGIC = b"GCCH"


def dump_cache(cache: GradientCache, path, view: int = 0) -> None:
    ex = cache.export(view)
    gs = cache.order is CacheOrder.GAUSSIAN_SORTED
    if gs:
        sel = ex["g_source_index"]
    else:
        sel = np.arange(ex["pixel_ids"].size)
    n = sel.size
    packed = np.empty((n, 8), dtype="<f8")
    packed[:, 0] = ex["pixel_ids"][sel]
    packed[:, 1] = ex["gaussian_ids"][sel]
    packed[:, 2] = ex["alphas"][sel]
    packed[:, 3] = ex["transmittances"][sel]
    packed[:, 4:7] = ex["dc_dalpha"][sel]
    packed[:, 7] = ex["dc_dcs"][sel]
    cam = cache.cacheset.cameras[view]
    with open(path, "wb") as f:
        f.write(_DUMP_MAGIC)
        f.write(struct.pack("<QBII", n, 1 if gs else 0, cam.num_pixels, cache.n_gaussians))
        f.write(packed.tobytes())


def load_cache_dump(path) -> dict:
    with open(path, "rb") as f:
        if f.read(4) != _DUMP_MAGIC:
            raise ValueError("not a cache dump file")
        n, order, n_pixels, n_gaussians = struct.unpack("<QBII", f.read(17))
        packed = np.frombuffer(f.read(n * 64), dtype="<f8").reshape(-1, 8)
    return {"order": CacheOrder.PIXEL_SORTED if order == 0 else CacheOrder.GAUSSIAN_SORTED,
            "n_pixels": n_pixels, "n_gaussians": n_gaussians,
            "pixel_ids": packed[:, 0].astype(np.int64), "gaussian_ids": packed[:, 1].astype(np.int64),
            "alphas": packed[:, 2].copy(), "transmittances": packed[:, 3].copy(),
            "dc_dalpha": packed[:, 4:7].copy(), "dc_dcs": packed[:, 7].copy()}
