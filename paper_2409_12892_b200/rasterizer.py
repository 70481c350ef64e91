"""Forward rendering with traversal records on the device.

Mirrors ref: rasterizer.py (RenderConfig 22-48, ProjectedSplats 63-75,
project_scene 116-165, Traversals 209-243, render 319-358) with a 16x16 tile
rasteriser in fp64 (csrc/raster.cu).  Traversal records are produced by the
same FILL pass that writes the gradient cache.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import call, ptr, stream_ptr
from .engine import ViewFrame, project_and_bin, rast_cfg_struct, raster_args, scan_i64
from .scene import Camera, GaussianScene


@dataclass(frozen=True)
class RenderConfig:
    """ref: rasterizer.py:22-48."""
    alpha_min: float = 1.0 / 255.0
    t_stop: float = 1e-4
    alpha_clamp: float = 0.99
    cov_eps: float = 0.3
    z_near: float = 0.01
    cull_sigma: float | None = 3.33

    @staticmethod
    def smooth() -> "RenderConfig":
        return RenderConfig(alpha_min=0.0, t_stop=0.0, cull_sigma=None)


DEFAULT_CONFIG = RenderConfig()


@dataclass
class ProjectedSplats:
    """Device struct-of-arrays view of one view's projected splats."""
    mean2d: torch.Tensor
    conic: torch.Tensor
    opacity: torch.Tensor
    color: torch.Tensor
    color_clamped: torch.Tensor
    valid: torch.Tensor
    bbox: torch.Tensor

    @staticmethod
    def from_bytes(raw: torch.Tensor, G: int) -> "ProjectedSplats":
        rec = raw.view(G, 96)
        d = rec[:, :72].contiguous().view(torch.float64).view(G, 9)
        ints = rec[:, 72:96].contiguous().view(torch.int32).view(G, 6)
        flags = ints[:, 4]
        return ProjectedSplats(mean2d=d[:, 0:2], conic=d[:, 2:5], opacity=d[:, 5], color=d[:, 6:9],
                               color_clamped=torch.stack([(flags >> (1 + c)) & 1 for c in range(3)], 1).bool(),
                               valid=(flags & 1).bool(), bbox=ints[:, 0:4])


def project_scene(scene: GaussianScene, camera: Camera, config: RenderConfig = DEFAULT_CONFIG) -> ProjectedSplats:
    if scene.num_gaussians == 0:
        return ProjectedSplats.from_bytes(torch.empty(0, dtype=torch.uint8, device=scene.device), 0)
    fr = ViewFrame(camera, 0)
    err = torch.zeros(1, dtype=torch.int32, device=scene.device)
    project_and_bin(scene, fr, rast_cfg_struct(config, scene.background), err, depth_only=True)
    _raise_scene_err(int(err.item()))
    return ProjectedSplats.from_bytes(fr.splats, scene.num_gaussians)


def _raise_scene_err(e: int):
    if e & 1:
        raise ValueError("scene contains non-finite parameters")
    if e & 2:
        raise ValueError("quaternion with (near-)zero norm")


@dataclass
class Traversals:
    """Per-pixel traversal records, pixel-sorted, front to back (ref: rasterizer.py:209-243)."""
    pixel_ids: torch.Tensor
    gaussian_ids: torch.Tensor
    alphas: torch.Tensor
    transmittances: torch.Tensor
    offsets: torch.Tensor
    t_final: torch.Tensor
    splat_colors: torch.Tensor
    width: int
    height: int

    @property
    def entry_count(self) -> int:
        return int(self.pixel_ids.shape[0])


@dataclass
class RenderResult:
    image: torch.Tensor          # (H, W, 3) float64
    traversals: Traversals | None
    splats: ProjectedSplats


def render(scene: GaussianScene, camera: Camera, config: RenderConfig = DEFAULT_CONFIG,
           traversals: bool = True) -> RenderResult:
    """ref: rasterizer.py:319-358."""
    dev = scene.device
    G = scene.num_gaussians
    if G == 0:
        return _render_empty(scene, camera, traversals)
    cfg_s = rast_cfg_struct(config, scene.background)
    fr = ViewFrame(camera, 0)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    project_and_bin(scene, fr, cfg_s, err)
    _raise_scene_err(int(err.item()))
    hw = camera.num_pixels
    cnt = torch.zeros(hw + 1, dtype=torch.int32, device=dev)
    pair_cnt = torch.zeros(G, dtype=torch.int32, device=dev)
    fr.rgb = torch.empty(hw * 3, dtype=torch.float64, device=dev)
    fr.t_final = torch.empty(hw, dtype=torch.float64, device=dev)
    a = raster_args(fr, cfg_s)
    a.px_count, a.rgb, a.t_final = ptr(cnt), ptr(fr.rgb), ptr(fr.t_final)
    inst_mask = torch.zeros(max(fr.n_inst, 1) * 8, dtype=torch.int32, device=dev) if traversals else None
    a.inst_mask = ptr(inst_mask)
    call("slm_raster_count", _lib.byref(a), stream_ptr())
    splats = ProjectedSplats.from_bytes(fr.splats, G)
    image = fr.rgb.view(camera.height, camera.width, 3)
    if not traversals:
        return RenderResult(image, None, splats)
    cnt64 = cnt.to(torch.int64)
    off = torch.empty_like(cnt64)
    scan_i64(cnt64, off)
    E = int(off[hw].item())
    tg = torch.empty(max(E, 1), dtype=torch.int64, device=dev)
    ta = torch.empty(max(E, 1), dtype=torch.float64, device=dev)
    tt = torch.empty(max(E, 1), dtype=torch.float64, device=dev)
    a = raster_args(fr, cfg_s)
    a.rgb, a.pix_off, a.inst_mask = ptr(fr.rgb), ptr(off), ptr(inst_mask)
    a.trav_gid, a.trav_alpha, a.trav_T = ptr(tg), ptr(ta), ptr(tt)
    call("slm_raster_fill", _lib.byref(a), stream_ptr())
    pix = torch.repeat_interleave(torch.arange(hw, device=dev), (off[1:] - off[:-1]))
    tr = Traversals(pixel_ids=pix, gaussian_ids=tg[:E], alphas=ta[:E], transmittances=tt[:E], offsets=off,
                    t_final=fr.t_final, splat_colors=splats.color, width=camera.width, height=camera.height)
    return RenderResult(image, tr, splats)


def _render_empty(scene: GaussianScene, camera: Camera, traversals: bool) -> RenderResult:
    """an empty scene renders the background with empty traversals."""
    dev = scene.device
    hw = camera.num_pixels
    bg = torch.tensor(scene.background, dtype=torch.float64, device=dev)
    image = bg.expand(camera.height, camera.width, 3).contiguous()
    splats = project_scene(scene, camera)
    if not traversals:
        return RenderResult(image, None, splats)
    e64 = torch.empty(0, dtype=torch.int64, device=dev)
    ef = torch.empty(0, dtype=torch.float64, device=dev)
    tr = Traversals(pixel_ids=e64, gaussian_ids=e64.clone(), alphas=ef, transmittances=ef.clone(),
                    offsets=torch.zeros(hw + 1, dtype=torch.int64, device=dev),
                    t_final=torch.ones(hw, dtype=torch.float64, device=dev), splat_colors=splats.color,
                    width=camera.width, height=camera.height)
    return RenderResult(image, tr, splats)
