"""Synthetic inputs (host numpy): the reference's generator, bit-compatible,
and the count/footprint-aware generator for the 1M-Gaussian configurations.

* `make_synthetic_scene` / `perturb` / `make_camera_ring` reproduce
  ref: scene.py:336-413 draw for draw (same numpy Generator call sequence), so
  the C1/C2 configurations get exactly the reference's scenes.  Ground-truth
  images are rendered separately (GPU `render` for the product, the oracle in
  parity tests).
* `make_footprint_scene` keeps the reference's
  distributions for rotation, opacity and SH but ties positions and scales to
  the camera footprint so that a target entries-per-pixel K is hit.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .scene import Camera, GaussianScene, look_at_camera, num_coefficients

PERTURB_SCALES = {"position": 0.12, "rotation": 0.15, "log_scale": 0.15, "opacity_logit": 0.3,
                  "sh_dc": 0.25, "sh_rest": 0.08}  # ref: scene.py:326-333


@dataclass
class HostScene:
    positions: np.ndarray
    rotations: np.ndarray
    log_scales: np.ndarray
    opacity_logits: np.ndarray
    sh_coeffs: np.ndarray
    sh_degree: int
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def num_gaussians(self):
        return self.positions.shape[0]

    def to_device(self, device=None) -> GaussianScene:
        return GaussianScene.from_arrays(self.positions, self.rotations, self.log_scales, self.opacity_logits,
                                         self.sh_coeffs, self.sh_degree, self.background, device)

    def matrix(self):
        g = self.num_gaussians
        return np.concatenate([self.positions, self.rotations, self.log_scales, self.opacity_logits[:, None],
                               self.sh_coeffs.reshape(g, -1)], axis=1)


def make_camera_ring(camera_count: int, width: int, height: int, radius: float = 4.0) -> list[Camera]:
    """ref: scene.py:360-370."""
    cams = []
    f = 1.2 * max(width, height)
    for i in range(camera_count):
        ang = 2.0 * np.pi * i / camera_count
        elev = 0.35 * np.sin(2.1 * ang + 0.4)
        eye = np.array([radius * np.cos(ang), elev * radius * 0.4, radius * np.sin(ang)])
        cams.append(look_at_camera(eye, (0.0, 0.0, 0.0), (0.0, 1.0, 0.0), f, f, width, height))
    return cams


def make_synthetic_scene(seed: int, gaussian_count: int, sh_degree: int = 1, background=(0.0, 0.0, 0.0)):
    """Truth scene of ref: scene.py:373-413 (same draws, same order)."""
    if gaussian_count < 1:
        raise ValueError("gaussian_count must be >= 1")
    rng = np.random.default_rng(seed)
    g, k = gaussian_count, num_coefficients(sh_degree)
    base = rng.uniform(-2.3, -1.55, size=g)
    sh = np.zeros((g, 3, k))
    sh[:, :, 0] = rng.uniform(-0.5, 1.0, size=(g, 3))
    if k > 1:
        sh[:, :, 1:] = rng.uniform(-0.15, 0.15, size=(g, 3, k - 1))
    pos = rng.uniform(-0.9, 0.9, size=(g, 3))
    rot = rng.standard_normal((g, 4)) + np.array([2.0, 0.0, 0.0, 0.0])
    ls = base[:, None] + rng.uniform(0.0, 1.0, size=(g, 3))
    op = rng.uniform(-1.0, 2.0, size=g)
    return HostScene(pos, rot, ls, op, sh, sh_degree, np.asarray(background, np.float64))


def perturb(scene: HostScene, seed: int, magnitude: float) -> HostScene:
    """ref: scene.py:336-357 (same draws, same order, same float expression order)."""
    if magnitude < 0:
        raise ValueError("perturbation magnitude must be >= 0")
    if magnitude == 0:
        return scene
    rng = np.random.default_rng(seed)
    g, k = scene.num_gaussians, num_coefficients(scene.sh_degree)
    noise = np.zeros((g, 3, k))
    noise[:, :, 0] = PERTURB_SCALES["sh_dc"] * rng.standard_normal((g, 3))
    if k > 1:
        noise[:, :, 1:] = PERTURB_SCALES["sh_rest"] * rng.standard_normal((g, 3, k - 1))
    S = PERTURB_SCALES
    return HostScene(
        positions=scene.positions + magnitude * S["position"] * rng.standard_normal((g, 3)),
        rotations=scene.rotations + magnitude * S["rotation"] * rng.standard_normal((g, 4)),
        log_scales=scene.log_scales + magnitude * S["log_scale"] * rng.standard_normal((g, 3)),
        opacity_logits=scene.opacity_logits + magnitude * S["opacity_logit"] * rng.standard_normal(g),
        sh_coeffs=scene.sh_coeffs + magnitude * noise,
        sh_degree=scene.sh_degree, background=scene.background)


def make_footprint_scene(seed: int, gaussian_count: int, width: int, height: int, sh_degree: int = 3,
                         k_target: float = 32.0, radius: float = 1.45, cam_radius: float = 4.0,
                         background=(0.0, 0.0, 0.0)) -> HostScene:
    """Count/footprint-aware generator for C3-C5.

    Gaussians fill a ball of `radius` seen by a camera ring at `cam_radius`
    with f = 1.2 max(W, H).  The mean pixel footprint is chosen so that the
    expected number of (pixel, splat) entries per pixel is ~`k_target`:
    an isotropic splat of pixel std s and opacity o covers
    2 pi ln(255 o) (s^2 + cov_eps) pixels above alpha_min (RenderConfig).
    Rotation / opacity / SH distributions are the reference's (scene.py:397-410).
    """
    rng = np.random.default_rng(seed)
    g, k = gaussian_count, num_coefficients(sh_degree)
    f = 1.2 * max(width, height)
    # fraction of the frame covered by the ball's silhouette
    half_w = 0.5 * width / f * cam_radius
    half_h = 0.5 * height / f * cam_radius
    cover = min(1.0, np.pi * radius * radius / (4.0 * half_w * half_h))
    mean_area = k_target / cover * width * height / g          # pixels per splat
    o_mean_log = 5.0                                            # E[ln(255 o)] for logit ~ U(-1, 2)
    s2_px = max(mean_area / (2.0 * np.pi * o_mean_log) - 0.3, 0.05)
    s_world = np.sqrt(s2_px) * cam_radius / f
    # uniform in the ball
    u = rng.uniform(0.0, 1.0, size=g) ** (1.0 / 3.0)
    d = rng.standard_normal((g, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    pos = radius * u[:, None] * d
    rot = rng.standard_normal((g, 4)) + np.array([2.0, 0.0, 0.0, 0.0])
    ls = np.log(s_world) + rng.uniform(-0.35, 0.35, size=g)[:, None] + rng.uniform(-0.35, 0.35, size=(g, 3))
    op = rng.uniform(-1.0, 2.0, size=g)
    sh = np.zeros((g, 3, k))
    sh[:, :, 0] = rng.uniform(-0.5, 1.0, size=(g, 3))
    if k > 1:
        sh[:, :, 1:] = rng.uniform(-0.15, 0.15, size=(g, 3, k - 1))
    return HostScene(pos, rot, ls, op, sh, sh_degree, np.asarray(background, np.float64))
