"""Shared test helpers: input generation and oracle <-> product conversions."""
import numpy as np

import oracle as O
from paper_2409_12892_b200 import synthetic as S


def oscene(h):
    return O.OScene(np.asarray(h.positions, float), np.asarray(h.rotations, float), np.asarray(h.log_scales, float),
                    np.asarray(h.opacity_logits, float), np.asarray(h.sh_coeffs, float), h.sh_degree,
                    np.asarray(h.background, float))


def ocam(c):
    return O.OCamera(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width, c.height)


def rel(a, b):
    a, b = np.asarray(a, float), np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def problem(seed=0, G=60, n_views=3, W=32, H=28, degree=3, mag=0.1):
    """(truth HostScene, init HostScene, cameras, gt images via the oracle)."""
    truth = S.make_synthetic_scene(seed, G, degree)
    init = S.perturb(truth, seed + 1, mag)
    cams = S.make_camera_ring(n_views, W, H)
    gts = [O.rasterize(oscene(truth), ocam(c))["image"] for c in cams]
    return truth, init, cams, gts
