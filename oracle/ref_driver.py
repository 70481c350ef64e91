"""LM direction driven by the REFERENCE's own functions (TEST / BASELINE
INFRASTRUCTURE ONLY -- never imported by the product path).

The reference (`splatlm`, pure numpy) implements render, compute_residuals,
build_cache, sort_cache_by_gaussians, diag_jtj, apply_j, weight_residuals and
apply_jt, but NOT the PCG loop or the Eq. 7 combine (SPEC-only).
This module wires the reference's functions into Alg. 1 (the
same restatement as lm_oracle.pcg) and Eq. 7 so that `bench.py --impl
reference` times the reference's own CPU code for every step that exists in
it.  The package is found, in order, at
  * `baseline/_ref` (pip-installed copy of /root/reference/pkg, git-ignored,
    travels to the GPU box), or
  * `/root/reference/pkg/src` (this container only).
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_CANDIDATES = [os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"]


def import_reference():
    """Return the reference modules (scene, rasterizer, residuals, jacobian, _parallel) or None."""
    for c in _CANDIDATES:
        if os.path.isdir(os.path.join(c, "splatlm")):
            if c not in sys.path:
                sys.path.insert(0, c)
            from splatlm import _parallel, jacobian, rasterizer, residuals, scene
            return dict(scene=scene, rasterizer=rasterizer, residuals=residuals, jacobian=jacobian,
                        parallel=_parallel, path=c)
    return None


def ref_scene(R, host):
    """HostScene (paper_2409_12892_b200.synthetic) -> reference GaussianScene."""
    return R["scene"].GaussianScene(np.asarray(host.positions, float), np.asarray(host.rotations, float),
                                    np.asarray(host.log_scales, float), np.asarray(host.opacity_logits, float),
                                    np.asarray(host.sh_coeffs, float), int(host.sh_degree),
                                    np.asarray(host.background, float))


def ref_camera(R, c):
    return R["scene"].Camera(c.rotation, c.translation, c.fx, c.fy, c.cx, c.cy, c.width, c.height)


def lm_direction(R, scene, cameras, gts, n_batches=1, lam=1e-4, n_iters=8, phases=None):
    """One LM direction with the reference's products (SPEC:400-408 restated).

    scene / cameras are reference objects, gts (H, W, 3) float64 arrays.
    Returns (delta attribute-major float64, entries, phases dict of seconds)."""
    S, RA, RE, J = R["scene"], R["rasterizer"], R["residuals"], R["jacobian"]
    ph = phases if phases is not None else {}

    def tick(name, t0):
        ph[name] = ph.get(name, 0.0) + time.perf_counter() - t0

    n = scene.param_count
    G, P = scene.num_gaussians, scene.params_per_gaussian
    num = np.zeros(n)
    den = np.zeros(n)
    entries = 0
    for j in range(n_batches):
        views = list(range(j, len(cameras), n_batches))        # strided selection
        if not views:
            continue
        caches, bundles = [], []
        b = np.zeros(n)
        M = np.zeros(n)
        for v in views:
            t0 = time.perf_counter()
            rr = RA.render(scene, cameras[v])
            tick("render", t0)
            t0 = time.perf_counter()
            bundle = RE.compute_residuals(rr.image.rgb, gts[v])
            tick("residuals", t0)
            t0 = time.perf_counter()
            bv, cache = J.build_cache(scene, cameras[v], bundle, render_result=rr, view_id=v)
            tick("build_cache", t0)
            t0 = time.perf_counter()
            gc = J.sort_cache_by_gaussians(cache)
            tick("sort", t0)
            t0 = time.perf_counter()
            M += J.diag_jtj(scene, gc).values
            tick("diag", t0)
            b += bv.values
            entries += gc.entry_count
            caches.append(gc)
            bundles.append(bundle)
        Mf = np.maximum(M, 1e-12)

        def A(p):
            t0 = time.perf_counter()
            pg = S.sort_x(S.ParamVector(p, S.Layout.ATTRIBUTE_MAJOR, G, P))
            out = lam * Mf * p
            for gc, bundle in zip(caches, bundles):
                u = J.weight_residuals(J.apply_j(pg, scene, gc), bundle)
                out = out + J.apply_jt(u, scene, gc).values
            tick("pcg_products", t0)
            return out

        # Alg. 1 with SPEC:394-395 exit / abort
        bb = float(b @ b)
        x = b / Mf
        if bb > 0.0:
            r = b - A(x)
            z = r / Mf
            p = z.copy()
            rz = float(r @ z)
            ok = True
            for _ in range(n_iters):
                g = A(p)
                pg_ = float(p @ g)
                if not pg_ > 0.0:
                    ok = False
                    break
                a = rz / pg_
                x = x + a * p
                r = r - a * g
                z = r / Mf
                rz_new = float(r @ z)
                p = z + (rz_new / rz) * p
                rz = rz_new
                if float(r @ r) < 0.01 * bb:
                    break
            if not ok:
                continue
        num += M * x                                             # Eq. 7
        den += M
    return num / np.maximum(den, 1e-12), entries, ph
