"""float64 numpy restatement of the 3DGS-LM solver path (TEST INFRASTRUCTURE ONLY).

Every function names the reference lines it restates.  `ref:` paths are
relative to /root/reference/pkg/src/splatlm/; `SPEC:` / `PAPER:` are
/root/reference/SPEC.md and PAPER.md.

Representation: a scene is an `OScene` (struct of float64 arrays), a camera an
`OCamera`; parameters are handled as a (G, P) matrix whose column order is the
reference's per-Gaussian attribute order (ref: scene.py:17-19): position 3,
quaternion wxyz 4, log scale 3, opacity logit 1, SH channel-major R[K] G[K] B[K].
Attribute-major flat index = a*G + g, gaussian-major = g*P + a (ref: scene.py:79-92).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "GEOM", "OConfig", "OScene", "OCamera", "OView", "NonSPDError",
    "sh_basis", "sh_basis_grad", "n_coeffs", "params_per_gaussian",
    "scene_matrix", "scene_from_matrix", "am_from_matrix", "matrix_from_am",
    "gm_from_am", "am_from_gm",
    "project", "rasterize", "ssim_blur", "center_weights", "residuals",
    "build_cache", "gaussian_order", "splat_tables", "apply_j", "apply_jt",
    "diag_jtj", "weight", "jtwj", "pcg", "combine", "strided_batches",
    "lm_direction", "energy", "line_search", "compute_rho", "trust_region_update",
]

GEOM = 11          # ref: scene.py:29
COLOR_OFFSET = 0.5  # ref: sh.py:28
M_FLOOR = 1e-12    # SPEC:474 (Jacobi floor and Eq. 7 denominator floor)


class NonSPDError(RuntimeError):
    """p^T g <= 0 inside PCG."""


@dataclass(frozen=True)
class OConfig:
    """ref: rasterizer.py:22-48 (RenderConfig)."""
    alpha_min: float = 1.0 / 255.0
    t_stop: float = 1e-4
    alpha_clamp: float = 0.99
    cov_eps: float = 0.3
    z_near: float = 0.01
    cull_sigma: float | None = 3.33


@dataclass
class OScene:
    pos: np.ndarray        # (G,3)
    quat: np.ndarray       # (G,4) wxyz, unnormalised
    log_scale: np.ndarray  # (G,3)
    logit: np.ndarray      # (G,)
    sh: np.ndarray         # (G,3,K)
    degree: int
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @property
    def G(self):
        return self.pos.shape[0]

    @property
    def P(self):
        return params_per_gaussian(self.degree)


@dataclass
class OCamera:
    R: np.ndarray   # (3,3) world->camera
    t: np.ndarray   # (3,)
    fx: float
    fy: float
    cx: float
    cy: float
    width: int
    height: int

    @property
    def center(self):
        return -self.R.T @ self.t


def n_coeffs(degree):
    return (degree + 1) ** 2


def params_per_gaussian(degree):
    return GEOM + 3 * n_coeffs(degree)


# ---------------------------------------------------------------------------
# SH basis as explicit polynomials (ref: sh.py:11-135).  Each basis function is
# a list of monomials (coefficient, power_x, power_y, power_z); values and
# gradients are evaluated from the same table.
# ---------------------------------------------------------------------------
_K0 = 0.28209479177387814
_K1 = 0.4886025119029199
_K2 = (1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
       -1.0925484305920792, 0.5462742152960396)
_K3 = (-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
       0.3731763325901154, -0.4570457994644658, 1.445305721320277,
       -0.5900435899266435)

_SH_POLY = [
    [(_K0, 0, 0, 0)],
    [(-_K1, 0, 1, 0)],
    [(_K1, 0, 0, 1)],
    [(-_K1, 1, 0, 0)],
    [(_K2[0], 1, 1, 0)],
    [(_K2[1], 0, 1, 1)],
    [(2 * _K2[2], 0, 0, 2), (-_K2[2], 2, 0, 0), (-_K2[2], 0, 2, 0)],
    [(_K2[3], 1, 0, 1)],
    [(_K2[4], 2, 0, 0), (-_K2[4], 0, 2, 0)],
    [(3 * _K3[0], 2, 1, 0), (-_K3[0], 0, 3, 0)],
    [(_K3[1], 1, 1, 1)],
    [(4 * _K3[2], 0, 1, 2), (-_K3[2], 2, 1, 0), (-_K3[2], 0, 3, 0)],
    [(2 * _K3[3], 0, 0, 3), (-3 * _K3[3], 2, 0, 1), (-3 * _K3[3], 0, 2, 1)],
    [(4 * _K3[4], 1, 0, 2), (-_K3[4], 3, 0, 0), (-_K3[4], 1, 2, 0)],
    [(_K3[5], 2, 0, 1), (-_K3[5], 0, 2, 1)],
    [(_K3[6], 3, 0, 0), (-3 * _K3[6], 1, 2, 0)],
]


def _pow(v, n):
    return np.ones_like(v) if n == 0 else v ** n


def sh_basis(dirs, degree):
    """ref: sh.py:38-77."""
    x, y, z = dirs[:, 0], dirs[:, 1], dirs[:, 2]
    out = np.zeros((dirs.shape[0], n_coeffs(degree)))
    for k in range(n_coeffs(degree)):
        for c, a, b, d in _SH_POLY[k]:
            out[:, k] += c * _pow(x, a) * _pow(y, b) * _pow(z, d)
    return out


def sh_basis_grad(dirs, degree):
    """d basis / d direction, (N, K, 3) (ref: sh.py:80-135)."""
    x, y, z = dirs[:, 0], dirs[:, 1], dirs[:, 2]
    out = np.zeros((dirs.shape[0], n_coeffs(degree), 3))
    for k in range(n_coeffs(degree)):
        for c, a, b, d in _SH_POLY[k]:
            if a:
                out[:, k, 0] += c * a * _pow(x, a - 1) * _pow(y, b) * _pow(z, d)
            if b:
                out[:, k, 1] += c * b * _pow(x, a) * _pow(y, b - 1) * _pow(z, d)
            if d:
                out[:, k, 2] += c * d * _pow(x, a) * _pow(y, b) * _pow(z, d - 1)
    return out


# ---------------------------------------------------------------------------
# Parameter layouts (ref: scene.py:79-92, 220-258)
# ---------------------------------------------------------------------------

def scene_matrix(s: OScene):
    """(G, P) per-Gaussian parameter matrix in the reference attribute order."""
    return np.concatenate([s.pos, s.quat, s.log_scale, s.logit[:, None],
                           s.sh.reshape(s.G, -1)], axis=1)


def scene_from_matrix(mat, degree, background):
    k = n_coeffs(degree)
    return OScene(pos=mat[:, 0:3].copy(), quat=mat[:, 3:7].copy(),
                  log_scale=mat[:, 7:10].copy(), logit=mat[:, 10].copy(),
                  sh=mat[:, 11:].reshape(-1, 3, k).copy(), degree=degree,
                  background=np.asarray(background, dtype=np.float64))


def am_from_matrix(mat):
    return np.ascontiguousarray(mat.T).reshape(-1)


def matrix_from_am(v, G):
    return v.reshape(-1, G).T


def gm_from_am(v, G):
    """sort_x (ref: scene.py:79-84)."""
    return np.ascontiguousarray(v.reshape(-1, G).T).reshape(-1)


def am_from_gm(v, G):
    """sort_x_inverse (ref: scene.py:87-92)."""
    return np.ascontiguousarray(v.reshape(G, -1).T).reshape(-1)


# ---------------------------------------------------------------------------
# Projection (ref: rasterizer.py:78-165)
# ---------------------------------------------------------------------------

def _rotations(quat):
    """Unit-quaternion rotation matrices, plus q_hat and |q| (ref: rasterizer.py:78-94)."""
    nrm = np.linalg.norm(quat, axis=1)
    if np.any(nrm < 1e-12):
        raise ValueError("quaternion with (near-)zero norm")
    qh = quat / nrm[:, None]
    w, x, y, z = qh[:, 0], qh[:, 1], qh[:, 2], qh[:, 3]
    R = np.stack([
        np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)], -1),
        np.stack([2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)], -1),
        np.stack([2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1),
    ], -2)
    return R, qh, nrm


def project(s: OScene, cam: OCamera, cfg: OConfig = OConfig()):
    """Per-Gaussian 2D splats for one view (ref: rasterizer.py:116-165).

    Returns a dict: mean (G,2), cov (G,3) packed a,b,c incl. cov_eps, conic
    (G,3), depth, color (G,3), clamped (G,3) bool, opacity, valid (G,) bool,
    cam (G,3) camera-space points.
    """
    arrs = (s.pos, s.quat, s.log_scale, s.logit, s.sh, s.background)
    if not all(np.isfinite(a).all() for a in arrs):
        raise ValueError("scene contains non-finite parameters")
    X = s.pos @ cam.R.T + cam.t
    valid = X[:, 2] > cfg.z_near
    zz = np.where(valid, X[:, 2], 1.0)
    mean = np.stack([cam.fx * X[:, 0] / zz + cam.cx, cam.fy * X[:, 1] / zz + cam.cy], 1)

    Rg, _, _ = _rotations(s.quat)
    s2 = np.exp(2.0 * s.log_scale)
    cov_w = (Rg * s2[:, None, :]) @ np.swapaxes(Rg, 1, 2)
    Xs = np.where(valid[:, None], X, np.array([0.0, 0.0, 1.0]))
    A = _proj_jac(Xs, cam)
    U = A @ cam.R                                     # (G,2,3)
    cov2 = U @ cov_w @ np.swapaxes(U, 1, 2)
    va = cov2[:, 0, 0] + cfg.cov_eps
    vb = cov2[:, 0, 1]
    vc = cov2[:, 1, 1] + cfg.cov_eps
    det = va * vc - vb * vb
    valid = valid & (det > 0)
    det = np.where(det > 0, det, 1.0)
    conic = np.stack([vc / det, -vb / det, va / det], 1)

    d = s.pos - cam.center
    d = d / np.linalg.norm(d, axis=1, keepdims=True)
    raw = np.einsum("gck,gk->gc", s.sh, sh_basis(d, s.degree)) + COLOR_OFFSET
    color = np.maximum(raw, 0.0)

    if cfg.cull_sigma is not None:
        lam = 0.5 * (va + vc) + np.sqrt(0.25 * (va - vc) ** 2 + vb * vb)
        rad = cfg.cull_sigma * np.sqrt(lam)
        valid = (valid & (mean[:, 0] + rad > 0) & (mean[:, 0] - rad < cam.width)
                 & (mean[:, 1] + rad > 0) & (mean[:, 1] - rad < cam.height))
    opacity = 1.0 / (1.0 + np.exp(-s.logit))
    return dict(mean=mean, cov=np.stack([va, vb, vc], 1), conic=conic, depth=X[:, 2],
                color=color, clamped=raw <= 0.0, opacity=opacity, valid=valid, cam=X)


def _proj_jac(X, cam):
    """ref: rasterizer.py:104-113."""
    iz = 1.0 / X[:, 2]
    A = np.zeros((X.shape[0], 2, 3))
    A[:, 0, 0] = cam.fx * iz
    A[:, 0, 2] = -cam.fx * X[:, 0] * iz * iz
    A[:, 1, 1] = cam.fy * iz
    A[:, 1, 2] = -cam.fy * X[:, 1] * iz * iz
    return A


# ---------------------------------------------------------------------------
# Rasterisation with traversal records (ref: rasterizer.py:253-358)
# ---------------------------------------------------------------------------

def rasterize(s: OScene, cam: OCamera, cfg: OConfig = OConfig(), proj=None):
    """Front-to-back blending at pixel centres; returns a dict with the image
    and the pixel-sorted traversal (ref: rasterizer.py:319-358).

    Keys: image (H,W,3), offsets (HW+1), pixel, gid, alpha, T (T before the
    entry), t_final (HW), colors (G,3), proj.
    """
    pr = project(s, cam, cfg) if proj is None else proj
    W, H = cam.width, cam.height
    ids = np.nonzero(pr["valid"])[0]
    order = ids[np.lexsort((ids, pr["depth"][ids]))]          # depth asc, gid tie-break
    cov = pr["cov"]
    if cfg.alpha_min > 0:
        lam = 0.5 * (cov[:, 0] + cov[:, 2]) + np.sqrt(0.25 * (cov[:, 0] - cov[:, 2]) ** 2
                                                       + cov[:, 1] ** 2)
        reach = np.sqrt(max(0.0, 2.0 * np.log(1.0 / cfg.alpha_min))) * np.sqrt(lam)
    else:
        reach = np.full(s.G, np.inf)

    T = np.ones((H, W))
    rgb = np.zeros((H, W, 3))
    cols = np.arange(W) + 0.5
    rec_pix, rec_gid, rec_a, rec_t = [], [], [], []
    for g in order:
        mx, my = pr["mean"][g]
        r = reach[g]
        if np.isfinite(r):
            x0, x1 = max(0, int(np.ceil(mx - r - 0.5))), min(W - 1, int(np.floor(mx + r - 0.5)))
            y0, y1 = max(0, int(np.ceil(my - r - 0.5))), min(H - 1, int(np.floor(my + r - 0.5)))
        else:
            x0, x1, y0, y1 = 0, W - 1, 0, H - 1
        if x0 > x1 or y0 > y1:
            continue
        ca, cb, cc = pr["conic"][g]
        dx = cols[x0:x1 + 1] - mx
        dy = (np.arange(y0, y1 + 1) + 0.5) - my
        q = ca * dx * dx + cc * (dy * dy)[:, None] + 2.0 * cb * dy[:, None] * dx
        a = np.minimum(pr["opacity"][g] * np.exp(-0.5 * q), cfg.alpha_clamp)
        Tb = T[y0:y1 + 1, x0:x1 + 1]
        keep = (a >= cfg.alpha_min) & (a > 0.0) & (Tb >= cfg.t_stop)
        if not keep.any():
            continue
        iy, ix = np.nonzero(keep)
        ak, tk = a[iy, ix], Tb[iy, ix]
        rgb[y0 + iy, x0 + ix] += (ak * tk)[:, None] * pr["color"][g]
        Tb[iy, ix] = tk * (1.0 - ak)
        rec_pix.append((y0 + iy) * W + (x0 + ix))
        rec_gid.append(np.full(iy.size, g, dtype=np.int64))
        rec_a.append(ak)
        rec_t.append(tk)

    def cat(lst, dt):
        return np.concatenate(lst) if lst else np.zeros(0, dt)
    pix, gid = cat(rec_pix, np.int64), cat(rec_gid, np.int64)
    alpha, tb = cat(rec_a, np.float64), cat(rec_t, np.float64)
    t_final = T.reshape(-1)
    rgb = rgb + s.background[None, None, :] * T[:, :, None]
    srt = np.argsort(pix, kind="stable")      # keep front-to-back order inside a pixel
    pix = pix[srt]
    offsets = np.zeros(H * W + 1, dtype=np.int64)
    offsets[1:] = np.cumsum(np.bincount(pix, minlength=H * W))
    return dict(image=rgb, offsets=offsets, pixel=pix, gid=gid[srt], alpha=alpha[srt],
                T=tb[srt], t_final=t_final, colors=pr["color"], proj=pr)


# ---------------------------------------------------------------------------
# Residuals (ref: residuals.py:49-296).  The reference filters with
# scipy.ndimage.correlate1d(mode="reflect") (scipy>=1.10, installed 1.18.1);
# restated here as an explicit half-sample-symmetric 11-tap correlation.
# ---------------------------------------------------------------------------
SSIM_C1 = 1e-4
SSIM_C2 = 9e-4


def _taps(window=11, sigma=1.5):
    o = np.arange(window) - window // 2
    k = np.exp(-0.5 * (o / sigma) ** 2)
    return k / k.sum()


def _reflect(idx, n):
    """scipy 'reflect' boundary: d c b a | a b c d | d c b a, period 2n."""
    idx = np.mod(idx, 2 * n)
    return np.where(idx >= n, 2 * n - 1 - idx, idx)


def _corr_axis(img, k, axis):
    n = img.shape[axis]
    half = k.size // 2
    out = np.zeros_like(img)
    base = np.arange(n)
    for j, w in enumerate(k):
        out += w * np.take(img, _reflect(base + j - half, n), axis=axis)
    return out


def ssim_blur(img, window=11, sigma=1.5):
    """ref: residuals.py:58-62."""
    k = _taps(window, sigma)
    return _corr_axis(_corr_axis(img, k, 0), k, 1)


def center_weights(H, W, window=11, sigma=1.5):
    """Self weight of each pixel in its own window (ref: residuals.py:71-91)."""
    k = _taps(window, sigma)
    half = window // 2

    def one(n):
        # single reflection, exactly as ref: residuals.py:65-68 (differs from
        # scipy's periodic 'reflect' only for n < window/2)
        pos = np.arange(n)
        acc = np.zeros(n)
        for j, w in enumerate(k):
            i = pos + j - half
            i = np.where(i < 0, -i - 1, i)
            i = np.where(i >= n, 2 * n - i - 1, i)
            acc += w * (i == pos)
        return acc
    return np.outer(one(H), one(W))


def residuals(img, gt, lambda1=0.8, lambda2=0.2, mode="l1ssim", eps_den=1e-8):
    """Residual weights for one view (ref: residuals.py:249-296).

    Returns dict: grad_r_sq, color_grad, r_abs, r_ssim, drabs_dc, drssim_dc,
    energy (all (H,W,3) except energy).
    """
    img = np.asarray(img, np.float64)
    gt = np.asarray(gt, np.float64)
    if img.shape != gt.shape or img.ndim != 3 or img.shape[2] != 3:
        raise ValueError(f"image shapes differ or are not (H,W,3): {img.shape} {gt.shape}")
    e = img - gt
    if mode == "l2":
        one = np.ones_like(e)
        return dict(grad_r_sq=one, color_grad=e.copy(), r_abs=e, r_ssim=None,
                    drabs_dc=one, drssim_dc=None, energy=float(np.sum(e * e)))
    if mode != "l1ssim":
        raise ValueError(f"unknown loss mode {mode!r}")
    if lambda1 < 0 or lambda2 < 0:
        raise ValueError("loss weights must be >= 0")
    ae = np.abs(e)
    r_abs = np.sqrt(lambda1 * ae)
    if lambda1 > 0:
        ge = np.maximum(ae, eps_den)
        drabs = lambda1 * np.sign(e) / (2.0 * np.sqrt(lambda1 * ge))
        w1 = lambda1 / (4.0 * ge)
    else:
        drabs = np.zeros_like(e)
        w1 = np.zeros_like(e)
    if lambda2 > 0:
        mx, my = ssim_blur(img), ssim_blur(gt)
        exx, eyy, exy = ssim_blur(img * img), ssim_blur(gt * gt), ssim_blur(img * gt)
        sxx, syy, sxy = exx - mx * mx, eyy - my * my, exy - mx * my
        a1, a2 = 2 * mx * my + SSIM_C1, 2 * sxy + SSIM_C2
        b1, b2 = mx * mx + my * my + SSIM_C1, sxx + syy + SSIM_C2
        score = (a1 * a2) / (b1 * b2)
        cw = center_weights(img.shape[0], img.shape[1])[:, :, None]
        dsc = (2.0 * cw / (b1 * b2)) * (my * a2 + a1 * (gt - my)) \
            - score * 2.0 * cw * (mx / b1 + (img - mx) / b2)
        om = np.maximum(1.0 - score, 0.0)
        r_ssim = np.sqrt(lambda2 * om)
        go = np.maximum(om, eps_den)
        drssim = -lambda2 * dsc / (2.0 * np.sqrt(lambda2 * go))
        w2 = lambda2 * dsc * dsc / (4.0 * go)
    else:
        r_ssim = np.zeros_like(e)
        drssim = np.zeros_like(e)
        w2 = np.zeros_like(e)
    return dict(grad_r_sq=w1 + w2, color_grad=drabs * r_abs + drssim * r_ssim,
                r_abs=r_abs, r_ssim=r_ssim, drabs_dc=drabs, drssim_dc=drssim,
                energy=float(np.sum(r_abs ** 2) + np.sum(r_ssim ** 2)))


# ---------------------------------------------------------------------------
# Per-view splat -> parameter tables (ref: jacobian.py:141-266)
# ---------------------------------------------------------------------------

def _drot_dq(qh):
    """d R / d q_hat for unit quaternions, (G, 4, 3, 3)."""
    w, x, y, z = qh[:, 0], qh[:, 1], qh[:, 2], qh[:, 3]
    o = np.zeros_like(w)
    m = lambda rows: 2.0 * np.stack([np.stack(r, -1) for r in rows], -2)  # noqa: E731
    return np.stack([
        m([(o, -z, y), (z, o, -x), (-y, x, o)]),
        m([(o, y, z), (y, -2 * x, -w), (z, w, -2 * x)]),
        m([(-2 * y, x, w), (x, o, z), (-w, z, -2 * y)]),
        m([(-2 * z, -w, x), (w, -2 * z, y), (x, y, o)]),
    ], 1)


def _sym3(m):
    return np.stack([m[..., 0, 0], m[..., 0, 1], m[..., 1, 1]], -1)


def splat_tables(s: OScene, cam: OCamera, pr):
    """Derivatives of the projected splat attributes w.r.t. the 11 geometry
    parameters, plus SH basis and colour mask (ref: jacobian.py:192-266).

    Returns dict: dmu (G,2,11), dcov (G,3,11), dcol (G,3,11), dopa (G,11),
    basis (G,K), mask (G,3) float.
    """
    G = s.G
    Rg, qh, qn = _rotations(s.quat)
    s2 = np.exp(2.0 * s.log_scale)
    cov_w = (Rg * s2[:, None, :]) @ np.swapaxes(Rg, 1, 2)
    X = np.where(pr["valid"][:, None], pr["cam"], np.array([0.0, 0.0, 1.0]))
    A = _proj_jac(X, cam)
    U = A @ cam.R
    cov_c = cam.R @ cov_w @ cam.R.T

    dmu = np.zeros((G, 2, GEOM))
    dmu[:, :, 0:3] = U

    # covariance w.r.t. camera-space point: the Jacobian A varies with X
    fx, fy = cam.fx, cam.fy
    x, y, z = X[:, 0], X[:, 1], X[:, 2]
    iz2 = 1.0 / (z * z)
    Pm = cov_c @ np.swapaxes(A, 1, 2)              # (G,3,2)
    dA = np.zeros((G, 3, 2, 3))                    # dA/dX_i
    dA[:, 0, 0, 2] = -fx * iz2
    dA[:, 1, 1, 2] = -fy * iz2
    dA[:, 2, 0, 0] = -fx * iz2
    dA[:, 2, 0, 2] = 2.0 * fx * x * iz2 / z
    dA[:, 2, 1, 1] = -fy * iz2
    dA[:, 2, 1, 2] = 2.0 * fy * y * iz2 / z
    Q = dA @ Pm[:, None]                           # (G,3,2,2)
    dcov_X = _sym3(Q + np.swapaxes(Q, -1, -2))     # (G,3X,3pack)
    dcov = np.zeros((G, 3, GEOM))
    dcov[:, :, 0:3] = np.einsum("gip,ij->gpj", dcov_X, cam.R)

    # quaternion path: dCov_w = dR S R^T + R S dR^T, chained through normalisation
    dRh = _drot_dq(qh)
    chain = (np.eye(4)[None] - qh[:, :, None] * qh[:, None, :]) / qn[:, None, None]
    dR = np.einsum("gkab,gkl->glab", dRh, chain)   # (G,4,3,3)
    half = dR @ (Rg * s2[:, None, :]).transpose(0, 2, 1)[:, None]
    dcw = half + np.swapaxes(half, -1, -2)
    dcq = U[:, None] @ dcw @ np.swapaxes(U, 1, 2)[:, None]
    dcov[:, :, 3:7] = np.swapaxes(_sym3(dcq), 1, 2)

    # log-scale path: d cov_w / d l_i = 2 s_i^2 r_i r_i^T
    UR = U @ Rg                                    # (G,2,3) columns U r_i
    outer = UR[:, :, None, :] * UR[:, None, :, :]  # (G,2,2,3)
    dcov[:, :, 7:10] = 2.0 * s2[:, None, :] * _sym3(np.moveaxis(outer, 3, 1)).transpose(0, 2, 1)

    # colour: SH basis w.r.t. coefficients; position moves the view direction
    v = s.pos - cam.center
    vn = np.linalg.norm(v, axis=1)
    d = v / vn[:, None]
    basis = sh_basis(d, s.degree)
    dbasis = sh_basis_grad(d, s.degree)
    mask = (~pr["clamped"]).astype(np.float64)
    dcol_dd = np.einsum("gck,gkj->gcj", s.sh, dbasis)
    dd_dp = (np.eye(3)[None] - d[:, :, None] * d[:, None, :]) / vn[:, None, None]
    dcol = np.zeros((G, 3, GEOM))
    dcol[:, :, 0:3] = mask[:, :, None] * (dcol_dd @ dd_dp)

    dopa = np.zeros((G, GEOM))
    o = pr["opacity"]
    dopa[:, 10] = o * (1.0 - o)

    bad = ~pr["valid"]
    for t in (dmu, dcov, dcol, dopa):
        t[bad] = 0.0
    return dict(dmu=dmu, dcov=dcov, dcol=dcol, dopa=dopa, basis=basis, mask=mask)


# ---------------------------------------------------------------------------
# Gradient cache (ref: jacobian.py:46-121, 360-416)
# ---------------------------------------------------------------------------

@dataclass
class OView:
    """One view's gradient cache plus what products need (ref: jacobian.py:46-84)."""
    cam: OCamera
    cfg: OConfig
    G: int
    pixel: np.ndarray
    gid: np.ndarray
    alpha: np.ndarray
    T: np.ndarray
    dcda: np.ndarray     # (E,3)
    dcdc: np.ndarray     # (E,)  alpha*T
    src: np.ndarray      # source_index
    offsets: np.ndarray
    order: str           # "pixel" | "gaussian"
    grad_r_sq: np.ndarray  # (HW*3,)

    @property
    def E(self):
        return self.pixel.size


def build_cache(s: OScene, cam: OCamera, res, cfg: OConfig = OConfig(), rast=None):
    """b = -J^T F and the pixel-sorted cache for one view (ref: jacobian.py:360-416)."""
    H, W = cam.height, cam.width
    if res["grad_r_sq"].shape[:2] != (H, W):
        raise ValueError("residual bundle does not match the camera resolution")
    rs = rasterize(s, cam, cfg) if rast is None else rast
    pix, gid, a, T = rs["pixel"], rs["gid"], rs["alpha"], rs["T"]
    off = rs["offsets"]
    col = rs["colors"][gid]
    w = a * T
    c = col * w[:, None]
    # colour strictly behind each entry within its pixel + background leak
    npx = np.diff(off)
    inc = np.cumsum(c, axis=0)
    seg_total = np.zeros((H * W, 3))
    nz = npx > 0
    seg_total[nz] = np.add.reduceat(c, off[:-1][nz], axis=0)
    start_base = np.zeros((E := pix.size, 3))
    if E:
        before = np.where(off[:-1] > 0, off[:-1] - 1, 0)
        base_px = np.where((off[:-1] > 0)[:, None], inc[before], 0.0)
        start_base = base_px[pix]
    prefix_incl = inc - start_base
    behind = seg_total[pix] - prefix_incl + s.background[None, :] * rs["t_final"][pix][:, None]
    dcda = col * T[:, None] - behind / (1.0 - a)[:, None]
    view = OView(cam=cam, cfg=cfg, G=s.G, pixel=pix.copy(), gid=gid.copy(), alpha=a.copy(),
                 T=T.copy(), dcda=dcda, dcdc=w, src=np.arange(E, dtype=np.int64),
                 offsets=off.copy(), order="pixel",
                 grad_r_sq=res["grad_r_sq"].reshape(-1).copy())
    b = -_jt_partials_to_params(view, s, rs["proj"], res["color_grad"].reshape(-1))
    return b, view


def gaussian_order(v: OView) -> OView:
    """Stable re-sort by (gaussian, pixel) (ref: jacobian.py:93-105)."""
    if v.order != "pixel":
        raise ValueError("expected pixel-sorted cache")
    perm = np.lexsort((v.pixel, v.gid))
    off = np.zeros(v.G + 1, dtype=np.int64)
    off[1:] = np.cumsum(np.bincount(v.gid, minlength=v.G))
    return OView(cam=v.cam, cfg=v.cfg, G=v.G, pixel=v.pixel[perm], gid=v.gid[perm],
                 alpha=v.alpha[perm], T=v.T[perm], dcda=v.dcda[perm], dcdc=v.dcdc[perm],
                 src=v.src[perm], offsets=off, order="gaussian", grad_r_sq=v.grad_r_sq)


def _entry_state(v: OView, pr):
    """e = conic (px - mean), alpha / exp-term with zero gradient through an
    active clamp (ref: jacobian.py:273-297)."""
    W = v.cam.width
    dx = (v.pixel % W) + 0.5 - pr["mean"][v.gid, 0]
    dy = (v.pixel // W) + 0.5 - pr["mean"][v.gid, 1]
    k = pr["conic"][v.gid]
    e1 = k[:, 0] * dx + k[:, 1] * dy
    e2 = k[:, 1] * dx + k[:, 2] * dy
    gv = np.exp(-0.5 * (dx * e1 + dy * e2))
    live = v.alpha < v.cfg.alpha_clamp
    return e1, e2, np.where(live, v.alpha, 0.0), np.where(live, gv, 0.0)


def _seg_sum(vals, gid, G, order, offsets):
    out = np.zeros((G,) + vals.shape[1:])
    if vals.shape[0] == 0:
        return out
    if order == "gaussian":
        st = offsets[:-1]
        nz = offsets[1:] > st
        out[nz] = np.add.reduceat(vals, st[nz], axis=0)
    else:
        np.add.at(out, gid, vals)
    return out


def _jt_partials_to_params(v: OView, s: OScene, pr, u):
    """J^T u for one view, attribute-major (ref: jacobian.py:324-353)."""
    e1, e2, ae, ge = _entry_state(v, pr)
    ue = u.reshape(-1, 3)[v.pixel]
    sa = np.sum(v.dcda * ue, axis=1)
    sc = v.dcdc[:, None] * ue
    t = sa * ae
    per = np.column_stack([t * e1, t * e2, 0.5 * t * e1 * e1, t * e1 * e2, 0.5 * t * e2 * e2,
                           sa * ge, sc])
    acc = _seg_sum(per, v.gid, s.G, v.order, v.offsets)
    tb = splat_tables(s, v.cam, pr)
    gg = (np.einsum("gi,gij->gj", acc[:, 0:2], tb["dmu"])
          + np.einsum("gi,gij->gj", acc[:, 2:5], tb["dcov"])
          + np.einsum("gc,gcj->gj", acc[:, 6:9], tb["dcol"])
          + acc[:, 5:6] * tb["dopa"])
    gsh = (acc[:, 6:9] * tb["mask"])[:, :, None] * tb["basis"][:, None, :]
    return am_from_matrix(np.concatenate([gg, gsh.reshape(s.G, -1)], 1))


def apply_j(p_am, s: OScene, v: OView):
    """u_hat = J p for one view; p attribute-major (ref: jacobian.py:419-455;
    the reference takes gaussian-major p -- layout handled by the caller)."""
    pr = project(s, v.cam, v.cfg)
    tb = splat_tables(s, v.cam, pr)
    e1, e2, ae, ge = _entry_state(v, pr)
    pm = matrix_from_am(p_am, s.G)
    pg, psh = pm[:, :GEOM], pm[:, GEOM:].reshape(s.G, 3, -1)
    m_mu = np.einsum("gij,gj->gi", tb["dmu"], pg)
    m_cov = np.einsum("gij,gj->gi", tb["dcov"], pg)
    m_col = np.einsum("gij,gj->gi", tb["dcol"], pg) + tb["mask"] * np.einsum("gk,gck->gc", tb["basis"], psh)
    m_o = np.einsum("gj,gj->g", tb["dopa"], pg)
    g = v.gid
    da = ae * (e1 * m_mu[g, 0] + e2 * m_mu[g, 1] + 0.5 * e1 * e1 * m_cov[g, 0]
               + e1 * e2 * m_cov[g, 1] + 0.5 * e2 * e2 * m_cov[g, 2]) + ge * m_o[g]
    contrib = v.dcda * da[:, None] + v.dcdc[:, None] * m_col[g]
    out = np.zeros((v.cam.width * v.cam.height, 3))
    np.add.at(out, v.pixel, contrib)
    return out.reshape(-1)


def weight(u_hat, v: OView):
    """ref: jacobian.py:458-464."""
    return u_hat * v.grad_r_sq


def apply_jt(u, s: OScene, v: OView):
    """ref: jacobian.py:467-483 (requires gaussian order)."""
    if v.order != "gaussian":
        raise ValueError("expected gaussian-sorted cache")
    return _jt_partials_to_params(v, s, project(s, v.cam, v.cfg), u)


def diag_jtj(s: OScene, v: OView):
    """diag(J^T W J), attribute-major (ref: jacobian.py:486-512)."""
    if v.order != "gaussian":
        raise ValueError("expected gaussian-sorted cache")
    pr = project(s, v.cam, v.cfg)
    tb = splat_tables(s, v.cam, pr)
    e1, e2, ae, ge = _entry_state(v, pr)
    g = v.gid
    wr = v.grad_r_sq.reshape(-1, 3)[v.pixel]
    coef = np.column_stack([ae * e1, ae * e2, 0.5 * ae * e1 * e1, ae * e1 * e2,
                            0.5 * ae * e2 * e2])                          # (E,5)
    D = np.concatenate([tb["dmu"], tb["dcov"]], axis=1)                   # (G,5,11)
    dadx = np.einsum("ek,ekj->ej", coef, D[g]) + ge[:, None] * tb["dopa"][g]
    acc = np.zeros((s.G, GEOM))
    for ch in range(3):
        dc = v.dcda[:, ch:ch + 1] * dadx + v.dcdc[:, None] * tb["dcol"][g, ch]
        acc += _seg_sum(wr[:, ch:ch + 1] * dc * dc, g, s.G, v.order, v.offsets)
    ssh = _seg_sum(wr * (v.dcdc ** 2)[:, None] * tb["mask"][g], g, s.G, v.order, v.offsets)
    msh = ssh[:, :, None] * (tb["basis"] ** 2)[:, None, :]
    return am_from_matrix(np.concatenate([acc, msh.reshape(s.G, -1)], 1))


# ---------------------------------------------------------------------------
# Solver (SPEC-only in the reference: SPEC:391-408, 473-479)
# ---------------------------------------------------------------------------

def jtwj(p_am, s: OScene, views):
    """Sum over a batch's views of J^T W J p."""
    out = np.zeros_like(p_am)
    for v in views:
        out += apply_jt(weight(apply_j(p_am, s, v), v), s, v)
    return out


def pcg(s: OScene, views, b, M, lam, n_iters, stats=None):
    """Alg. 1 with SPEC:394-395 exit/abort rules.

    A = J^T W J + lam * diag(Mf), Mf = max(M, 1e-12).
    Makes n_iters + 1 products at most.  Raises NonSPDError if p^T g <= 0.
    """
    Mf = np.maximum(M, M_FLOOR)
    bb = float(b @ b)
    x = b / Mf
    if bb == 0.0:
        return x
    r = b - (jtwj(x, s, views) + lam * Mf * x)
    z = r / Mf
    p = z.copy()
    rz = float(r @ z)
    n_prod = 1
    for _ in range(n_iters):
        g = jtwj(p, s, views) + lam * Mf * p
        n_prod += 1
        pg = float(p @ g)
        if not pg > 0.0:
            raise NonSPDError(f"p^T g = {pg} <= 0")
        a = rz / pg
        x = x + a * p
        r = r - a * g
        z = r / Mf
        rz_new = float(r @ z)
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
        if float(r @ r) < 0.01 * bb:
            break
    if stats is not None:
        stats["products"] = n_prod
    return x


def combine(deltas, Ms):
    """Eq. 7 weighted mean."""
    num = np.zeros_like(deltas[0])
    den = np.zeros_like(deltas[0])
    for d, m in zip(deltas, Ms):
        num += m * d
        den += m
    return num / np.maximum(den, M_FLOOR)


def strided_batches(n_views, n_batches):
    """Batch j takes views {j, j+n_b, ...}."""
    return [list(range(j, n_views, n_batches)) for j in range(n_batches)]


def lm_direction(s: OScene, cams, gts, n_batches=1, lam=1e-4, n_iters=8,
                 lambda1=0.8, lambda2=0.2, mode="l1ssim", cfg: OConfig = OConfig(),
                 trace=None):
    """One LM update direction: per batch cache build, b, M, PCG, then the
    Eq. 7 combine.  `trace` (dict) receives per-batch
    intermediates for parity tests."""
    deltas, Ms = [], []
    for j, idx in enumerate(strided_batches(len(cams), n_batches)):
        b = np.zeros(s.G * s.P)
        M = np.zeros(s.G * s.P)
        views = []
        for i in idx:
            rs = rasterize(s, cams[i], cfg)
            res = residuals(rs["image"], gts[i], lambda1, lambda2, mode)
            bv, v = build_cache(s, cams[i], res, cfg, rast=rs)
            v = gaussian_order(v)
            b += bv
            M += diag_jtj(s, v)
            views.append(v)
        try:
            d = pcg(s, views, b, M, lam, n_iters)
        except NonSPDError:
            continue
        deltas.append(d)
        Ms.append(M)
        if trace is not None:
            trace.setdefault("b", []).append(b)
            trace.setdefault("M", []).append(M)
            trace.setdefault("delta", []).append(d)
    if not deltas:
        raise NonSPDError("all batches rejected by PCG failure")
    return combine(deltas, Ms)


# ---------------------------------------------------------------------------
# LM outer-loop helpers -- the "next" rows of SURVEY 8(f)
# ---------------------------------------------------------------------------

def energy(s: OScene, cams, gts, lambda1=0.8, lambda2=0.2, mode="l1ssim", cfg=OConfig()):
    return sum(residuals(rasterize(s, c, cfg)["image"], g, lambda1, lambda2, mode)["energy"]
               for c, g in zip(cams, gts))


def line_search(s: OScene, delta_am, cams, gts, depth=8, **kw):
    """Dyadic grid {1, 1/2, ..., 2^-depth} u {0}; ties go to the smaller
    gamma."""
    base = scene_matrix(s)
    grid = [2.0 ** -i for i in range(depth + 1)]
    best_g, best_e = 0.0, energy(s, cams, gts, **kw)
    for gma in sorted(grid):
        sm = scene_from_matrix(base + gma * matrix_from_am(delta_am, s.G), s.degree, s.background)
        e = energy(sm, cams, gts, **kw)
        if e < best_e:
            best_g, best_e = gma, e
    return best_g, best_e


def compute_rho(e_old, e_new, model_reduction):
    """Eq. 6 ratio; denominator |.| < 1e-12 -> -inf sentinel."""
    if abs(model_reduction) < 1e-12:
        return -np.inf
    return (e_old - e_new) / model_reduction


def trust_region_update(lam, rho, lam_min=1e-4, lam_max=1e4):
    """SPEC:418-426."""
    if rho > 1e-5:
        lam = lam * (1.0 - (2.0 * rho - 1.0) ** 3)
        return True, float(min(max(lam, lam_min), lam_max))
    return False, float(min(max(2.0 * lam, lam_min), lam_max))
