"""Size-independent properties of the products at the full C3 subset size
(1M Gaussians, 25 views @ 1024^2, ~1e9 cache entries) -- where the fp64
oracle cannot run, the operators are checked against each other:

  * adjointness   u.(J p) == (J^T u).p             (apply_j vs apply_jt)
  * symmetry      q.(A p) == p.(A q),  A = J^T W J (fused product)
  * linearity     A(p + 2q) == A p + 2 A q
  * PSD / weights p.(A p) == sum_i w_i (J p)_i^2    (fused vs apply_j + grad_r_sq)
  * diagonal      (A e_k)_k == diag(A)_k            (fused product vs diag kernel)
  * rhs           b == -J^T color_grad             (rhs vs apply_jt with cgrad)

fp32 products accumulate over ~1e9 entries; tolerances are stated per check.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c3():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import bench
    from paper_2409_12892_b200.engine import CacheSet
    from paper_2409_12892_b200.solver import BatchSchedule
    cfg = dict(bench.CONFIGS["c3"])
    dev = torch.device("cuda", 0)
    views = BatchSchedule(cfg["subsets"]).batches(cfg["views"])[0]
    init, cams, gts = bench.make_workload(cfg, dev, only=set(views))
    scene = init.to_device(dev)
    cs = CacheSet(scene, [cams[i] for i in views], [gts[i] for i in views])
    assert cs.E > 5e8  # the full-size regime, not a toy
    yield scene, cs
    del cs
    torch.cuda.empty_cache()


def _d(a, b):
    return float(torch.dot(a.double().flatten(), b.double().flatten()))


def _rand(n, seed):
    g = torch.Generator("cuda").manual_seed(seed)
    return torch.randn(n, device="cuda", generator=g)


def _A(cs, p):
    out = torch.empty_like(p)
    cs.jtwj(p, out)
    return out


def _Jp(cs, p):
    cs.pair_forward(p)
    cs.apply_j_raw(weighted=False)
    return cs.u.clone()


def test_adjoint(c3):
    scene, cs = c3
    p = _rand(scene.param_count, 1)
    u = _rand(cs.N * 4, 2)
    u.view(-1, 4)[:, 3] = 0.0
    jp = _Jp(cs, p)
    jtu = torch.empty_like(p)
    cs.apply_jt_raw(u, jtu)
    lhs, rhs = _d(u, jp), _d(jtu, p)
    scale = float(u.double().norm() * jp.double().norm())
    assert abs(lhs - rhs) <= 1e-5 * scale, (lhs, rhs, scale)


def test_symmetry_linearity_psd(c3):
    scene, cs = c3
    p, q = _rand(scene.param_count, 3), _rand(scene.param_count, 4)
    Ap, Aq = _A(cs, p), _A(cs, q)
    pAp, qAq = _d(p, Ap), _d(q, Aq)
    assert pAp > 0 and qAq > 0
    # symmetry, relative to the Cauchy-Schwarz bound sqrt(pAp qAq)
    assert abs(_d(q, Ap) - _d(p, Aq)) <= 1e-4 * np.sqrt(pAp * qAq)
    # linearity (fp32 products, relative L2)
    A2 = _A(cs, p + 2.0 * q)
    ref = Ap.double() + 2.0 * Aq.double()
    assert float((A2.double() - ref).norm() / ref.norm()) < 1e-4
    # p.(J^T W J p) == sum_i w_i (J p)_i^2 with W = grad_r_sq (float4 per pixel, .w unused)
    jp = _Jp(cs, p).view(-1, 4)[:, :3].double()
    w = cs.gradr.view(-1, 4)[:, :3].double()
    wsum = float((w * jp * jp).sum())
    assert abs(pAp - wsum) <= 1e-4 * wsum, (pAp, wsum)


def test_diag_equals_unit_products(c3):
    scene, cs = c3
    M = cs.diag()
    G, P = scene.num_gaussians, scene.params_per_gaussian
    med = float(M[M > 0].median())
    rng = np.random.default_rng(5)
    # one parameter of each kind: position, quaternion, log-scale, opacity, SH dc, SH higher
    checked = 0
    for attr in (0, 4, 8, 10, 11, 20):
        for g in rng.permutation(G)[:64]:
            k = attr * G + int(g)
            if float(M[k]) > 1e-3 * med:
                e = torch.zeros(scene.param_count, device="cuda")
                e[k] = 1.0
                col = _A(cs, e)
                assert abs(float(col[k]) - float(M[k])) <= 1e-4 * float(M[k]), (attr, k)
                checked += 1
                break
    assert checked >= 5


def test_rhs_is_minus_jt_color_grad(c3):
    scene, cs = c3
    b = cs.rhs()
    g = torch.empty_like(b)
    cs.apply_jt_raw(cs.cgrad, g)
    assert float((b.double() + g.double()).norm()) <= 1e-6 * float(b.double().norm())
