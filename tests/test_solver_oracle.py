"""CPU: the PCG / Eq. 7 / LM-helper restatements against the SPEC's
known-answer examples and a dense solve."""
import numpy as np
import pytest

import oracle as O
from helpers import ocam, oscene, problem, rel


@pytest.fixture(scope="module")
def tiny():
    truth, init, cams, gts = problem(seed=11, G=12, n_views=2, W=14, H=12, degree=0)
    s = oscene(init)
    views, b, M = [], 0.0, 0.0
    for c, gt in zip(cams, gts):
        oc = ocam(c)
        rs = O.rasterize(s, oc)
        res = O.residuals(rs["image"], gt)
        bv, v = O.build_cache(s, oc, res, rast=rs)
        v = O.gaussian_order(v)
        views.append(v)
        b = b + bv
        M = M + O.diag_jtj(s, v)
    return s, views, b, M


def dense_A(s, views):
    n = s.G * s.P
    return np.stack([O.jtwj(np.eye(n)[i], s, views) for i in range(n)], 1)


def test_jtwj_symmetric_psd_and_diag(tiny):
    s, views, b, M = tiny
    A = dense_A(s, views)
    assert rel(A, A.T) < 1e-12
    assert rel(np.diag(A), M) < 1e-10          # diag_jtj == one-hot J^T W J
    assert np.linalg.eigvalsh(0.5 * (A + A.T)).min() > -1e-8 * np.abs(A).max()


def test_pcg_matches_dense_solve_well_conditioned(tiny):
    s, views, b, M = tiny
    n = b.size
    lam = 1.0
    A = dense_A(s, views) + lam * np.diag(np.maximum(M, 1e-12))
    x_dense = np.linalg.solve(A, b)
    st = {}
    x = O.pcg(s, views, b, M, lam, n_iters=n, stats=st)
    r = b - A @ x
    # either converged to the dense solve or stopped by the 0.01 ||b||^2 exit rule
    assert rel(x, x_dense) < 1e-5 or float(r @ r) < 0.01 * float(b @ b)
    assert st["products"] <= n + 1


def test_pcg_b_zero_gives_zero(tiny):
    s, views, b, M = tiny
    x = O.pcg(s, views, np.zeros_like(b), M, 1e-4, 8)
    assert np.all(x == 0.0)


def test_pcg_huge_damping(tiny):
    s, views, b, M = tiny
    lam = 1e6
    x = O.pcg(s, views, b, M, lam, 8)
    Mf = np.maximum(M, 1e-12)
    obs = M > 1e-6 * M.max()
    assert rel(x[obs], (b / (lam * Mf))[obs]) < 1e-2


def test_pcg_product_count(tiny):
    s, views, b, M = tiny
    st = {}
    O.pcg(s, views, b, M, 1e-4, 8, stats=st)
    assert st["products"] <= 9                    # n_iters + 1


def test_combine_identities():
    rng = np.random.default_rng(0)
    d1, d2 = rng.standard_normal(50), rng.standard_normal(50)
    M1 = rng.random(50)
    assert np.array_equal(O.combine([d1], [M1]), d1 * M1 / np.maximum(M1, 1e-12))     # n_b = 1
    assert rel(O.combine([d1], [M1]), d1) < 1e-14
    assert rel(O.combine([d1, d2], [M1, M1]), 0.5 * (d1 + d2)) < 1e-14              # equal weights
    z = np.zeros(50)
    assert np.all(O.combine([d1], [z]) == 0.0)                                        # 1e-12 floor


def test_combine_exact_for_diagonal_jtj():
    """with diagonal J^T J per batch, the Eq. 7 combine of the
    per-batch solutions equals the full-batch solution."""
    rng = np.random.default_rng(1)
    M1, M2 = rng.random(20) + 0.1, rng.random(20) + 0.1
    g1, g2 = rng.standard_normal(20), rng.standard_normal(20)
    full = (g1 + g2) / (M1 + M2)
    assert rel(O.combine([g1 / M1, g2 / M2], [M1, M2]), full) < 1e-12


def test_trust_region_cases():
    assert O.trust_region_update(1e-3, 0.5) == (True, 1e-3)
    acc, lam = O.trust_region_update(1e-3, 1e-6)
    assert not acc and lam == 2e-3
    acc, lam = O.trust_region_update(1e-2, 1.0)
    assert acc and lam == 1e-4                                                         # clamps to lambda_min
    rng = np.random.default_rng(2)
    lam = 1e-4
    for rho in rng.uniform(-2, 2, 1000):
        _, lam = O.trust_region_update(lam, rho)
        assert 1e-4 <= lam <= 1e4


def test_compute_rho_guard():
    assert O.compute_rho(1.0, 0.5, 0.0) == -np.inf
    assert O.compute_rho(2.0, 1.0, 1.0) == 1.0


def test_strided_batches():
    assert O.strided_batches(10, 3) == [[0, 3, 6, 9], [1, 4, 7], [2, 5, 8]]
