"""LM outer-loop rows: trust region / rho on CPU (SPEC
examples), and the device energy / line search / model reduction against the
fp64 oracle on a GPU."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import ocam, oscene, problem, rel
from paper_2409_12892_b200 import lm as L


def test_trust_region_spec_examples():
    # SPEC:418-426 examples
    assert L.trust_region_update(1.0, 0.5) == (True, 1.0)
    assert L.trust_region_update(1.0, 1e-6) == (False, 2.0)
    assert L.trust_region_update(1.0, 1.0) == (True, L.LAMBDA_MIN)
    assert L.trust_region_update(1e4, 1e-9) == (False, L.LAMBDA_MAX)
    for lam, rho in ((3e-3, 0.9), (0.5, 0.01), (2.0, -1.0)):
        assert L.trust_region_update(lam, rho) == O.trust_region_update(lam, rho)


def test_rho_guard():
    # |denominator| < 1e-12 -> rejection sentinel
    assert L.compute_rho(2.0, 1.0, 0.0) == -np.inf
    assert not L.trust_region_update(1.0, L.compute_rho(2.0, 1.0, 1e-13))[0]
    assert L.compute_rho(2.0, 1.0, 0.5) == 2.0 == O.compute_rho(2.0, 1.0, 0.5)


@pytest.fixture(scope="module")
def lmprob():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    truth, init, cams, gts = problem(seed=2, G=100, n_views=6, W=48, H=48, degree=3)
    osc = oscene(init)
    ocs = [ocam(c) for c in cams]
    delta = O.lm_direction(osc, ocs, gts, n_batches=2, lam=1e-2, n_iters=8).astype(np.float32)
    return dict(init=init, cams=cams, gts=gts, osc=osc, ocams=ocs, delta=delta, scene=init.to_device(),
                gts_d=[torch.from_numpy(g).cuda() for g in gts])


@pytest.mark.gpu
def test_energy_matches_oracle(lmprob):
    e = L.energy(lmprob["scene"], lmprob["cams"], lmprob["gts_d"])
    ref = O.energy(lmprob["osc"], lmprob["ocams"], lmprob["gts"])
    assert abs(e - ref) <= 1e-11 * abs(ref)


@pytest.mark.gpu
def test_line_search_matches_oracle(lmprob):
    d = torch.from_numpy(lmprob["delta"]).cuda()
    g, e = L.line_search(lmprob["scene"], d, lmprob["cams"][::3], lmprob["gts_d"][::3])
    g_ref, e_ref = O.line_search(lmprob["osc"], lmprob["delta"].astype(np.float64), lmprob["ocams"][::3],
                                 lmprob["gts"][::3])
    assert g == g_ref
    assert abs(e - e_ref) <= 1e-10 * abs(e_ref)
    # delta = 0 -> gamma = 0 (ties go to 0)
    assert L.line_search(lmprob["scene"], torch.zeros_like(d), lmprob["cams"][:1], lmprob["gts_d"][:1])[0] == 0.0


@pytest.mark.gpu
def test_model_reduction_matches_oracle(lmprob):
    from paper_2409_12892_b200.engine import CacheSet
    views = [0, 2, 4]
    cs = CacheSet(lmprob["scene"], [lmprob["cams"][i] for i in views], [lmprob["gts_d"][i] for i in views])
    d64 = lmprob["delta"].astype(np.float64)
    gv, b = [], 0
    for i in views:
        rs = O.rasterize(lmprob["osc"], lmprob["ocams"][i])
        bb, v = O.build_cache(lmprob["osc"], lmprob["ocams"][i], O.residuals(rs["image"], lmprob["gts"][i]), rast=rs)
        gv.append(O.gaussian_order(v))
        b = b + bb
    for gamma in (1.0, 0.25):
        ref = 2 * gamma * (b @ d64) - gamma ** 2 * (d64 @ O.jtwj(d64, lmprob["osc"], gv))
        got = L.model_reduction(cs, torch.from_numpy(lmprob["delta"]).cuda(), gamma)
        assert abs(got - ref) <= 1e-5 * abs(ref)


@pytest.mark.gpu
def test_lm_step_accepts_descent(lmprob):
    """A problem whose oracle line search descends: the step must be accepted,
    lower the energy and shrink lambda; the fixture-pinned
    version against the reference is tests/test_c1_end_to_end.py."""
    from paper_2409_12892_b200.solver import BatchSchedule
    rep = L.lm_step(lmprob["scene"], lmprob["cams"], lmprob["gts_d"], BatchSchedule(2), lam=1e-2, n_iters=8)
    e0 = L.energy(lmprob["scene"], lmprob["cams"], lmprob["gts_d"])
    g_ref, _ = O.line_search(lmprob["osc"], lmprob["delta"].astype(np.float64), lmprob["ocams"][::3],
                             lmprob["gts"][::3])
    assert g_ref > 0                                  # the problem is a descent case
    assert rep.accepted and rep.gamma == g_ref and rep.rho > 1e-5
    assert rep.lam <= 1e-2
    assert L.energy(rep.scene, lmprob["cams"], lmprob["gts_d"]) < e0
