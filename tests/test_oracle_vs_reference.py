"""Oracle vs the live reference (only where /root/reference is mounted)."""
import numpy as np
import pytest

import oracle as O
from helpers import ocam, oscene, rel
from paper_2409_12892_b200 import synthetic as S

pytestmark = pytest.mark.reference


def test_generator_bit_compatible(ref_modules):
    RS = ref_modules[0]
    truth, cams, _ = RS.make_synthetic_dataset(4, 50, 3, (16, 12), sh_degree=2)
    h = S.make_synthetic_scene(4, 50, 2)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "sh_coeffs"):
        assert np.array_equal(getattr(h, f), getattr(truth, f)), f
    pi, hi = RS.perturb(truth, 9, 0.3), S.perturb(h, 9, 0.3)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "sh_coeffs"):
        assert np.array_equal(getattr(hi, f), getattr(pi, f)), f
    for a, b in zip(S.make_camera_ring(3, 16, 12), cams):
        assert np.array_equal(a.rotation, b.rotation) and np.array_equal(a.translation, b.translation)


@pytest.mark.parametrize("seed,degree,res", [(0, 3, (32, 28)), (2, 0, (17, 23)), (5, 1, (40, 8))])
def test_oracle_equals_reference(ref_modules, seed, degree, res):
    RS, RR, RE, RJ = ref_modules
    truth, cams, imgs = RS.make_synthetic_dataset(seed, 30, 2, res, sh_degree=degree)
    init = RS.perturb(truth, seed + 1, 0.1)
    s = oscene(init)
    rng = np.random.default_rng(seed)
    for c, gt in zip(cams, imgs):
        oc = ocam(c)
        rr = RR.render(init, c)
        ro = O.rasterize(s, oc)
        assert np.array_equal(ro["offsets"], rr.traversals.offsets)
        assert np.array_equal(ro["gid"], rr.traversals.gaussian_ids)
        assert rel(ro["image"], rr.image.rgb) < 1e-13
        bund = RE.compute_residuals(rr.image.rgb, gt)
        res = O.residuals(ro["image"], gt)
        assert rel(res["grad_r_sq"], bund.grad_r_sq) < 1e-10
        b_ref, cache = RJ.build_cache(init, c, bund, render_result=rr)
        b_o, v = O.build_cache(s, oc, res, rast=ro)
        assert rel(b_o, b_ref.values) < 1e-10
        gc = RJ.sort_cache_by_gaussians(cache)
        gv = O.gaussian_order(v)
        assert np.array_equal(gv.src, gc.source_index)
        p = rng.standard_normal(init.param_count)
        pv = RS.ParamVector(p, RS.Layout.ATTRIBUTE_MAJOR, init.num_gaussians, init.params_per_gaussian)
        assert rel(O.apply_j(p, s, gv), RJ.apply_j(RS.sort_x(pv), init, gc)) < 1e-10
        u = rng.standard_normal(c.num_pixels * 3)
        assert rel(O.apply_jt(u, s, gv), RJ.apply_jt(u, init, gc).values) < 1e-10
        assert rel(O.diag_jtj(s, gv), RJ.diag_jtj(init, gc).values) < 1e-10


def test_ssim_blur_equals_scipy():
    from scipy.ndimage import correlate1d
    rng = np.random.default_rng(0)
    for shape in ((20, 30, 3), (4, 7, 3), (1, 13, 3)):
        img = rng.random(shape)
        k = O.lm_oracle._taps()
        ref = correlate1d(correlate1d(img, k, axis=0, mode="reflect"), k, axis=1, mode="reflect")
        assert rel(O.ssim_blur(img), ref) < 1e-14


def test_lm_direction_oracle_equals_reference_driver():
    """The oracle's PCG + Eq. 7 restatement against the same loop driven by the
    reference's own products (oracle/ref_driver.py, the bench reference arm)."""
    from oracle import ref_driver as RD
    R = RD.import_reference()
    if R is None:
        pytest.skip("reference package not available")
    truth = S.make_synthetic_scene(2, 40, 2)
    init = S.perturb(truth, 3, 0.1)
    cams = S.make_camera_ring(4, 24, 20)
    gts = [O.rasterize(oscene(truth), ocam(c))["image"] for c in cams]
    ref, entries, ph = RD.lm_direction(R, RD.ref_scene(R, init), [RD.ref_camera(R, c) for c in cams], gts,
                                       n_batches=2, lam=1e-2, n_iters=5)
    got = O.lm_direction(oscene(init), [ocam(c) for c in cams], gts, n_batches=2, lam=1e-2, n_iters=5)
    assert entries > 0 and "pcg_products" in ph
    assert rel(got, ref) < 1e-9
