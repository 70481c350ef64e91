"""SPEC known-answer examples and edge cases on the CUDA path.

SPEC:60-62 (sort_x), SPEC:149-151 and 157 (render)
(residuals), SPEC:313 (diag of a culled Gaussian), SPEC:397 (b = 0), plus an
all-culled scene (E = 0) and an empty scene (G = 0) through CacheSet, b, M,
PCG and the LM direction, and RenderConfig.smooth() (alpha_min = 0,
t_stop = 0, no cull; ref rasterizer.py:42-45, 292-296) traversals against the
oracle.
"""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import ocam, oscene, problem, rel
from paper_2409_12892_b200 import rasterizer as R
from paper_2409_12892_b200 import residuals as RES
from paper_2409_12892_b200.engine import CacheSet
from paper_2409_12892_b200.errors import ImageSizeError
from paper_2409_12892_b200.scene import Camera, GaussianScene, Layout, ParamVector, sort_x, sort_x_inverse
from paper_2409_12892_b200.solver import BatchSchedule, lm_direction, pcg_run

pytestmark = pytest.mark.gpu
SH_C0 = 0.28209479177387814


@pytest.fixture(autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


def _cam(W=8, H=8):
    # identity pose: camera at the origin looking down +z; pixel (3, 3)'s
    # centre (3.5, 3.5) is the principal point
    return Camera(np.eye(3), np.zeros(3), 10.0, 10.0, 3.5, 3.5, W, H)


def _scene(pos, rgb, logit=0.0, log_scale=-3.0, background=(0.0, 0.0, 0.0)):
    """Degree-0 scene whose Gaussians have colour `rgb` exactly:
    colour = max(SH_C0 * c0 + 0.5, 0) (ref rasterizer.py:149-153)."""
    pos = np.asarray(pos, float).reshape(-1, 3)
    g = pos.shape[0]
    rgb = np.asarray(rgb, float).reshape(g, 3)
    sh = ((rgb - 0.5) / SH_C0)[:, :, None]
    rot = np.tile([1.0, 0.0, 0.0, 0.0], (g, 1))
    return GaussianScene.from_arrays(pos, rot, np.full((g, 3), log_scale), np.full(g, logit), sh, 0, background)


def test_sort_x_spec_examples():
    """G=2, P=2, [a1,a2,b1,b2] -> [a1,b1,a2,b2]; G=1 identity; round trip."""
    v = ParamVector(torch.tensor([1.0, 2.0, 3.0, 4.0], dtype=torch.float64, device="cuda"),
                    Layout.ATTRIBUTE_MAJOR, 2, 2)
    assert sort_x(v).values.tolist() == [1.0, 3.0, 2.0, 4.0]
    one = ParamVector(torch.arange(14, dtype=torch.float64, device="cuda"), Layout.ATTRIBUTE_MAJOR, 1, 14)
    assert torch.equal(sort_x(one).values, one.values)
    r = ParamVector(torch.randn(7 * 59, dtype=torch.float64, device="cuda"), Layout.ATTRIBUTE_MAJOR, 7, 59)
    assert torch.equal(sort_x_inverse(sort_x(r)).values, r.values)


def test_render_empty_scene():
    """empty scene -> background image, empty traversals."""
    s = GaussianScene.from_arrays(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                                  np.zeros((0, 3, 1)), 0, (0.0, 0.0, 0.0))
    rr = R.render(s, _cam())
    assert torch.count_nonzero(rr.image) == 0
    assert rr.traversals.entry_count == 0
    assert torch.count_nonzero(rr.traversals.offsets) == 0
    assert torch.all(rr.traversals.t_final == 1.0)
    s_bg = GaussianScene(s.x, 0, (0.25, 0.5, 0.75))
    img = R.render(s_bg, _cam()).image
    assert torch.equal(img, torch.tensor([0.25, 0.5, 0.75], dtype=torch.float64, device="cuda").expand_as(img))


def test_render_one_splat_known_answer():
    """one splat at a pixel centre, opacity 0.5, colour (1,0,0), black
    background -> that pixel is (0.5, 0, 0)."""
    s = _scene([0.0, 0.0, 2.0], [1.0, 0.0, 0.0])
    rr = R.render(s, _cam())
    assert rr.image[3, 3].tolist() == [0.5, 0.0, 0.0]
    tr = rr.traversals
    p = 3 * 8 + 3
    o0, o1 = int(tr.offsets[p]), int(tr.offsets[p + 1])
    assert o1 - o0 == 1 and tr.alphas[o0].item() == 0.5 and tr.transmittances[o0].item() == 1.0


def test_render_two_stacked_splats_known_answer():
    """two stacked splats, alpha 0.5 each, (1,0,0) in front of
    (0,1,0) -> (0.5, 0.25, 0) with T = [1, 0.5]; the list order does not matter
    (depth order is canonical)."""
    for pos, rgb in (([[0, 0, 2.0], [0, 0, 3.0]], [[1, 0, 0], [0, 1, 0]]),
                     ([[0, 0, 3.0], [0, 0, 2.0]], [[0, 1, 0], [1, 0, 0]])):
        s = _scene(pos, rgb, log_scale=-4.0)
        rr = R.render(s, _cam())
        assert rr.image[3, 3].tolist() == [0.5, 0.25, 0.0]
        tr = rr.traversals
        p = 3 * 8 + 3
        o0, o1 = int(tr.offsets[p]), int(tr.offsets[p + 1])
        assert tr.transmittances[o0:o1].tolist() == [1.0, 0.5]
        assert tr.alphas[o0:o1].tolist() == [0.5, 0.5]


def test_render_zero_opacity_gives_background():
    """all opacities -> 0 gives the background everywhere."""
    truth, init, cams, gts = problem(seed=1, G=30, n_views=1, W=24, H=20, degree=1)
    h = init
    s = GaussianScene.from_arrays(h.positions, h.rotations, h.log_scales, np.full(30, -60.0), h.sh_coeffs,
                                  h.sh_degree, (0.2, 0.3, 0.4))
    rr = R.render(s, cams[0])
    bg = torch.tensor([0.2, 0.3, 0.4], dtype=torch.float64, device="cuda")
    assert torch.equal(rr.image, bg.expand_as(rr.image)) and rr.traversals.entry_count == 0


def test_residual_known_answers():
    """SPEC:218 (r_abs = sqrt(0.08) for |e| = 0.1), SPEC:227 (grad_r_sq 2.5 for
    |e| = 0.08), SPEC:228 (rendered = gt: finite), SPEC:229 (lambda1 = 0 and
    SSIM = 1 -> weight 0), SPEC:222 (rendered = gt -> energy 0) and the
    size / negative-weight guards."""
    gt = torch.full((9, 9, 3), 0.5, dtype=torch.float64, device="cuda")
    img = gt.clone()
    img[4, 4, 0] += 0.1
    b = RES.compute_residuals(img, gt, lambda1=0.8, lambda2=0.0)
    assert b.r_abs[4, 4, 0].item() == pytest.approx(np.sqrt(0.08), rel=1e-15)
    img2 = gt.clone()
    img2[4, 4, 1] -= 0.08
    b2 = RES.compute_residuals(img2, gt, lambda1=0.8, lambda2=0.0)
    assert b2.grad_r_sq[4, 4, 1].item() == pytest.approx(2.5, rel=1e-12)
    same = RES.compute_residuals(gt, gt)
    assert same.energy == 0.0 and torch.all(torch.isfinite(same.grad_r_sq))
    assert torch.count_nonzero(same.color_grad) == 0
    zero = RES.compute_residuals(gt, gt, lambda1=0.0, lambda2=0.2)
    # dSSIM/dc at img = gt is 0 up to the rounding of the windowed sums (1e-26
    # here, as in the fp64 oracle), so the weight is 0 to that level
    assert float(zero.grad_r_sq.abs().max()) < 1e-20
    ref = O.residuals(gt.cpu().numpy(), gt.cpu().numpy(), lambda1=0.0, lambda2=0.2)
    assert float(np.abs(ref["grad_r_sq"]).max()) < 1e-20
    with pytest.raises(ImageSizeError):
        RES.compute_residuals(gt, gt[:8])
    with pytest.raises(ValueError):
        RES.compute_residuals(gt, gt, lambda1=-1.0)


def _culled_problem():
    """Gaussian 0 sits behind the camera (culled); the others are seen."""
    truth, init, cams, gts = problem(seed=5, G=20, n_views=1, W=24, H=20, degree=1)
    c = cams[0]
    behind = c.center + 2.0 * (c.center - np.zeros(3))   # further out along the view axis, behind the eye
    pos = init.positions.copy()
    pos[0] = behind
    s = GaussianScene.from_arrays(pos, init.rotations, init.log_scales, init.opacity_logits, init.sh_coeffs,
                                  init.sh_degree)
    hs = type(init)(pos, init.rotations, init.log_scales, init.opacity_logits, init.sh_coeffs, init.sh_degree)
    return s, hs, c, gts[0]


def test_culled_gaussian_has_zero_diag_and_rhs():
    """a culled Gaussian's parameters get M = 0 (and b = 0) exactly."""
    s, hs, cam, gt = _culled_problem()
    assert not bool(R.project_scene(s, cam).valid[0])
    cs = CacheSet(s, [cam], [torch.from_numpy(gt).cuda()])
    G, P = s.num_gaussians, s.params_per_gaussian
    M = cs.diag().view(P, G)
    b = cs.rhs().view(P, G)
    assert torch.count_nonzero(M[:, 0]) == 0 and torch.count_nonzero(b[:, 0]) == 0
    assert torch.count_nonzero(M[:, 1:]) > 0
    osc, oc = oscene(hs), ocam(cam)
    rs = O.rasterize(osc, oc)
    bb, v = O.build_cache(osc, oc, O.residuals(rs["image"], gt), rast=rs)
    assert rel(cs.rhs().cpu().numpy(), bb) < 1e-5
    assert rel(cs.diag().cpu().numpy(), O.diag_jtj(osc, O.gaussian_order(v))) < 1e-5


def test_all_culled_scene_through_solver():
    """Every Gaussian behind the camera: E = 0, b = 0, M = 0; PCG returns
    Delta = 0 without a product and the LM direction is 0."""
    truth, init, cams, gts = problem(seed=6, G=12, n_views=2, W=24, H=20, degree=2)
    pos = np.tile(cams[0].center * 3.0, (12, 1))            # all behind view 0 ...
    s = GaussianScene.from_arrays(pos, init.rotations, init.log_scales, init.opacity_logits, init.sh_coeffs, 2)
    cam = [cams[0]]
    gt = [torch.from_numpy(gts[0]).cuda()]
    cs = CacheSet(s, cam, gt)
    assert cs.E == 0 and cs.R == 0
    assert torch.count_nonzero(cs.rhs()) == 0 and torch.count_nonzero(cs.diag()) == 0
    st = {}
    x = pcg_run(cs, cs.rhs(), cs.diag(), 1e-4, 8, stats=st)
    assert torch.count_nonzero(x) == 0 and st["iterations"] == 0
    out = torch.empty(s.param_count, dtype=torch.float32, device="cuda")
    cs.jtwj(torch.randn(s.param_count, device="cuda"), out)
    assert torch.count_nonzero(out) == 0
    rep = lm_direction(s, cam, gt, BatchSchedule(1), 1e-4, 8)
    assert torch.count_nonzero(rep.delta) == 0
    assert cs.energies[0] == pytest.approx(RES.compute_residuals(torch.zeros_like(gt[0]), gt[0]).energy, rel=1e-12)


def test_empty_scene_cache():
    """empty scene -> empty cache, b = 0 (length 0); the energy is
    that of the background image."""
    s = GaussianScene.from_arrays(np.zeros((0, 3)), np.zeros((0, 4)), np.zeros((0, 3)), np.zeros(0),
                                  np.zeros((0, 3, 16)), 3, (0.0, 0.0, 0.0))
    cam = _cam(16, 12)
    gt = torch.rand(12, 16, 3, dtype=torch.float64, device="cuda", generator=torch.Generator("cuda").manual_seed(0))
    cs = CacheSet(s, [cam], [gt])
    assert cs.E == 0 and cs.rhs().numel() == 0 and cs.diag().numel() == 0
    assert cs.energies[0] == pytest.approx(RES.compute_residuals(torch.zeros_like(gt), gt).energy, rel=1e-12)
    rep = lm_direction(s, [cam], [gt], BatchSchedule(1), 1e-4, 8)
    assert rep.delta.numel() == 0


def test_smooth_config_traversals_and_products():
    """RenderConfig.smooth(): every alpha > 0 down to exp underflow is kept,
    no termination, no cull -- traversals bit-exact vs the oracle with the same
    config, products within the fp32 tolerance."""
    truth, init, cams, gts = problem(seed=3, G=25, n_views=2, W=20, H=16, degree=1)
    cfg = R.RenderConfig.smooth()
    ocfg = O.OConfig(alpha_min=0.0, t_stop=0.0, cull_sigma=None)
    s, osc = init.to_device(), oscene(init)
    views = []
    for c in cams:
        oc = ocam(c)
        rr = R.render(s, c, config=cfg)
        rs = O.rasterize(osc, oc, ocfg)
        tr = rr.traversals
        assert np.array_equal(tr.offsets.cpu().numpy(), rs["offsets"])
        assert np.array_equal(tr.gaussian_ids.cpu().numpy(), rs["gid"])
        assert rel(tr.alphas.cpu().numpy(), rs["alpha"]) < 1e-12
        assert rel(rr.image.cpu().numpy(), rs["image"]) < 1e-12
        # far tails are kept: far more entries than under the default config
        assert tr.entry_count > 3 * R.render(s, c).traversals.entry_count
        gt = gts[cams.index(c)]
        _, v = O.build_cache(osc, oc, O.residuals(rs["image"], gt), ocfg, rast=rs)
        views.append(O.gaussian_order(v))
    cs = CacheSet(s, cams, [torch.from_numpy(g).cuda() for g in gts], config=cfg)
    assert cs.E == sum(v.E for v in views)
    ex = cs.export_view(0)
    assert np.array_equal(ex["g_source_index"], views[0].src)
    p = np.random.default_rng(1).standard_normal(s.param_count)
    out = torch.empty(s.param_count, dtype=torch.float32, device="cuda")
    cs.jtwj(torch.from_numpy(p).float().cuda(), out)
    assert rel(out.cpu().numpy(), O.jtwj(p, osc, views)) < 1e-5
    assert rel(cs.diag().cpu().numpy(), sum(O.diag_jtj(osc, v) for v in views)) < 1e-5
