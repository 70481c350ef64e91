"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle.

Bit-exact: valid mask, per-pixel entry sequence and offsets, gaussian-order
permutation (= source_index) and offsets.  Float: images/alpha/T 1e-12
(fp64 rasteriser); cache records and products rel-L2 <= 1e-5 (fp32 cache,
tolerance of BASELINE.json north_star / SURVEY 8c).
"""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import ocam, oscene, problem, rel
from paper_2409_12892_b200 import jacobian as J
from paper_2409_12892_b200 import rasterizer as R
from paper_2409_12892_b200 import residuals as RES
from paper_2409_12892_b200.engine import CacheSet, LossConfig
from paper_2409_12892_b200.scene import Layout, ParamVector, flatten, sort_x, sort_x_inverse
from paper_2409_12892_b200.solver import BatchSchedule, lm_direction, pcg_run

pytestmark = pytest.mark.gpu

FTOL = 1e-5


@pytest.fixture(scope="module")
def prob():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    truth, init, cams, gts = problem(seed=0, G=60, n_views=3, W=32, H=28, degree=3)
    scene = init.to_device()
    gts_d = [torch.from_numpy(g).cuda() for g in gts]
    return dict(init=init, cams=cams, gts=gts, scene=scene, gts_d=gts_d, osc=oscene(init),
                ocams=[ocam(c) for c in cams])


@pytest.fixture(scope="module")
def oracle_views(prob):
    out = []
    for c, gt in zip(prob["ocams"], prob["gts"]):
        rs = O.rasterize(prob["osc"], c)
        res = O.residuals(rs["image"], gt)
        b, v = O.build_cache(prob["osc"], c, res, rast=rs)
        out.append(dict(rast=rs, res=res, b=b, view=v, gview=O.gaussian_order(v)))
    return out


@pytest.fixture(scope="module")
def cacheset(prob):
    return CacheSet(prob["scene"], prob["cams"], prob["gts_d"], residual_exports=True)


def test_sort_x_roundtrip(prob):
    s = prob["scene"]
    v = flatten(s)
    gm = sort_x(v)
    ref = O.gm_from_am(v.values.cpu().numpy(), s.num_gaussians)
    assert np.array_equal(gm.values.cpu().numpy(), ref)
    assert torch.equal(sort_x_inverse(gm).values, v.values)


def test_project_valid_mask(prob):
    for c, oc in zip(prob["cams"], prob["ocams"]):
        pr = R.project_scene(prob["scene"], c)
        po = O.project(prob["osc"], oc)
        assert np.array_equal(pr.valid.cpu().numpy(), po["valid"])
        m = po["valid"]
        assert rel(pr.mean2d.cpu().numpy()[m], po["mean"][m]) < 1e-13
        assert rel(pr.conic.cpu().numpy()[m], po["conic"][m]) < 1e-12
        assert np.array_equal(pr.color_clamped.cpu().numpy()[m], po["clamped"][m])


def test_render_traversals_bit_exact(prob, oracle_views):
    for c, ov in zip(prob["cams"], oracle_views):
        rr = R.render(prob["scene"], c)
        rs = ov["rast"]
        tr = rr.traversals
        assert rel(rr.image.cpu().numpy(), rs["image"]) < 1e-12
        assert np.array_equal(tr.offsets.cpu().numpy(), rs["offsets"])
        assert np.array_equal(tr.gaussian_ids.cpu().numpy(), rs["gid"])
        assert rel(tr.alphas.cpu().numpy(), rs["alpha"]) < 1e-12
        assert rel(tr.transmittances.cpu().numpy(), rs["T"]) < 1e-12
        assert rel(tr.t_final.cpu().numpy(), rs["t_final"]) < 1e-12


def test_residuals(prob, oracle_views):
    for v, ov in enumerate(oracle_views):
        img = torch.from_numpy(ov["rast"]["image"]).cuda()
        b = RES.compute_residuals(img, prob["gts_d"][v])
        for k_ours, k_or in (("grad_r_sq", "grad_r_sq"), ("color_grad", "color_grad"), ("r_abs", "r_abs"),
                             ("r_ssim", "r_ssim")):
            assert rel(getattr(b, k_ours).cpu().numpy(), ov["res"][k_or]) < 1e-10, k_ours
        assert abs(b.energy - ov["res"]["energy"]) <= 1e-12 * abs(ov["res"]["energy"])


def test_residuals_l2_mode(prob, oracle_views):
    img = torch.from_numpy(oracle_views[0]["rast"]["image"]).cuda()
    b = RES.compute_residuals(img, prob["gts_d"][0], mode="l2")
    assert torch.all(b.grad_r_sq == 1)
    ref = O.residuals(oracle_views[0]["rast"]["image"], prob["gts"][0], mode="l2")
    assert rel(b.color_grad.cpu().numpy(), ref["color_grad"]) < 1e-14


def test_cache_indexing_bit_exact(cacheset, oracle_views):
    for v, ov in enumerate(oracle_views):
        ex = cacheset.export_view(v)
        ref, gref = ov["view"], ov["gview"]
        assert np.array_equal(ex["offsets"], ref.offsets)
        assert np.array_equal(ex["pixel_ids"], ref.pixel)
        assert np.array_equal(ex["gaussian_ids"], ref.gid)
        assert np.array_equal(ex["g_gaussian_ids"], gref.gid)
        assert np.array_equal(ex["g_pixel_ids"], gref.pixel)
        assert np.array_equal(ex["g_offsets"], gref.offsets)
        assert np.array_equal(ex["g_source_index"], gref.src)
        assert rel(ex["alphas"], ref.alpha) < 1e-7
        assert rel(ex["dc_dcs"], ref.dcdc) < 1e-7
        assert rel(ex["dc_dalpha"], ref.dcda) < 1e-6
        assert rel(ex["g_dc_dalpha"], gref.dcda) < 1e-6


def test_rhs_and_diag(prob, cacheset, oracle_views):
    b_ref = sum(ov["b"] for ov in oracle_views)
    M_ref = sum(O.diag_jtj(prob["osc"], ov["gview"]) for ov in oracle_views)
    assert rel(cacheset.rhs().cpu().numpy(), b_ref) < FTOL
    assert rel(cacheset.diag().cpu().numpy(), M_ref) < FTOL


def test_products(prob, cacheset, oracle_views):
    s = prob["scene"]
    rng = np.random.default_rng(3)
    p = rng.standard_normal(s.param_count)
    u_ref = np.concatenate([O.apply_j(p, prob["osc"], ov["gview"]) for ov in oracle_views])
    pd = torch.from_numpy(p).float().cuda()
    cacheset.pair_forward(pd)
    u = cacheset.apply_j_raw(weighted=False).view(-1, 4)[:, :3].reshape(-1).cpu().numpy()
    assert rel(u, u_ref) < FTOL
    uu = rng.standard_normal(u_ref.size)
    off = 0
    g_ref = np.zeros(s.param_count)
    for ov in oracle_views:
        n = ov["view"].cam.width * ov["view"].cam.height * 3
        g_ref += O.apply_jt(uu[off:off + n], prob["osc"], ov["gview"])
        off += n
    u4 = torch.zeros(u_ref.size // 3, 4, dtype=torch.float32, device="cuda")
    u4[:, :3] = torch.from_numpy(uu).view(-1, 3)
    g = torch.empty(s.param_count, dtype=torch.float32, device="cuda")
    cacheset.apply_jt_raw(u4.view(-1), g)
    assert rel(g.cpu().numpy(), g_ref) < FTOL
    # fused J^T W J p with the residual weighting
    jtwj_ref = O.jtwj(p, prob["osc"], [ov["gview"] for ov in oracle_views])
    out = torch.empty_like(g)
    cacheset.jtwj(pd, out)
    assert rel(out.cpu().numpy(), jtwj_ref) < FTOL


def test_reference_api_products(prob, oracle_views):
    s, c = prob["scene"], prob["cams"][0]
    ov = oracle_views[0]
    bundle = RES.compute_residuals(R.render(s, c, traversals=False).image, prob["gts_d"][0])
    b, cache = J.build_cache(s, c, bundle)
    assert rel(b.values.cpu().numpy(), ov["b"]) < FTOL
    with pytest.raises(J.CacheOrderError):
        J.apply_jt(torch.zeros(c.num_pixels * 3, device="cuda"), s, cache)
    gc = J.sort_cache_by_gaussians(cache)
    rng = np.random.default_rng(9)
    p = rng.standard_normal(s.param_count)
    pv = ParamVector(torch.from_numpy(p).cuda(), Layout.ATTRIBUTE_MAJOR, s.num_gaussians, s.params_per_gaussian)
    with pytest.raises(J.LayoutError if hasattr(J, "LayoutError") else Exception):
        J.apply_j(pv, s, gc)
    u = J.apply_j(sort_x(pv), s, gc)
    assert rel(u.cpu().numpy(), O.apply_j(p, prob["osc"], ov["gview"])) < FTOL
    w = J.weight_residuals(u, bundle)
    g = J.apply_jt(w, s, gc)
    ref = O.apply_jt(O.weight(O.apply_j(p, prob["osc"], ov["gview"]), ov["gview"]), prob["osc"], ov["gview"])
    assert rel(g.values.cpu().numpy(), ref) < FTOL
    M = J.diag_jtj(s, gc)
    assert rel(M.values.cpu().numpy(), O.diag_jtj(prob["osc"], ov["gview"])) < FTOL


@pytest.fixture(scope="module")
def posed():
    """A well-posed solve (every Gaussian seen by several 48x48 views).  The
    3-view 32x28 problem above is so under-determined that 8 PCG iterations
    amplify 2e-7 product rounding into 1e-3..1e-2 changes of Delta (measured,
    tools/diag_precision.py); here the same kernels agree to ~5e-6."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    truth, init, cams, gts = problem(seed=2, G=100, n_views=6, W=48, H=48, degree=3)
    osc = oscene(init)
    ocs = [ocam(c) for c in cams]
    views, b = [], 0
    for c, gt in zip(ocs, gts):
        rs = O.rasterize(osc, c)
        bb, v = O.build_cache(osc, c, O.residuals(rs["image"], gt), rast=rs)
        views.append(O.gaussian_order(v))
        b = b + bb
    M = sum(O.diag_jtj(osc, v) for v in views)
    return dict(init=init, cams=cams, gts=gts, osc=osc, ocams=ocs, views=views, b=b, M=M,
                scene=init.to_device(), gts_d=[torch.from_numpy(g).cuda() for g in gts])


PCG_TOL = 1e-4  # rel-L2 of Delta vs the fp64 oracle after n iterations (measured <= 6e-6)


def test_pcg_parity(posed):
    cs = CacheSet(posed["scene"], posed["cams"], posed["gts_d"])
    assert rel(cs.rhs().cpu().numpy(), posed["b"]) < FTOL
    assert rel(cs.diag().cpu().numpy(), posed["M"]) < FTOL
    for lam, iters in ((1.0, 6), (1e-4, 8)):
        st = {}
        ref = O.pcg(posed["osc"], posed["views"], posed["b"], posed["M"], lam, iters, stats=st)
        gst = {}
        x = pcg_run(cs, cs.rhs(), cs.diag(), lam, iters, stats=gst).cpu().numpy()
        assert gst["products"] == st["products"]
        assert rel(x, ref) < PCG_TOL, (lam, rel(x, ref))
        assert np.all(np.isfinite(x))


def test_pcg_large_lambda(posed):
    """lambda = 1e6 gives Delta ~= b / (lambda M) within 1%."""
    cs = CacheSet(posed["scene"], posed["cams"], posed["gts_d"])
    lam = 1e6
    x = pcg_run(cs, cs.rhs(), cs.diag(), lam, 8).cpu().numpy()
    approx = posed["b"] / (lam * np.maximum(posed["M"], 1e-12))
    assert rel(x, approx) < 1e-2


def test_pcg_zero_rhs(posed):
    """b = 0 gives Delta = 0 without a product."""
    cs = CacheSet(posed["scene"], posed["cams"], posed["gts_d"])
    st = {}
    x = pcg_run(cs, torch.zeros_like(cs.rhs()), cs.diag(), 1e-4, 8, stats=st)
    assert torch.count_nonzero(x) == 0


def test_lm_direction_batched(posed):
    ref = O.lm_direction(posed["osc"], posed["ocams"], posed["gts"], n_batches=2, lam=1e-4, n_iters=8)
    rep = lm_direction(posed["scene"], posed["cams"], posed["gts_d"], BatchSchedule(2), 1e-4, 8)
    assert rep.batches_accepted == 2
    assert rel(rep.delta.cpu().numpy(), ref) < PCG_TOL


def test_lm_direction_host_images(posed):
    """Ground truth in pinned host memory (copied per subset on a side stream
    while the previous subset is solved) gives the same bits as device images."""
    dev = lm_direction(posed["scene"], posed["cams"], posed["gts_d"], BatchSchedule(2), 1e-4, 8)
    host = [g.cpu().pin_memory() for g in posed["gts_d"]]
    hst = lm_direction(posed["scene"], posed["cams"], host, BatchSchedule(2), 1e-4, 8)
    assert torch.equal(dev.delta, hst.delta)


def test_determinism(prob):
    outs = []
    for _ in range(2):
        cs = CacheSet(prob["scene"], prob["cams"], prob["gts_d"])
        x = pcg_run(cs, cs.rhs(), cs.diag(), 1e-2, 4)
        outs.append((cs.rhs().clone(), cs.diag().clone(), x.clone()))
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_entry_count_matches_traversals(prob, cacheset, oracle_views):
    assert cacheset.E == sum(ov["rast"]["pixel"].size for ov in oracle_views)


@pytest.fixture(scope="module")
def dense():
    """C1-density view (2k Gaussians, 64x64, ~77 entries/pixel): tiles hold more
    than 256 runs and rasteriser batches of more than 256 splats."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    truth, init, cams, gts = problem(seed=0, G=2000, n_views=1, W=64, H=64, degree=3)
    osc, oc = oscene(init), ocam(cams[0])
    rs = O.rasterize(osc, oc)
    res = O.residuals(rs["image"], gts[0])
    b, v = O.build_cache(osc, oc, res, rast=rs)
    scene = init.to_device()
    cs = CacheSet(scene, cams, [torch.from_numpy(gts[0]).cuda()])
    return dict(osc=osc, scene=scene, cs=cs, b=b, view=v, gview=O.gaussian_order(v), rast=rs)


def test_dense_indexing_and_products(dense):
    cs, v, gv = dense["cs"], dense["view"], dense["gview"]
    assert cs.E == v.E and cs.R > 256 * 4
    ex = cs.export_view(0)
    assert np.array_equal(ex["offsets"], v.offsets)
    assert np.array_equal(ex["gaussian_ids"], v.gid)
    assert np.array_equal(ex["g_source_index"], gv.src)
    assert rel(cs.rhs().cpu().numpy(), dense["b"]) < FTOL
    assert rel(cs.diag().cpu().numpy(), O.diag_jtj(dense["osc"], gv)) < FTOL
    rng = np.random.default_rng(5)
    p = rng.standard_normal(dense["scene"].param_count)
    out = torch.empty(p.size, dtype=torch.float32, device="cuda")
    cs.jtwj(torch.from_numpy(p).float().cuda(), out)
    assert rel(out.cpu().numpy(), O.jtwj(p, dense["osc"], [gv])) < FTOL


@pytest.mark.parametrize("degree", [0, 1, 2])
def test_products_all_sh_degrees(degree):
    """b, M and J^T W J p at every SH degree (P = 14 .. 38 < 64 exercises the
    partial-row paths of the per-gaussian backward)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    truth, init, cams, gts = problem(seed=4, G=40, n_views=2, W=24, H=20, degree=degree)
    osc = oscene(init)
    gv, b = [], 0
    for c, gt in zip(cams, gts):
        oc = ocam(c)
        rs = O.rasterize(osc, oc)
        bb, v = O.build_cache(osc, oc, O.residuals(rs["image"], gt), rast=rs)
        gv.append(O.gaussian_order(v))
        b = b + bb
    scene = init.to_device()
    cs = CacheSet(scene, cams, [torch.from_numpy(g).cuda() for g in gts])
    assert rel(cs.rhs().cpu().numpy(), b) < FTOL
    assert rel(cs.diag().cpu().numpy(), sum(O.diag_jtj(osc, v) for v in gv)) < FTOL
    p = np.random.default_rng(degree).standard_normal(scene.param_count)
    out = torch.empty(p.size, dtype=torch.float32, device="cuda")
    cs.jtwj(torch.from_numpy(p).float().cuda(), out)
    assert rel(out.cpu().numpy(), O.jtwj(p, osc, gv)) < FTOL


def test_determinism_at_scale():
    """Bitwise run-to-run determinism of b, M and J^T W J p on a C2-sized subset
    (100k Gaussians, 8 views @ 256^2): the streaming kernel's shared-memory ring
    is reused many times per CTA here (the small problems above never wrap it)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2409_12892_b200 import synthetic as S
    from paper_2409_12892_b200.rasterizer import render
    truth = S.make_synthetic_scene(0, 100_000, 3)
    init = S.perturb(truth, 1, 0.1)
    cams = S.make_camera_ring(8, 256, 256)
    ts = truth.to_device()
    gts = [render(ts, c, traversals=False).image.float().contiguous() for c in cams]
    scene = init.to_device()
    p = torch.randn(scene.param_count, device="cuda", generator=torch.Generator("cuda").manual_seed(7))
    outs = []
    for _ in range(2):
        cs = CacheSet(scene, cams, gts)
        g = torch.empty_like(p)
        cs.jtwj(p, g, 1e-4, cs.diag())
        outs.append((cs.rhs().clone(), cs.diag().clone(), g))
        del cs
    for a, b in zip(outs[0], outs[1]):
        assert torch.equal(a, b)


def test_forward_chain_dsigma_path(prob, cacheset, oracle_views):
    """The PCG path's forward chain (padded gaussian-major p carrying the
    world-covariance perturbation, slm_gm_pack / slm_pcg_p*) gives the same
    product as the attribute-major path and the oracle."""
    s = prob["scene"]
    p = np.random.default_rng(11).standard_normal(s.param_count)
    pd = torch.from_numpy(p).float().cuda()
    ref = O.jtwj(p, prob["osc"], [ov["gview"] for ov in oracle_views])
    a, b = torch.empty_like(pd), torch.empty_like(pd)
    cacheset.jtwj(pd, a)
    cacheset.jtwj(pd, b, p_gm=cacheset.gm_pack(pd))
    assert rel(b.cpu().numpy(), a.cpu().numpy()) < 1e-5
    assert rel(b.cpu().numpy(), ref) < FTOL


@pytest.mark.gpu
@pytest.mark.parametrize("lanes_threshold", [0, 10 ** 9])   # 0: always 8 J^T lanes per run; 1e9: always 4
def test_jt_group_widths(prob, cacheset, oracle_views, monkeypatch, lanes_threshold):
    """Both J^T group widths (stream.cu launch_stream: 8 lanes per run, or 4
    below engine.JT4_ENTRIES_PER_RUN entries per run) against the oracle."""
    from paper_2409_12892_b200 import engine
    monkeypatch.setattr(engine, "JT4_ENTRIES_PER_RUN", lanes_threshold)
    assert cacheset._tile_args().jt_lanes == (8 if lanes_threshold == 0 else 4)
    s = prob["scene"]
    rng = np.random.default_rng(7)
    p = rng.standard_normal(s.param_count)
    out = torch.empty(s.param_count, dtype=torch.float32, device="cuda")
    cacheset.jtwj(torch.from_numpy(p).float().cuda(), out)
    assert rel(out.cpu().numpy(), O.jtwj(p, prob["osc"], [ov["gview"] for ov in oracle_views])) < FTOL
    uu = rng.standard_normal(sum(ov["view"].cam.width * ov["view"].cam.height * 3 for ov in oracle_views))
    g_ref, off = np.zeros(s.param_count), 0
    for ov in oracle_views:
        n = ov["view"].cam.width * ov["view"].cam.height * 3
        g_ref += O.apply_jt(uu[off:off + n], prob["osc"], ov["gview"])
        off += n
    u4 = torch.zeros(uu.size // 3, 4, dtype=torch.float32, device="cuda")
    u4[:, :3] = torch.from_numpy(uu).float().view(-1, 3)
    g = torch.empty(s.param_count, dtype=torch.float32, device="cuda")
    cacheset.apply_jt_raw(u4.view(-1), g)
    assert rel(g.cpu().numpy(), g_ref) < FTOL
