"""GPU parity in the C3 regime (BASELINE configs[2] generator, 1M Gaussians,
K ~ 39-62 entries per pixel) against the fp64 oracle.

The oracle cannot run a 1024x1024 view in test time, so the view is a window
of the C3 camera: same pose and focal length, principal point shifted, 144 x
120 pixels (a partial tile row and column) where the footprint generator is
densest.  Every pixel of the window sees exactly the splats of the full view
(per-pixel blending, global depth order), so the cache has the C3 shape:
multi-chunk tiles (tens of thousands of entries per tile), long runs, the
dynamic tile queue and many wraps of the streaming kernel's ring.

Bit-exact: per-pixel entry sequence, offsets, gaussian-order permutation
(source_index) and offsets, exported from the device run order.  Float:
energy 1e-12, records 1e-6..1e-7, b, M and one fused J^T W J p <= 1e-5
(fp32 cache).
"""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import ocam, oscene, rel
from paper_2409_12892_b200 import synthetic as S
from paper_2409_12892_b200.scene import Camera

pytestmark = pytest.mark.gpu
FTOL = 1e-5
WIN = (440, 452, 144, 120)   # x0, y0, width, height of the window of view 0


@pytest.fixture(scope="module")
def big():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2409_12892_b200.engine import CacheSet
    from paper_2409_12892_b200.rasterizer import render
    truth = S.make_footprint_scene(0, 1_000_000, 1024, 1024, 3, k_target=32.0)
    init = S.perturb(truth, 1, 0.02)
    c = S.make_camera_ring(200, 1024, 1024)[0]
    ox, oy, w, h = WIN
    cam = Camera(c.rotation, c.translation, c.fx, c.fy, c.cx - ox, c.cy - oy, w, h)
    gt = render(truth.to_device(), cam, traversals=False).image
    scene = init.to_device()
    cs = CacheSet(scene, [cam], [gt])
    osc = oscene(init)
    rs = O.rasterize(osc, ocam(cam))
    res = O.residuals(rs["image"], gt.cpu().numpy())
    b, v = O.build_cache(osc, ocam(cam), res, rast=rs)
    return dict(cs=cs, osc=osc, cam=cam, rs=rs, res=res, b=b, view=v, gview=O.gaussian_order(v), scene=scene)


def test_regime_shape(big):
    """The window really is in the C3 regime the bench runs."""
    cs = big["cs"]
    k = cs.E / cs.N
    assert 30 < k < 120, k
    assert cs.E == big["view"].pixel.size
    assert cs.n_chunks > 4 * cs.n_tiles_total        # multi-chunk tiles
    assert cs.E / cs.R > 15                           # long runs


def test_energy_and_image(big):
    cs = big["cs"]
    assert abs(cs.energies[0] - big["res"]["energy"]) <= 1e-12 * big["res"]["energy"]
    img = cs.image(0).cpu().numpy()
    assert np.max(np.abs(img - big["rs"]["image"])) < 1e-12


def test_indices_bit_exact(big):
    ex = big["cs"].export_view(0)
    ref, gref = big["view"], big["gview"]
    assert np.array_equal(ex["offsets"], ref.offsets)
    assert np.array_equal(ex["pixel_ids"], ref.pixel)
    assert np.array_equal(ex["gaussian_ids"], ref.gid)
    assert np.array_equal(ex["g_offsets"], gref.offsets)
    assert np.array_equal(ex["g_pixel_ids"], gref.pixel)
    assert np.array_equal(ex["g_gaussian_ids"], gref.gid)
    assert np.array_equal(ex["g_source_index"], gref.src)
    assert rel(ex["alphas"], ref.alpha) < 1e-7
    assert rel(ex["dc_dcs"], ref.dcdc) < 1e-7
    assert rel(ex["dc_dalpha"], ref.dcda) < 1e-6


def test_rhs_diag_product(big):
    cs, osc, gv = big["cs"], big["osc"], big["gview"]
    assert rel(cs.rhs().cpu().numpy(), big["b"]) < FTOL
    M = O.diag_jtj(osc, gv)
    assert rel(cs.diag().cpu().numpy(), M) < FTOL
    p = np.random.default_rng(5).standard_normal(osc.G * O.params_per_gaussian(osc.degree))
    ref = O.jtwj(p, osc, [gv])
    out = torch.empty(p.size, dtype=torch.float32, device="cuda")
    cs.jtwj(torch.from_numpy(p).float().cuda(), out)
    assert rel(out.cpu().numpy(), ref) < FTOL
