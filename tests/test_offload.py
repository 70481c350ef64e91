"""Cache offload ("CPU offloading of cache parts"): the tail
of the run-ordered record streams lives in host-pinned, device-mapped memory
that the FILL pass writes and the streaming kernels' TMA reads over the host
link.  The arithmetic is unchanged, so every product, b, M, the exports and
the PCG direction must be BIT-identical to the all-HBM cache."""
import numpy as np
import pytest
import torch

from paper_2409_12892_b200 import synthetic as S

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def caches():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2409_12892_b200.engine import CacheSet
    from paper_2409_12892_b200.rasterizer import render
    truth = S.make_footprint_scene(0, 20000, 128, 128, 3, k_target=32.0)
    init = S.perturb(truth, 1, 0.02)
    cams = S.make_camera_ring(4, 128, 128)
    tsc = truth.to_device()
    gts = [render(tsc, c, traversals=False).image for c in cams]
    scene = init.to_device()
    out = {f: CacheSet(scene, cams, gts, offload=f) for f in (None, 0.5, 1.0, "auto")}
    return dict(c=out, scene=scene, cams=cams, gts=gts)


def test_split(caches):
    c = caches["c"]
    E = c[None].E
    assert c[None].offloaded_entries == 0 and c["auto"].offloaded_entries == 0   # fits in HBM
    assert 0 < c[0.5].offloaded_entries < E
    assert abs(c[0.5].offloaded_entries - E / 2) < 0.05 * E
    assert c[1.0].offloaded_entries == E and c[1.0].e_split == 0
    assert c[0.5].rec4_h.is_pinned()


@pytest.mark.parametrize("f", [0.5, 1.0])
def test_products_bit_identical(caches, f):
    a, b = caches["c"][None], caches["c"][f]
    assert torch.equal(a.rhs(), b.rhs())
    assert torch.equal(a.diag(), b.diag())
    p = torch.from_numpy(np.random.default_rng(1).standard_normal(a.G * a.P)).float().cuda()
    ga, gb = torch.empty_like(p), torch.empty_like(p)
    a.jtwj(p, ga, 1e-4, a.diag())
    b.jtwj(p, gb, 1e-4, b.diag())
    assert torch.equal(ga, gb)
    a.pair_forward(p)
    b.pair_forward(p)
    assert torch.equal(a.apply_j_raw(True).clone(), b.apply_j_raw(True).clone())


def test_exports_identical(caches):
    a, b = caches["c"][None], caches["c"][0.5]
    for v in range(len(caches["cams"])):
        ea, eb = a.export_view(v), b.export_view(v)
        for k in ea:
            assert np.array_equal(ea[k], eb[k]), (v, k)


def test_direction_identical(caches):
    from paper_2409_12892_b200.solver import BatchSchedule, lm_direction
    s, cams, gts = caches["scene"], caches["cams"], caches["gts"]
    d0 = lm_direction(s, cams, gts, BatchSchedule(2), 1e-4, 6)
    d1 = lm_direction(s, cams, gts, BatchSchedule(2), 1e-4, 6, offload=0.5)
    assert all(e > 0 for e in d1.offloaded_entries)
    assert torch.equal(d0.delta, d1.delta)
