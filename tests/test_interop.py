"""Interop formats: scene / camera JSON (ref: scene.py:420-472)
and the GCCH cache dump (ref: jacobian.py:618-656)."""
import numpy as np
import pytest
import torch

import oracle as O
from helpers import ocam, oscene, problem, rel
from paper_2409_12892_b200 import scene as SC
from paper_2409_12892_b200 import synthetic as S


@pytest.mark.reference
def test_scene_and_camera_json_match_reference(ref_modules):
    RS = ref_modules[0]
    truth, cams, _ = RS.make_synthetic_dataset(3, 12, 2, (8, 6), sh_degree=2)
    h = S.make_synthetic_scene(3, 12, 2)
    ours = SC.GaussianScene.from_arrays(h.positions, h.rotations, h.log_scales, h.opacity_logits, h.sh_coeffs,
                                        h.sh_degree, h.background, device="cpu")
    txt = SC.scene_to_json(ours)
    assert txt == RS.scene_to_json(truth)                      # byte-identical
    back = RS.scene_from_json(txt)
    for f in ("positions", "rotations", "log_scales", "opacity_logits", "sh_coeffs"):
        assert np.array_equal(getattr(back, f), getattr(truth, f))
    again = SC.scene_from_json(RS.scene_to_json(truth), device="cpu")
    assert torch.equal(again.x, ours.x)
    ctxt = SC.cameras_to_json(S.make_camera_ring(2, 8, 6))
    assert ctxt == RS.cameras_to_json(cams)
    for a, b in zip(SC.cameras_from_json(ctxt), cams):
        assert np.array_equal(a.rotation, b.rotation) and np.array_equal(a.translation, b.translation)


@pytest.mark.gpu
def test_cache_dump_matches_oracle(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2409_12892_b200 import jacobian as J
    from paper_2409_12892_b200 import rasterizer as R
    from paper_2409_12892_b200 import residuals as RES
    truth, init, cams, gts = problem(seed=5, G=50, n_views=1, W=32, H=24, degree=1)
    s, c = init.to_device(), cams[0]
    bundle = RES.compute_residuals(R.render(s, c, traversals=False).image, torch.from_numpy(gts[0]).cuda())
    _, cache = J.build_cache(s, c, bundle)
    path = tmp_path / "cache.gcch"
    J.dump_cache(cache, path)
    d = J.load_cache_dump(path)
    osc, oc = oscene(init), ocam(c)
    rs = O.rasterize(osc, oc)
    _, v = O.build_cache(osc, oc, O.residuals(rs["image"], gts[0]), rast=rs)
    assert d["order"] is J.CacheOrder.PIXEL_SORTED and d["n_pixels"] == c.num_pixels
    assert np.array_equal(d["pixel_ids"], v.pixel) and np.array_equal(d["gaussian_ids"], v.gid)
    assert rel(d["alphas"], v.alpha) < 1e-7 and rel(d["transmittances"], v.T) < 1e-6
    assert rel(d["dc_dalpha"], v.dcda) < 1e-6 and rel(d["dc_dcs"], v.dcdc) < 1e-7


def test_pfm_roundtrip(tmp_path):
    from paper_2409_12892_b200 import imageio as IO
    img = np.random.default_rng(0).standard_normal((5, 7, 3)).astype(np.float32)
    IO.write_pfm(tmp_path / "a.pfm", torch.from_numpy(img))
    back = IO.read_pfm(tmp_path / "a.pfm")
    assert back.dtype == np.float64 and np.array_equal(back, img.astype(np.float64))
    with pytest.raises(ValueError):
        IO.write_pfm(tmp_path / "b.pfm", img[..., :2])


@pytest.mark.reference
def test_pfm_png_match_reference(ref_modules, tmp_path):
    import sys
    from paper_2409_12892_b200 import imageio as IO
    sys.path.insert(0, "/root/reference/pkg/src")
    from splatlm import imageio as RI
    img = np.random.default_rng(1).uniform(-0.2, 1.2, (6, 9, 3))
    IO.write_pfm(tmp_path / "o.pfm", img)
    RI.write_pfm(tmp_path / "r.pfm", img)
    assert (tmp_path / "o.pfm").read_bytes() == (tmp_path / "r.pfm").read_bytes()
    assert np.array_equal(IO.read_pfm(tmp_path / "r.pfm"), RI.read_pfm(tmp_path / "o.pfm"))
    IO.write_png(tmp_path / "o.png", img)
    RI.write_png(tmp_path / "r.png", img)
    assert np.array_equal(IO.read_png(tmp_path / "o.png"), RI.read_png(tmp_path / "r.png"))
