"""Stage 1 (ADAM), lm_fit, the two-stage driver and the CLI (SURVEY 8(f) row
4).  The reference has these as SPEC only, so the
gradient is pinned to the oracle's b (itself pinned to the reference's
build_cache) and the drivers to the SPEC's examples."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import oracle as O
from helpers import ocam, oscene, problem, rel
from paper_2409_12892_b200 import __main__ as cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_parse_config():
    cfg = cli.parse_config("# comment\nlm_iters = 3\n\nloss = l2  # trailing\nlambda_reg=0.01\n")
    assert cfg["lm_iters"] == 3 and cfg["loss"] == "l2" and cfg["lambda_reg"] == 0.01
    assert cfg["pcg_iters"] == 8 and cfg["stage1_iters"] == 200          # defaults
    for text, line in (("lm_iters = 3\nbogus = 1\n", 2), ("pcg_iters = eight\n", 1), ("\n\nno equals\n", 3)):
        with pytest.raises(cli.ConfigError, match=f"line {line}"):
            cli.parse_config(text)
    with pytest.raises(cli.ConfigError):
        cli.parse_config("loss = l3\n")


def test_psnr_cap():
    a = np.random.RandomState(0).rand(4, 5, 3)
    assert cli.psnr(a, a) == 100.0
    assert abs(cli.psnr(a, a + 0.1) - 20.0) < 1e-9


def test_cli_exit_codes(tmp_path):
    bad = tmp_path / "bad.cfg"
    bad.write_text("lm_iters = 3\nbogus = 1\n")
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2409_12892_b200", *a], cwd=ROOT,
                                    capture_output=True, text=True)
    r = run("fit", "--dataset", str(tmp_path), "--out", str(tmp_path / "o"), "--config", str(bad))
    assert r.returncode == 2 and "line 2" in r.stderr
    r = run("fit", "--dataset", str(tmp_path / "missing"), "--out", str(tmp_path / "o"))
    assert r.returncode == 4


@pytest.fixture(scope="module")
def fitprob():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    truth, init, cams, gts = problem(seed=2, G=100, n_views=6, W=48, H=48, degree=3)  # = test_lm_outer (a descending problem)
    return dict(truth=truth, init=init, cams=cams, gts=gts, scene=init.to_device(),
                gts_d=[torch.from_numpy(g).cuda() for g in gts])


@pytest.mark.gpu
def test_gradient_matches_oracle(fitprob):
    """the ADAM gradient is the analytic -2 b of build_cache (E = sum r^2)."""
    from paper_2409_12892_b200.fit import loss_gradient
    osc = oscene(fitprob["init"])
    for i in (0, 2):
        g, e = loss_gradient(fitprob["scene"], fitprob["cams"][i], fitprob["gts_d"][i])
        oc = ocam(fitprob["cams"][i])
        rs = O.rasterize(osc, oc)
        res = O.residuals(rs["image"], fitprob["gts"][i])
        b, _ = O.build_cache(osc, oc, res, rast=rs)
        assert rel(g.cpu().numpy(), -2.0 * b) < 1e-5
        assert abs(e - float(res["energy"])) <= 1e-10 * abs(float(res["energy"]))


@pytest.mark.gpu
def test_adam_zero_lr_keeps_scene(fitprob):
    from paper_2409_12892_b200.fit import adam_fit
    zero = dict(position=0.0, rotation=0.0, log_scale=0.0, opacity=0.0, sh=0.0)
    out, hist = adam_fit(fitprob["scene"], fitprob["cams"], fitprob["gts_d"], 3, zero)
    assert torch.equal(out.x, fitprob["scene"].x) and len(hist) == 3


@pytest.mark.gpu
def test_adam_descends_and_is_deterministic(fitprob):
    from paper_2409_12892_b200.fit import adam_fit
    from paper_2409_12892_b200.lm import energy
    e0 = energy(fitprob["scene"], fitprob["cams"], fitprob["gts_d"])
    a, _ = adam_fit(fitprob["scene"], fitprob["cams"], fitprob["gts_d"], 40, seed=3)
    b, _ = adam_fit(fitprob["scene"], fitprob["cams"], fitprob["gts_d"], 40, seed=3)
    assert torch.equal(a.x, b.x)
    assert energy(a, fitprob["cams"], fitprob["gts_d"]) < e0


@pytest.mark.gpu
def test_lm_fit_monotone_and_two_stage(fitprob):
    from paper_2409_12892_b200.fit import lm_fit, two_stage_fit
    s, lam, hist = lm_fit(fitprob["scene"], fitprob["cams"], fitprob["gts_d"], 3, 8, 1, 1e-2)
    acc = [h.energy for h in hist if h.accepted]
    assert len(hist) == 4 and all(x >= y for x, y in zip(acc, acc[1:]))   # n_b = 1: non-increasing
    assert any(h.accepted for h in hist[1:]) and acc[-1] < acc[0]
    # K = 0: pure LM from the same start
    s0, h0 = two_stage_fit(fitprob["scene"], fitprob["cams"], fitprob["gts_d"], 0, 3, 8, 1, 1e-2)
    assert torch.equal(s0.x, s.x) and [h.stage for h in h0] == ["lm"] * 4
    s1, h1 = two_stage_fit(fitprob["scene"], fitprob["cams"], fitprob["gts_d"], 5, 1, 8, 1, 1e-2)
    assert [h.stage for h in h1] == ["adam"] * 5 + ["lm"] * 2


@pytest.mark.gpu
def test_cli_generate_fit_eval(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    run = lambda *a: subprocess.run([sys.executable, "-m", "paper_2409_12892_b200", *a], cwd=ROOT,
                                    capture_output=True, text=True, timeout=600)
    d, o = str(tmp_path / "data"), str(tmp_path / "out")
    r = run("generate", "--out", d, "--gaussians", "80", "--cameras", "3", "--width", "32", "--height", "32")
    assert r.returncode == 0, r.stderr
    r = run("fit", "--mode", "two-stage", "--dataset", d, "--out", o, "--stage1-iters", "3", "--lm-iters", "1")
    assert r.returncode == 0, r.stderr
    rows = open(os.path.join(o, "convergence.csv")).read().splitlines()
    assert rows[0].startswith("stage,iter") and len(rows) == 1 + 3 + 2
    assert json.load(open(os.path.join(o, "report.json")))["mode"] == "two-stage"
    r = run("eval", "--scene", os.path.join(d, "scene.json"), "--dataset", d)
    assert r.returncode == 0, r.stderr
    assert json.loads(r.stdout)["mean"]["psnr"] == 100.0      # truth vs its own images
