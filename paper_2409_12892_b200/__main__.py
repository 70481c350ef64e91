"""Command-line driver (SPEC cli module; SPEC-only in the
reference): generate / fit (adam | lm | two-stage) / eval / render.

    python -m paper_2409_12892_b200 generate --out DIR [--gaussians N --cameras V --width W --height H ...]
    python -m paper_2409_12892_b200 fit --mode lm --dataset DIR --out DIR [--config FILE] [flags]
    python -m paper_2409_12892_b200 eval --scene FILE --dataset DIR
    python -m paper_2409_12892_b200 render --scene FILE --cameras FILE --index I --out IMAGE

Exit codes: 0 success, 2 config error, 3 solver failure, 4 IO error.
The config file is `key = value` lines (`#` comments); errors name the line.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
import time

EXIT_OK, EXIT_CONFIG, EXIT_SOLVER, EXIT_IO = 0, 2, 3, 4

# config keys (SPEC External Interfaces) -> (type, default)
CONFIG_KEYS = {
    "lambda1": (float, 0.8), "lambda2": (float, 0.2), "loss": (str, "l1ssim"), "lambda_reg": (float, 1e-4),
    "pcg_iters": (int, 8), "lm_iters": (int, 5), "num_batches": (int, 1), "ls_fraction": (float, 0.3),
    "stage1_iters": (int, 200), "seed": (int, 0), "lr_position": (float, 1.6e-4), "lr_rotation": (float, 1e-3),
    "lr_log_scale": (float, 5e-3), "lr_opacity": (float, 5e-2), "lr_sh": (float, 2.5e-3),
}


class ConfigError(ValueError):
    pass


def parse_config(text: str) -> dict:
    """`key = value` lines -> typed dict over CONFIG_KEYS defaults; raises
    ConfigError naming the offending line."""
    cfg = {k: d for k, (_, d) in CONFIG_KEYS.items()}
    for n, raw in enumerate(text.splitlines(), 1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"line {n}: expected 'key = value', got {raw!r}")
        k, v = (s.strip() for s in line.split("=", 1))
        if k not in CONFIG_KEYS:
            raise ConfigError(f"line {n}: unknown key {k!r}")
        typ = CONFIG_KEYS[k][0]
        try:
            cfg[k] = typ(v)
        except ValueError:
            raise ConfigError(f"line {n}: {k} expects {typ.__name__}, got {v!r}") from None
    if cfg["loss"] not in ("l1ssim", "l2"):
        raise ConfigError(f"loss must be l1ssim or l2, got {cfg['loss']!r}")
    return cfg


def psnr(img, gt) -> float:
    """PSNR in dB against a [0, 1] reference, capped at 100 dB."""
    import numpy as np
    mse = float(np.mean((np.asarray(img, float) - np.asarray(gt, float)) ** 2))
    return 100.0 if mse <= 1e-10 else min(100.0, 10.0 * np.log10(1.0 / mse))


def _dataset(path, device, scene_file=None):
    from . import imageio
    from .scene import cameras_from_json, scene_from_json
    with open(os.path.join(path, "cameras.json")) as f:
        cams = cameras_from_json(f.read())
    gts = [imageio.read_pfm(os.path.join(path, f"gt_{i:03d}.pfm"), device=device) for i in range(len(cams))]
    scene = None
    sf = scene_file or os.path.join(path, "init.json")
    if os.path.exists(sf):
        with open(sf) as f:
            scene = scene_from_json(f.read(), device)
    return scene, cams, gts


def _loss(cfg):
    from .engine import LossConfig
    return LossConfig(cfg["lambda1"], cfg["lambda2"], cfg["loss"])


def cmd_generate(a) -> int:
    import numpy as np
    from . import imageio
    from . import synthetic as S
    from .rasterizer import render
    from .scene import cameras_to_json, scene_to_json
    os.makedirs(a.out, exist_ok=True)
    truth = S.make_synthetic_scene(a.seed, a.gaussians, a.sh_degree)
    init = S.perturb(truth, a.seed + 1, a.perturb)
    cams = S.make_camera_ring(a.cameras, a.width, a.height)
    t, i0 = truth.to_device(), init.to_device()
    with open(os.path.join(a.out, "scene.json"), "w") as f:
        f.write(scene_to_json(t))
    with open(os.path.join(a.out, "init.json"), "w") as f:
        f.write(scene_to_json(i0))
    with open(os.path.join(a.out, "cameras.json"), "w") as f:
        f.write(cameras_to_json(cams))
    for k, c in enumerate(cams):
        img = render(t, c, traversals=False).image
        imageio.write_pfm(os.path.join(a.out, f"gt_{k:03d}.pfm"), img)
        imageio.write_png(os.path.join(a.out, f"gt_{k:03d}.png"), np.asarray(img.cpu()))
    with open(os.path.join(a.out, "manifest.json"), "w") as f:
        json.dump({"seed": a.seed, "gaussians": a.gaussians, "cameras": a.cameras, "width": a.width,
                   "height": a.height, "sh_degree": a.sh_degree, "perturb": a.perturb}, f, indent=1)
    return EXIT_OK


def cmd_fit(a, cfg) -> int:
    import torch
    from . import fit as F
    from .scene import scene_to_json
    dev = torch.device("cuda")
    scene, cams, gts = _dataset(a.dataset, dev, a.scene)
    if scene is None:
        raise FileNotFoundError("no init.json in the dataset and no --scene given")
    loss = _loss(cfg)
    lr = {c: cfg["lr_" + c] for c in ("position", "rotation", "log_scale", "opacity", "sh")}
    t0 = time.perf_counter()
    if a.mode == "adam":
        out, hist = F.adam_fit(scene, cams, gts, cfg["stage1_iters"], lr, seed=cfg["seed"], loss=loss)
    elif a.mode == "lm":
        out, _, hist = F.lm_fit(scene, cams, gts, cfg["lm_iters"], cfg["pcg_iters"], cfg["num_batches"],
                                cfg["lambda_reg"], cfg["ls_fraction"], loss=loss)
    else:
        out, hist = F.two_stage_fit(scene, cams, gts, cfg["stage1_iters"], cfg["lm_iters"], cfg["pcg_iters"],
                                    cfg["num_batches"], cfg["lambda_reg"], lr, cfg["seed"], loss=loss)
    wall = time.perf_counter() - t0
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "scene.json"), "w") as f:
        f.write(scene_to_json(out))
    with open(os.path.join(a.out, "convergence.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["stage", "iter", "time_s", "energy", "accepted", "lambda_reg", "gamma"])
        for r in hist:
            w.writerow([r.stage, r.iteration, f"{r.time_s:.6f}", repr(r.energy), int(r.accepted), repr(r.lam),
                        repr(r.gamma)])
    from .lm import energy
    e = energy(out, cams, gts, loss=loss)
    with open(os.path.join(a.out, "report.json"), "w") as f:
        json.dump({"mode": a.mode, "config": cfg, "final": {"energy": e}, "wall_s": wall,
                   "iterations": len(hist)}, f, indent=1)
    print(json.dumps({"mode": a.mode, "energy": e, "iterations": len(hist), "wall_s": round(wall, 3)}))
    return EXIT_OK


def cmd_eval(a) -> int:
    import torch
    from .lm import view_energy
    from .rasterizer import render
    dev = torch.device("cuda")
    scene, cams, gts = _dataset(a.dataset, dev, a.scene)
    per = []
    for c, g in zip(cams, gts):
        img = render(scene, c, traversals=False).image
        per.append({"psnr": psnr(img.cpu().numpy(), g.cpu().numpy()), "energy": float(view_energy(scene, c, g))})
    agg = {k: sum(p[k] for p in per) / len(per) for k in ("psnr", "energy")}
    print(json.dumps({"per_image": per, "mean": agg}))
    return EXIT_OK


def cmd_render(a) -> int:
    import torch
    from . import imageio
    from .rasterizer import render
    from .scene import cameras_from_json, scene_from_json
    dev = torch.device("cuda")
    with open(a.scene) as f:
        scene = scene_from_json(f.read(), dev)
    with open(a.cameras) as f:
        cams = cameras_from_json(f.read())
    img = render(scene, cams[a.index], traversals=False).image
    if a.out.endswith(".png"):
        imageio.write_png(a.out, img.cpu().numpy())
    else:
        imageio.write_pfm(a.out, img)
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2409_12892_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("generate")
    g.add_argument("--out", required=True)
    g.add_argument("--gaussians", type=int, default=2000)
    g.add_argument("--cameras", type=int, default=8)
    g.add_argument("--width", type=int, default=64)
    g.add_argument("--height", type=int, default=64)
    g.add_argument("--sh-degree", type=int, default=3)
    g.add_argument("--perturb", type=float, default=0.1)
    g.add_argument("--seed", type=int, default=0)
    f = sub.add_parser("fit")
    f.add_argument("--mode", choices=("adam", "lm", "two-stage"), default="lm")
    f.add_argument("--dataset", required=True)
    f.add_argument("--out", required=True)
    f.add_argument("--scene", default=None, help="starting scene (default: DATASET/init.json)")
    f.add_argument("--config", default=None)
    for k in ("stage1_iters", "lm_iters", "pcg_iters", "num_batches", "seed"):
        f.add_argument("--" + k.replace("_", "-"), type=int, default=None)
    f.add_argument("--lambda-reg", type=float, default=None)
    f.add_argument("--loss", choices=("l1ssim", "l2"), default=None)
    e = sub.add_parser("eval")
    e.add_argument("--scene", required=True)
    e.add_argument("--dataset", required=True)
    r = sub.add_parser("render")
    r.add_argument("--scene", required=True)
    r.add_argument("--cameras", required=True)
    r.add_argument("--index", type=int, default=0)
    r.add_argument("--out", required=True)
    a = ap.parse_args(argv)
    try:
        cfg = None
        if a.cmd == "fit":
            text = ""
            if a.config:
                with open(a.config) as fh:
                    text = fh.read()
            cfg = parse_config(text)
            for k in ("stage1_iters", "lm_iters", "pcg_iters", "num_batches", "seed", "lambda_reg", "loss"):
                if getattr(a, k) is not None:
                    cfg[k] = getattr(a, k)
        from .errors import NonSPDError
        try:
            return {"generate": lambda: cmd_generate(a), "fit": lambda: cmd_fit(a, cfg),
                    "eval": lambda: cmd_eval(a), "render": lambda: cmd_render(a)}[a.cmd]()
        except NonSPDError as ex:
            print(f"solver failure: {ex}", file=sys.stderr)
            return EXIT_SOLVER
    except ConfigError as ex:
        print(f"config error: {ex}", file=sys.stderr)
        return EXIT_CONFIG
    except OSError as ex:
        print(f"io error: {ex}", file=sys.stderr)
        return EXIT_IO


if __name__ == "__main__":
    sys.exit(main())
