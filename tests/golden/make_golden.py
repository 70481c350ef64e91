"""Generate golden fixtures from the REFERENCE implementation (run here, where
/root/reference is mounted):  python tests/golden/make_golden.py

Each case stores the inputs (scene matrix, cameras, gt images) and the
reference's outputs for the hot path: render traversals, residual maps, b,
the gaussian-order permutation, apply_j / apply_jt / diag_jtj on fixed
random vectors.  The oracle is pinned against these in test_oracle_golden.py
(CPU) and the CUDA path against the oracle in test_gpu_parity.py.
"""
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from splatlm import jacobian as RJ  # noqa: E402
from splatlm import rasterizer as RR  # noqa: E402
from splatlm import residuals as RE  # noqa: E402
from splatlm import scene as RS  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = {"g20_l3_2v": dict(seed=3, G=20, views=2, res=(24, 20), degree=3),
         "g40_l1_3v": dict(seed=7, G=40, views=3, res=(20, 22), degree=1)}


def make(name, seed, G, views, res, degree):
    truth, cams, imgs = RS.make_synthetic_dataset(seed, G, views, res, sh_degree=degree)
    init = RS.perturb(truth, seed + 1, 0.1)
    x = RS.flatten(init).values
    out = {"x_am": x, "degree": degree, "background": init.background,
           "cam_R": np.stack([c.rotation for c in cams]), "cam_t": np.stack([c.translation for c in cams]),
           "cam_f": np.array([[c.fx, c.fy, c.cx, c.cy, c.width, c.height] for c in cams])}
    rng = np.random.default_rng(seed + 100)
    p = rng.standard_normal(init.param_count)
    out["p_am"] = p
    pv = RS.ParamVector(p, RS.Layout.ATTRIBUTE_MAJOR, init.num_gaussians, init.params_per_gaussian)
    for v, (c, gt) in enumerate(zip(cams, imgs)):
        rr = RR.render(init, c)
        tr = rr.traversals
        bund = RE.compute_residuals(rr.image.rgb, gt)
        b, cache = RJ.build_cache(init, c, bund, render_result=rr)
        gc = RJ.sort_cache_by_gaussians(cache)
        u = rng.standard_normal(c.num_pixels * 3)
        out.update({f"v{v}_gt": gt, f"v{v}_image": rr.image.rgb, f"v{v}_offsets": tr.offsets,
                    f"v{v}_gid": tr.gaussian_ids, f"v{v}_alpha": tr.alphas, f"v{v}_T": tr.transmittances,
                    f"v{v}_valid": rr.splats.valid, f"v{v}_grad_r_sq": bund.grad_r_sq,
                    f"v{v}_color_grad": bund.color_grad, f"v{v}_energy": bund.energy, f"v{v}_b": b.values,
                    f"v{v}_dc_dalpha": cache.dc_dalpha, f"v{v}_source_index": gc.source_index,
                    f"v{v}_goffsets": gc.offsets, f"v{v}_u": u,
                    f"v{v}_apply_j": RJ.apply_j(RS.sort_x(pv), init, gc),
                    f"v{v}_apply_jt": RJ.apply_jt(u, init, gc).values,
                    f"v{v}_diag": RJ.diag_jtj(init, gc).values})
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)


if __name__ == "__main__":
    for k, kw in CASES.items():
        make(k, **kw)
        print("wrote", k)
