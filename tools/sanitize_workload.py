"""compute-sanitizer workload (tools/sanitize.sh): one small cache built all
in HBM and one with half its records offloaded, every product mode, diag,
the device order export, a PCG solve on the padded gaussian-major p and one
LM direction -- synchronised after each step so a report names the step."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

from helpers import problem  # noqa: E402
from paper_2409_12892_b200.engine import CacheSet  # noqa: E402
from paper_2409_12892_b200.solver import BatchSchedule, lm_direction, pcg_run  # noqa: E402


def step(name):
    torch.cuda.synchronize()
    print(name, "ok", flush=True)


G = int(sys.argv[1]) if len(sys.argv) > 1 else 60
truth, init, cams, gts = problem(seed=0, G=G, n_views=3, W=32, H=28, degree=3)
scene = init.to_device()
gts_d = [torch.from_numpy(g).cuda() for g in gts]
for off in (None, 0.5):
    cs = CacheSet(scene, cams, gts_d, offload=off)
    step(f"build offload={off} E={cs.E} R={cs.R} chunks={cs.n_chunks} host={cs.offloaded_entries}")
    b = cs.rhs()
    step("rhs")
    M = cs.diag()
    step("diag")
    p = torch.randn(scene.param_count, device="cuda")
    cs.pair_forward(p)
    cs.apply_j_raw(weighted=False)
    step("apply_j")
    out = torch.empty_like(p)
    cs.apply_jt_raw(cs.u, out)
    step("apply_jt")
    cs.jtwj(p, out, 1e-4, M)
    step("jtwj")
    for v in range(len(cams)):
        cs.export_view(v)
    step("export")
    pcg_run(cs, b, M, 1e-4, 3)
    step("pcg")
    del cs
lm_direction(scene, cams, gts_d, BatchSchedule(2), 1e-4, 3)
step("lm_direction")
