"""Debug harness: one small CacheSet and each product mode, synchronised."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import torch  # noqa: E402

from helpers import problem  # noqa: E402
from paper_2409_12892_b200.engine import CacheSet  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 60
truth, init, cams, gts = problem(seed=0, G=G, n_views=3, W=32, H=28, degree=3)
scene = init.to_device()
cs = CacheSet(scene, cams, [torch.from_numpy(g).cuda() for g in gts])
torch.cuda.synchronize()
print("built", cs.E, cs.R, cs.n_chunks, flush=True)
print("perm", cs.chunk_perm[:64].cpu().tolist(), flush=True)
b = cs.rhs()
torch.cuda.synchronize()
print("rhs ok", flush=True)
p = torch.randn(scene.param_count, device="cuda")
cs.pair_forward(p)
torch.cuda.synchronize()
print("fwd ok", flush=True)
cs.apply_j_raw(weighted=False)
torch.cuda.synchronize()
print("apply_j ok", flush=True)
out = torch.empty_like(p)
cs.jtwj(p, out)
torch.cuda.synchronize()
print("jtwj ok", flush=True)
M = cs.diag()
torch.cuda.synchronize()
print("diag ok", flush=True)
from paper_2409_12892_b200.solver import pcg_run  # noqa: E402
x = pcg_run(cs, b, M, 1e-4, 3)
torch.cuda.synchronize()
print("pcg ok", flush=True)
