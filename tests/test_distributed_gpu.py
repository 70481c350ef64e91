"""Multi-rank LM direction on one GPU: two processes (gloo, both on cuda:0)
run the REAL lm_direction / Combiner path -- subset j on rank j mod 2, one
packed all_reduce of [num; den; energy; accepted] -- and must
reproduce the single-process direction:

  * Delta of 2 ranks == Delta of 1 rank to <= 1e-12 relative (only the fp64
    summation order of the Eq. 7 sums differs), identical bits on both ranks;
  * the reported energy is the global sum over all subsets on every rank;
  * a subset rejected by NonSPDError on one rank drops out of the combine
    exactly as in the single-process run (accepted count 3 of 4 everywhere).

The NCCL path differs only in the backend of the same torch.distributed
all_reduce call.
"""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

N_SUBSETS = 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _problem():
    from helpers import problem
    truth, init, cams, gts = problem(seed=2, G=100, n_views=8, W=40, H=40, degree=3)
    return init, cams, gts


def _patch_reject(reject_call):
    """Make the reject_call-th pcg_run of this process raise NonSPDError."""
    from paper_2409_12892_b200 import solver
    from paper_2409_12892_b200.errors import NonSPDError
    orig = solver.pcg_run
    calls = [0]

    def pcg_run(*a, **k):
        calls[0] += 1
        if calls[0] == reject_call:
            raise NonSPDError("injected p^T g <= 0")
        return orig(*a, **k)
    solver.pcg_run = pcg_run

    def restore():
        solver.pcg_run = orig
    return restore


def _run(rank, world, reject_call=None):
    from paper_2409_12892_b200.solver import BatchSchedule, lm_direction
    restore = _patch_reject(reject_call) if reject_call else None
    try:
        init, cams, gts = _problem()
        scene = init.to_device()
        rep = lm_direction(scene, cams, [torch.from_numpy(g).cuda() for g in gts], BatchSchedule(N_SUBSETS), 1e-4,
                           6, rank=rank, world_size=world)
    finally:
        if restore:
            restore()
    return rep.delta.cpu().numpy(), rep.energy, rep.batches_accepted


def _worker(rank, world, port, outdir, reject_call):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    d, e, a = _run(rank, world, reject_call if rank == 1 else None)
    np.savez(os.path.join(outdir, f"r{rank}.npz"), delta=d, energy=e, accepted=a)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")


@pytest.mark.parametrize("reject", [False, True], ids=["all_accepted", "rank1_subset_rejected"])
def test_two_ranks_equal_one_rank(reject):
    import torch.multiprocessing as mp
    # single process: subsets 0,1,2,3 in order; the rejected one is subset 3
    # (rank 1's second subset in the 2-rank run)
    d1, e1, a1 = _run(0, 1, 4 if reject else None)
    with tempfile.TemporaryDirectory() as td:
        mp.spawn(_worker, args=(2, _free_port(), td, 2 if reject else None), nprocs=2, join=True)
        outs = [np.load(os.path.join(td, f"r{r}.npz")) for r in range(2)]
    assert a1 == (3 if reject else 4)
    for o in outs:
        assert int(o["accepted"]) == a1
        assert abs(float(o["energy"]) - e1) <= 1e-12 * e1
        err = np.linalg.norm(o["delta"].astype(np.float64) - d1) / np.linalg.norm(d1)
        assert err <= 1e-12, err
    assert np.array_equal(outs[0]["delta"], outs[1]["delta"])      # identical bits on both ranks
    if reject:
        # the rejected subset really changed the direction
        d_all, _, _ = _run(0, 1, None)
        assert not np.array_equal(d_all, d1)
