"""CPU, world_size 2 over gloo: subset sharding + the single packed
all_reduce of [num; den] reproduce the single-process Eq. 7 combine.

Per-subset directions and diagonals come from the oracle; each rank keeps
only its shard (subset j -> rank j mod W), accumulates num/den locally and
calls solver.allreduce_sum_ exactly as lm_direction does on NCCL.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2409_12892_b200.solver import BatchSchedule, allreduce_sum_


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _subset_data(n_subsets, n):
    rng = np.random.default_rng(42)
    deltas = [rng.standard_normal(n) for _ in range(n_subsets)]
    Ms = [rng.random(n) * (rng.random(n) > 0.2) for _ in range(n_subsets)]
    return deltas, Ms


def _worker(rank, world, port, n_views, n_subsets, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    deltas, Ms = _subset_data(n_subsets, n)
    sched = BatchSchedule(n_subsets)
    buf = torch.zeros(2 * n, dtype=torch.float64)
    owned = []
    for j, views in sched.shard(n_views, rank, world):
        owned.append(j)
        buf[:n] += torch.from_numpy(Ms[j] * deltas[j])
        buf[n:] += torch.from_numpy(Ms[j])
    allreduce_sum_(buf)
    delta = (buf[:n] / torch.clamp(buf[n:], min=1e-12)).numpy()
    out[rank] = (owned, delta)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_combine_equals_single_process(world):
    n_views, n_subsets, n = 40, 8, 300
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_views, n_subsets, n, out), nprocs=world, join=True)
    deltas, Ms = _subset_data(n_subsets, n)
    ref = O.combine(deltas, Ms)
    owned = sorted(j for r in range(world) for j in out[r][0])
    assert owned == list(range(n_subsets))                  # every subset exactly once
    assert set(out[0][0]).isdisjoint(out[1][0])
    for r in range(world):
        # only the summation order differs from the single-process combine
        np.testing.assert_allclose(out[r][1], ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    np.testing.assert_array_equal(out[0][1], out[1][1])      # identical bits on all ranks


def test_shard_assignment():
    s = BatchSchedule(8)
    assert [j for j, _ in s.shard(200, 1, 4)] == [1, 5]
    assert s.shard(200, 0, 1)[0][1][:3] == [0, 8, 16]
