"""Multi-rank CS ensemble plumbing on CPU (gloo, world_size 2 and 4).

The GPU kernels cannot run here, so these tests drive the host-side sharding and the single
exchange step of paper_2605_29284_b200.distributed with synthetic per-realization errors e_j,
converted to the library's fixed-point digits by the host restatement (tests/fx_ref.py):
(a) the rank blocks cover every realization exactly once, (b) the all-reduced int64 moments
are bitwise identical for 1, 2 and 4 ranks and equal the exact sums of the terms -- the
property that makes ensemble mean / SE independent of the GPU count.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from fx_ref import moments, value
from paper_2605_29284_b200.distributed import allreduce_moments, rank_range

SHAPE = (3, 4)
SIGMA2 = 2.7


def _errors(j):
    """Deterministic fake e_j for realization j (mixed magnitudes and signs)."""
    g = np.random.default_rng(1000 + j)
    return g.normal(size=SHAPE) * np.exp(g.uniform(-8, 3, size=SHAPE))


def _local_acc(n_draws, rank, world):
    j0, j1 = rank_range(n_draws, rank, world)
    acc = np.zeros((6,) + SHAPE, dtype=np.int64)
    for j in range(j0, j1):
        acc += moments(_errors(j)[None], SIGMA2)
    return torch.from_numpy(acc), (j0, j1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_draws, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        acc, rng = _local_acc(n_draws, rank, world)
        allreduce_moments(acc)
        q.put((rank, acc.numpy().tobytes(), rng))
    finally:
        dist.destroy_process_group()


def _run(world, n_draws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_draws, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world,n_draws", [(2, 37), (4, 37), (2, 3), (4, 5)])
def test_sharded_moments_bitwise_equal_single_process(world, n_draws):
    single, _ = _local_acc(n_draws, 0, 1)
    res = _run(world, n_draws)
    covered = []
    for rank, b, rng in res:
        assert b == single.numpy().tobytes(), rank
        covered += list(range(*rng))
    assert sorted(covered) == list(range(n_draws))


def test_fixed_point_sums_are_exact():
    """Digit sums equal the exact (Python-int) sums of trunc(v 2^64), and reconstruct the
    float sums to ~1e-19 relative."""
    from fx_ref import digits, fx_scale
    n_draws = 23
    acc, _ = _local_acc(n_draws, 0, 1)
    acc = acc.numpy()
    s = fx_scale(SIGMA2)
    for idx in np.ndindex(SHAPE):
        exact1 = sum(value(*digits(float(_errors(j)[idx] / s))) for j in range(n_draws))
        exact2 = sum(value(*digits(float((_errors(j)[idx] / s) ** 2))) for j in range(n_draws))
        assert value(*acc[0:3][(slice(None),) + idx]) == exact1
        assert value(*acc[3:6][(slice(None),) + idx]) == exact2
        ref = sum(_errors(j)[idx] for j in range(n_draws))
        assert abs(exact1 / 2.0 ** 64 * s - ref) <= 1e-15 * max(1.0, abs(ref))


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_rank_ranges_partition(world):
    seen = []
    for r in range(world):
        seen += list(range(*rank_range(1024, r, world)))
    assert seen == list(range(1024))
