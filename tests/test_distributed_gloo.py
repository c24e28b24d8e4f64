"""Multi-rank CS ensemble plumbing on CPU (gloo, world_size 2).

The GPU kernels cannot run here, so these tests drive the host-side sharding and
the single exchange step of paper_2605_29284_b200.distributed with synthetic
per-chunk partial moments, and check that (a) every chunk is owned by exactly one
rank, (b) the all-gathered partials arrive in chunk order, and (c) the combined
moments are bitwise identical to the single-process combine — the property that
makes ensemble SE independent of the GPU count.
"""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_29284_b200.distributed import exchange_partials, rank_chunks
from paper_2605_29284_b200.simulate import combine_chunks, ensemble_chunks

SHAPE = (5, 7)


def _partials(n_draws, seed=0):
    """Deterministic fake per-chunk (s1, s2) moments, one pair per chunk."""
    g = torch.Generator().manual_seed(seed)
    out = []
    for j0, j1 in ensemble_chunks(n_draws):
        s1 = torch.randn(SHAPE, generator=g, dtype=torch.float64) * (j1 - j0)
        s2 = torch.rand(SHAPE, generator=g, dtype=torch.float64) * (j1 - j0)
        out.append((s1, s2))
    return out


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_draws, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        allp = _partials(n_draws)
        mine = [allp[k] for k in rank_chunks(len(allp), rank, world)]
        parts = exchange_partials(mine, len(allp), SHAPE, device="cpu")
        s1, s2 = combine_chunks(parts)
        q.put((rank, s1.numpy().tobytes(), s2.numpy().tobytes(), len(mine)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_draws", [(2, 1024), (2, 7), (2, 3)])
def test_sharded_combine_matches_single_process(world, n_draws):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_draws, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref1, ref2 = combine_chunks(_partials(n_draws))
    owned = 0
    for rank, b1, b2, nmine in res:
        assert b1 == ref1.numpy().tobytes(), rank
        assert b2 == ref2.numpy().tobytes(), rank
        owned += nmine
    assert owned == len(ensemble_chunks(n_draws))


@pytest.mark.parametrize("n_chunks", [1, 3, 8, 13])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rank_chunks_partition(n_chunks, world):
    seen = []
    for r in range(world):
        seen += rank_chunks(n_chunks, r, world)
    assert seen == list(range(n_chunks))
