"""Conditional-simulation ensembles sharded over torch.distributed ranks (one GPU each).

Realization j depends only on (seed, j) (simulate.py:60-62, 186), so the fixed
realization chunks of simulate.ensemble_chunks are split into contiguous blocks
per rank; every rank builds the (immutable) setup and fit itself from the same
inputs, so no setup broadcast is needed.  The only exchange is ONE all-gather of
the per-chunk partial moments (2 x m2 x m1 fp64 per chunk) over NCCL; every rank
then sums the chunks in chunk order, which makes mean/SE bitwise identical for
1, 2, 4 or 8 GPUs.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import _device as D
from .simulate import (Ensemble, _prepare, accumulate_chunk, combine_chunks, ensemble_chunks,
                       finalize)
from .errors import DomainError

__all__ = ["rank_chunks", "exchange_partials", "generate_ensemble_sharded"]


def rank_chunks(n_chunks: int, rank: int, world: int):
    """Contiguous block of chunk indices owned by ``rank``."""
    return list(range((rank * n_chunks) // world, ((rank + 1) * n_chunks) // world))


def exchange_partials(local, n_chunks: int, shape, group=None, device=None):
    """All-gather per-chunk (s1, s2) partials; returns the full list in chunk order.

    ``local`` holds this rank's partials (in its chunk order).  Works with NCCL
    (CUDA tensors) and gloo (CPU tensors)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        return list(local)
    cmax = -(-n_chunks // world)
    dev = device if device is not None else (local[0][0].device if local else "cpu")
    buf = torch.zeros((cmax, 2) + tuple(shape), dtype=torch.float64, device=dev)
    for k, (a, b) in enumerate(local):
        buf[k, 0] = a
        buf[k, 1] = b
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf, group=group)
    out = []
    for r in range(world):
        for k in range(len(rank_chunks(n_chunks, r, world))):
            out.append((gathered[r][k, 0], gathered[r][k, 1]))
    return out


def generate_ensemble_sharded(krig, setup, n_draws: int, seed: int, grid_covariates=None, *,
                              group=None, batch: int = 32, host: bool = False):
    """Ensemble mean / SE over all ranks (draws are not materialised)."""
    if n_draws < 2:
        raise DomainError(f"need at least 2 draws, got {n_draws}")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    chunks = ensemble_chunks(n_draws)
    f, xd, dp = _prepare(krig, setup, grid_covariates)
    local = [accumulate_chunk(setup, f, seed, *chunks[k], xd, dp, None, batch)
             for k in rank_chunks(len(chunks), rank, world)]
    m1, m2 = setup.grid.interior_dims
    parts = exchange_partials(local, len(chunks), (m2, m1), group, device=dp.device)
    s1, s2 = combine_chunks(parts)
    mean, se = finalize(dp, s1, s2, n_draws)
    if host:
        return Ensemble(None, int(seed), int(n_draws), mean.cpu().numpy(), se.cpu().numpy())
    return Ensemble(None, int(seed), int(n_draws), mean, se)
