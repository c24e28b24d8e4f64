"""Conditional-simulation ensembles over torch.distributed ranks (one process per GPU).

Realization j depends only on (seed, j) (simulate.py:60-62, 186), so rank r of N runs the
contiguous block [r R / N, (r + 1) R / N).  Rank 0 builds the fit and the setup once; the
other ranks receive them over NCCL (NVLink) instead of repeating the n x n Cholesky:
``broadcast_fit`` sends the fit's device arrays in place (factor, inverse factor, covariates,
coefficients) and ``broadcast_setup`` the setup as one device blob.  Each rank accumulates
exact fixed-point moments (simulate.py docs); the ONLY data-path collective is one int64
all-reduce (sum) of the 6 x m2 x m1 accumulator.  Integer sums are associative, so mean and
SE are bitwise identical for any number of ranks and any split.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import _device as D
from . import _native as N
from .errors import DomainError
from .simulate import Ensemble, _prepare, accumulate, finalize, new_accumulator, shard_ranges

__all__ = ["rank_range", "allreduce_moments", "broadcast_fit", "broadcast_setup", "generate_ensemble_sharded"]


def rank_range(n_draws: int, rank: int, world: int):
    """Realizations [j0, j1) of ``rank``: contiguous, sizes differ by at most one."""
    return shard_ranges(n_draws, world)[rank]


def allreduce_moments(acc, group=None):
    """Sum the int64 moment accumulators of all ranks in place (exact; NCCL or gloo)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(acc, op=dist.ReduceOp.SUM, group=group)
    return acc


class _CudaBuffer:
    """Zero-copy view of a library-owned device array (``__cuda_array_interface__``)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _view(ptr, nbytes):
    return torch.as_tensor(_CudaBuffer(ptr, nbytes), device="cuda")


def broadcast_fit(krig, group=None, src: int = 0):
    """The fit of rank ``src`` on every rank: its device arrays are broadcast in place into a
    fit shell (no re-factorisation).  Ranks other than ``src`` may pass None."""
    from .exact import KrigingFit, _FitHandle, as_device_fit
    rank = dist.get_rank(group)
    meta = [None]
    if rank == src:
        f = as_device_fit(krig)
        f.prepare_refit()   # the inverse factor travels too
        meta = [(f.model, f.obs_locs, f.X, np.asarray(f.beta_hat), np.asarray(f.c))]
    dist.broadcast_object_list(meta, src=src, group=group)
    model, obs, X, beta, c = meta[0]
    n, p = X.shape
    if rank == src:
        h = f.handle
    else:
        hp = N.C.c_void_p()
        N.call("rk_fit_shell", N.C.byref(model.native()), n, p, 1, N.C.byref(hp))
        f = KrigingFit(model, obs, X, beta, c, _FitHandle(hp))
        h = hp
    ptrs = (N.C.c_void_p * 7)()
    sizes = (N.C.c_int64 * 7)()
    N.call("rk_fit_fields", h, N.C.byref(ptrs), N.C.byref(sizes))
    for i in range(7):
        if sizes[i]:
            dist.broadcast(_view(ptrs[i], sizes[i]), src=src, group=group)
    gram = torch.zeros(p * p + p, dtype=torch.float64)
    piv = np.zeros(p, dtype=np.int32)
    lu = np.zeros(p * p)
    if rank == src:
        N.call("rk_fit_get_gram", h, N.ptr(lu), N.ptr(piv))
        gram[: p * p] = torch.from_numpy(lu)
        gram[p * p:] = torch.from_numpy(piv.astype(np.float64))
    gram = gram.to("cuda")
    dist.broadcast(gram, src=src, group=group)
    if rank != src:
        g = gram.cpu().numpy()
        lu = np.ascontiguousarray(g[: p * p])
        piv = np.ascontiguousarray(g[p * p:].astype(np.int32))
        N.call("rk_fit_set_gram", h, N.ptr(lu), N.ptr(piv))
    torch.cuda.synchronize()
    return f


def broadcast_setup(setup, group=None, src: int = 0):
    """The setup of rank ``src`` (incl. its simulation embedding) on every rank, as one device
    blob broadcast over NCCL.  Ranks other than ``src`` may pass None."""
    from .rapid import RapidSetup, _Handle
    from .simulate import embedding_dims
    rank = dist.get_rank(group)
    meta = [None]
    if rank == src:
        embedding_dims(setup.model, setup)
        nb = N.C.c_int64()
        N.call("rk_setup_blob_bytes", setup.handle, N.C.byref(nb))
        meta = [(setup.model, setup.grid, setup.L, setup.ridge_applied, int(nb.value))]
    dist.broadcast_object_list(meta, src=src, group=group)
    model, grid, L, ridge, nbytes = meta[0]
    blob = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    if rank == src:
        N.call("rk_setup_export", setup.handle, N.ptr(blob), N.stream_ptr())
    dist.broadcast(blob, src=src, group=group)
    if rank == src:
        return setup
    torch.cuda.synchronize()
    h = N.C.c_void_p()
    N.call("rk_setup_import", N.ptr(blob), nbytes, N.C.byref(h))
    return RapidSetup(model, grid, L, _Handle(h), ridge)


def generate_ensemble_sharded(krig, setup, n_draws: int, seed: int, grid_covariates=None, *,
                              group=None, batch: int = 64, host: bool = False):
    """Ensemble mean / SE over all ranks (draws are not materialised): rank r runs its
    contiguous block of realizations, then one int64 all-reduce combines the moments."""
    if n_draws < 2:
        raise DomainError(f"need at least 2 draws, got {n_draws}")
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    f, xd, dp = _prepare(krig, setup, grid_covariates)
    j0, j1 = rank_range(n_draws, rank, world)
    acc = accumulate(setup, f, seed, j0, j1, xd, dp, new_accumulator(setup), None, batch)
    allreduce_moments(acc, group)
    mean, se = finalize(dp, acc, n_draws, f.model.sigma2)
    if host:
        return Ensemble(None, int(seed), int(n_draws), mean.cpu().numpy(), se.cpu().numpy())
    return Ensemble(None, int(seed), int(n_draws), mean, se)
