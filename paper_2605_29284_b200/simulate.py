"""Conditional-simulation ensembles on the B200.

Interface of reference simulate.py:52-192: ``draw_seed``, ``sim_unconditional_grid``,
``sim_obs_local``, ``conditional_draw``, ``generate_ensemble`` and ``Ensemble``,
with the same Philox4x64-10 streams (key = (seed, stream), pre-incremented
counter) and inverse-CDF normals, so draws match the reference to roundoff.

``generate_ensemble`` runs realizations in batches through one fused device
pipeline (rk_ensemble_accumulate): Philox+normal+sqrt(lambda) fused into the
row IFFT pass, column IFFT, local observation simulation, batched GLS refit
(FP64 tensor cores), the rapid predict passes with the draw epilogue, and
per-pixel moments accumulated as exact fixed-point integers.  Integer sums do
not depend on order, so the ensemble is bitwise identical however the
realizations are batched or split over GPUs -- within one process
(``devices="all"``, setup and fit copied peer to peer) or over
torch.distributed ranks (distributed.py, one int64 all-reduce).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .errors import DomainError
from .exact import as_device_fit, refit_coefficients
from .rapid import GRID_SETUPS, _fixed_inputs, predict_rapid

__all__ = ["Ensemble", "RNG_ALGORITHM", "draw_seed", "std_normals", "sim_unconditional_grid", "sim_obs_local",
           "conditional_draw", "generate_ensemble", "shard_ranges", "new_accumulator", "accumulate",
           "combine", "finalize"]

RNG_ALGORITHM = "philox4x64-10"
_M64 = (1 << 64) - 1


def _splitmix64(v: int) -> int:
    z = (v + 0x9E3779B97F4A7C15) & _M64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _M64
    return (z ^ (z >> 31)) & _M64


def draw_seed(seed: int, j: int) -> int:
    """seed XOR splitmix64(j) (simulate.py:52-62)."""
    return (int(seed) ^ _splitmix64(int(j))) & _M64


@dataclass(frozen=True)
class Ensemble:
    draws: object            # (n_draws, m2, m1) numpy array, or None with keep_draws=False
    seed: int
    n_draws: int
    mean_field: np.ndarray
    empirical_se: np.ndarray
    rng_algorithm: str = RNG_ALGORITHM


def std_normals(seed: int, stream: int, count: int, start: int = 0, device: bool = False):
    """``_std_normals(_rng(seed, stream), count)`` (simulate.py:65-74) on the GPU: Philox4x64-10
    words ``start .. start + count - 1`` of the (seed, stream) key, bit-exact, through ndtri."""
    out = D.empty((int(count),))
    if count:
        N.call("rk_philox_normals", int(seed) & _M64, int(stream) & _M64, int(start), int(count), N.ptr(out),
               N.stream_ptr())
    return out if device else out.cpu().numpy()


def _embedding_handle(model, setup_or_grid):
    """Device object carrying the circulant embedding of (model, grid)."""
    from .rapid import RapidSetup
    if isinstance(setup_or_grid, RapidSetup) and setup_or_grid.model == model:
        return setup_or_grid.handle
    grid = setup_or_grid.grid if isinstance(setup_or_grid, RapidSetup) else setup_or_grid
    return GRID_SETUPS.get(model, grid).ptr


def embedding_dims(model, grid):
    emb = (N.C.c_int32 * 2)()
    dbl = N.C.c_int32()
    N.call("rk_setup_embedding", _embedding_handle(model, grid), N.C.byref(emb), N.C.byref(dbl))
    return int(emb[0]), int(emb[1]), bool(dbl.value)


def sim_unconditional_grid(model, grid, seed: int, device: bool = False):
    """Stationary field on the padded grid, (M2, M1), by circulant embedding (simulate.py:103-118)."""
    h = _embedding_handle(model, grid)
    g = grid.grid if hasattr(grid, "embed_dims") else grid
    M1, M2 = g.total_dims
    out = D.empty((M2, M1))
    N.call("rk_sim_unconditional_dev", h, int(seed) & _M64, N.ptr(out), N.stream_ptr())
    return out if device else out.cpu().numpy()


def sim_obs_local(model, setup, grid_field, seed: int):
    """z_i = A_i . g[N(i)] + sqrt(cond_var_i) eta_i + sqrt(tau2) eps_i (simulate.py:121-143)."""
    expect = tuple(setup.grid.total_dims[::-1])
    if tuple(grid_field.shape) != expect:
        raise DomainError(f"grid field shape {tuple(grid_field.shape)} does not match {expect}")
    dev = D.is_device_tensor(grid_field)
    g = D.to_device(grid_field)
    z = D.empty((setup.n_obs,))
    N.call("rk_sim_obs_local_dev", setup.handle, float(model.tau2), N.ptr(g), int(seed) & _M64,
           N.ptr(z), N.stream_ptr())
    return z if dev else z.cpu().numpy()


def conditional_draw(krig, setup, seed: int, grid_covariates=None, data_prediction=None):
    """data_prediction + (interior(g_uncond) - predict_rapid(refit(z_sim))) (simulate.py:146-159)."""
    f = as_device_fit(krig)
    g = sim_unconditional_grid(f.model, setup, draw_seed(seed, 101), device=True)
    zs = sim_obs_local(f.model, setup, g, draw_seed(seed, 202))
    bs, cs = refit_coefficients(f, D.to_device(zs))
    if data_prediction is None:
        data_prediction = predict_rapid(setup, D.to_device(f.c), f.beta_hat, grid_covariates)
    sim = predict_rapid(setup, cs, bs, grid_covariates)
    l, _, b, _ = setup.grid.pad
    m1, m2 = setup.grid.interior_dims
    dp = D.to_device(data_prediction)
    draw = dp + (g[b:b + m2, l:l + m1] - sim)
    return draw.cpu().numpy()


def shard_ranges(n_draws: int, n_shards: int):
    """Contiguous realization blocks [j0, j1) of ``n_shards`` workers (empty blocks dropped)."""
    k = max(1, int(n_shards))
    b = [(i * n_draws) // k for i in range(k + 1)]
    return [(b[i], b[i + 1]) for i in range(k)]


def _prepare(krig, setup, grid_covariates):
    f = as_device_fit(krig)
    beta, xg = _fixed_inputs(setup, f.beta_hat, grid_covariates)
    xd = None if xg is None else D.to_device(xg)
    dp = predict_rapid(setup, D.to_device(f.c), f.beta_hat, grid_covariates)
    return f, xd, dp


def new_accumulator(setup):
    """Exact fixed-point moment accumulator of one ensemble (int64, 6 x m2 x m1), zeroed."""
    m1, m2 = setup.grid.interior_dims
    return D.zeros((6, m2, m1), dtype=D.torch().int64)


def accumulate(setup, f, seed, j0, j1, xd, dp, acc, draws=None, batch=64, stream=None):
    """Adds the moments of e_j = draw_j - data_pred, j in [j0, j1), into ``acc`` (exact
    integer sums: the result does not depend on how the range is split or batched)."""
    if j1 <= j0:
        return acc
    N.call("rk_ensemble_accumulate", setup.handle, f.handle, int(seed) & _M64, int(j0), int(j1 - j0),
           N.ptr(xd), N.ptr(dp), N.ptr(acc), N.ptr(draws), int(batch), N.stream_ptr(stream))
    return acc


def combine(dst, src, stream=None):
    """dst += src for two accumulators on the same device (exact)."""
    N.call("rk_ensemble_combine", N.ptr(dst), N.ptr(src), dst.shape[1] * dst.shape[2], N.stream_ptr(stream))
    return dst


def finalize(dp, acc, n_draws, sigma2):
    mean = D.empty(dp.shape)
    se = D.empty(dp.shape)
    N.call("rk_ensemble_finalize", dp.numel(), int(n_draws), float(sigma2), N.ptr(dp), N.ptr(acc),
           N.ptr(mean), N.ptr(se), N.stream_ptr())
    return mean, se


def _devices(devices):
    """None: every visible GPU of this process -- unless torch.distributed runs one process per
    GPU, where each rank keeps to its own (use distributed.generate_ensemble_sharded there)."""
    torch = D.torch()
    if devices is None:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return [torch.cuda.current_device()]
        cur = torch.cuda.current_device()
        return [cur] + [d for d in range(torch.cuda.device_count()) if d != cur]
    if devices == "all":
        return list(range(torch.cuda.device_count()))
    return [int(d) for d in devices]


def _ensemble_multi(setup, f, seed, n_draws, xd, dp, devs, draws, batch):
    """Realization blocks on several GPUs of this process (setup / fit replicated peer to peer),
    one thread per GPU; accumulators summed exactly on the first GPU."""
    import threading
    torch = D.torch()
    ranges = shard_ranges(n_draws, len(devs))
    embedding_dims(setup.model, setup)   # simulation embedding and inverse factor built once,
    f.prepare_refit()                    # then copied with the replicas
    accs = [None] * len(devs)
    errs = []

    def work(i, d):
        try:
            with torch.cuda.device(d):
                st = setup.replica(d)
                fr = f.replica(d)
                s = torch.cuda.Stream(d)
                with torch.cuda.stream(s):
                    x = None if xd is None else xd.to(d)
                    p = dp.to(d)
                    acc = new_accumulator(setup)
                    j0, j1 = ranges[i]
                    dv = None
                    if draws is not None:
                        dv = draws[j0:j1] if d == draws.device.index else torch.empty(
                            (j1 - j0,) + tuple(dp.shape), dtype=torch.float64, device=d)
                    accumulate(st, fr, seed, j0, j1, x, p, acc, dv, batch, stream=s)
                    if draws is not None and dv.device != draws.device:
                        draws[j0:j1].copy_(dv)
                s.synchronize()
                accs[i] = acc
        except BaseException as e:   # re-raised on the calling thread
            errs.append(e)

    th = [threading.Thread(target=work, args=(i, d)) for i, d in enumerate(devs)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    total = accs[0] if accs[0].device == dp.device else accs[0].to(dp.device)
    for a in accs[1:]:
        combine(total, a.to(dp.device))
    return total


def generate_ensemble(krig, setup, n_draws: int, seed: int, grid_covariates=None, *,
                      keep_draws: bool = True, batch: int = 64, device: bool = False, devices=None):
    """n_draws conditional draws; draw j uses sub-seed draw_seed(seed, j) (simulate.py:174-192).

    ``devices``: None (every visible GPU of this process, the current one first; one GPU per
    rank under torch.distributed), "all" or a list of device indices; realizations are split into contiguous blocks, one per GPU, and the moments
    are combined exactly, so mean / SE are bitwise identical for any GPU count.
    ``keep_draws=False`` skips materialising the (n_draws, m2, m1) stack (the reference always
    returns it; at 4096^2 x 256 it is 34 GB) -- mean and SE are accumulated on the fly either way.
    """
    if n_draws < 2:
        raise DomainError(f"need at least 2 draws, got {n_draws}")
    f, xd, dp = _prepare(krig, setup, grid_covariates)
    m1, m2 = setup.grid.interior_dims
    draws = D.empty((n_draws, m2, m1)) if keep_draws else None
    devs = _devices(devices)
    if len(devs) > 1:
        acc = _ensemble_multi(setup, f, seed, n_draws, xd, dp, devs, draws, batch)
    else:
        acc = accumulate(setup, f, seed, 0, n_draws, xd, dp, new_accumulator(setup), draws, batch)
    mean, se = finalize(dp, acc, n_draws, f.model.sigma2)
    if device:
        return Ensemble(draws, int(seed), int(n_draws), mean, se)
    return Ensemble(None if draws is None else draws.cpu().numpy(), int(seed), int(n_draws),
                    mean.cpu().numpy(), se.cpu().numpy())
