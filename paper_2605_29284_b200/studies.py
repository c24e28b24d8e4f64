"""The timing study (reference studies.py:289-390: ``run_timing``) on the GPU path.

Same protocol and rows: for every (n, grid, method) cell one warm-up run, then the median of
``reps`` timed runs (wall clock around the synchronous public calls); a warm-up longer than
``timeout_seconds`` censors the cell; setup (fit / weights) and the per-prediction phase are
timed separately.  Data: n uniform locations from the (seed, n) Philox stream and z from
``std_normals`` (identical to the reference's draws).  Methods: ``exact`` (GPU fit +
``predict_exact`` at every interior node), ``rapid-L{2,4,8}``, ``cs-fast`` (a
``cs_draws``-member ensemble); ``cs-exact`` (``simulate_exact_ensemble``) is not provided by
this build.  The error and convergence studies are outside the hot-path scope.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .covariance import CovarianceModel
from .errors import DomainError
from .exact import fit, predict_exact
from .gridding import build_padded_grid
from .rapid import build_setup, predict_rapid
from .simulate import generate_ensemble, std_normals

__all__ = ["TimingRow", "TIMING_METHODS", "run_timing"]


@dataclass(frozen=True)
class TimingRow:
    method: str
    n: int
    grid: tuple
    setup_seconds: float
    predict_seconds: float
    reps: int
    censored: bool = False


TIMING_METHODS = ("exact", "rapid-L2", "rapid-L4", "rapid-L8", "cs-exact", "cs-fast")


def _median_time(fn, reps, timeout_seconds):
    t0 = time.perf_counter()
    fn()
    warm = time.perf_counter() - t0
    if warm > timeout_seconds:
        return warm, True
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)), False


def _locations(seed, n):
    """Uniform locations like studies.py:324-325 (two uniform draws from the (seed, n) stream)."""
    rng = np.random.Generator(np.random.Philox(key=(int(seed) & ((1 << 64) - 1)) + (int(n) << 64)))
    x = rng.uniform(0, 1, n)
    y = rng.uniform(0, 1, n)
    # the reference then draws z from the same generator: the words after 2n
    return np.column_stack([x, y])


def _cell(method, model, obs, z, dims, reps, timeout, seed, cs_draws):
    n = obs.shape[0]
    if method == "exact":
        t0 = time.perf_counter()
        krig = fit(model, obs, z)
        setup_s = time.perf_counter() - t0
        nodes = build_padded_grid((0, 1, 0, 1), dims, 1, obs).interior_nodes()
        pred_s, cen = _median_time(lambda: predict_exact(krig, nodes), reps, timeout)
        return TimingRow(method, n, tuple(dims), setup_s, pred_s, reps, cen)
    if method.startswith("rapid-L"):
        L = int(method.split("L")[1])
        krig = fit(model, obs, z)
        t0 = time.perf_counter()
        grid = build_padded_grid((0, 1, 0, 1), dims, L, obs)
        setup = build_setup(model, grid, L, obs)
        setup_s = time.perf_counter() - t0
        pred_s, cen = _median_time(lambda: predict_rapid(setup, krig.c, krig.beta_hat), reps, timeout)
        return TimingRow(method, n, tuple(dims), setup_s, pred_s, reps, cen)
    if method == "cs-fast":
        t0 = time.perf_counter()
        krig = fit(model, obs, z)
        grid = build_padded_grid((0, 1, 0, 1), dims, 4, obs)
        setup = build_setup(model, grid, 4, obs)
        setup_s = time.perf_counter() - t0
        pred_s, cen = _median_time(lambda: generate_ensemble(krig, setup, cs_draws, seed), reps, timeout)
        return TimingRow(method, n, tuple(dims), setup_s, pred_s, reps, cen)
    raise DomainError(f"timing method {method!r} (simulate_exact_ensemble) is not provided by this build")


def run_timing(ns=(200, 1500), grid_ladder=((60, 60), (100, 100), (140, 140)), methods=("exact", "rapid-L4"),
               reps: int = 3, timeout_seconds: float = 60.0, seed: int = 1, nu: float = 0.5,
               corr_range: float = 0.05, sigma2: float = 1.0, tau2: float = 0.1, cs_draws: int = 10) -> list:
    for m in methods:
        if m not in TIMING_METHODS:
            raise DomainError(f"unknown timing method {m!r}; choose from {TIMING_METHODS}")
    if reps < 1:
        raise DomainError("reps must be >= 1")
    model = CovarianceModel(sigma2, 1.0 / corr_range, nu, tau2)
    rows = []
    for n in ns:
        obs = _locations(seed, n)
        # z = _std_normals(rng, n) after the 2n uniform draws of the same (seed, n) stream
        z = std_normals(seed, n, n, start=2 * n)
        for dims in grid_ladder:
            for method in methods:
                rows.append(_cell(method, model, obs, z, dims, reps, timeout_seconds, seed, cs_draws))
    return rows
