"""The timing study on the GPU path (reference studies.run_timing).

Contract kept: ``run_timing(ns, grid_ladder, methods, reps, timeout_seconds, seed, nu,
corr_range, sigma2, tau2, cs_draws)`` returns one ``TimingRow(method, n, grid, setup_seconds,
predict_seconds, reps, censored)`` per (n, grid, method), n outermost; each cell's repeated
phase gets one untimed warm-up, then the median of ``reps`` timed calls; a warm-up longer than
``timeout_seconds`` censors the cell (its warm-up time is reported); setup and the repeated
phase are timed apart.  Data: n uniform locations (x then y) followed by n standard normals,
all from the (seed, n) Philox stream -- the same numbers as the reference draws.

Structure: each method is a ``Method`` whose ``prepare`` does (and times) the setup and
returns the zero-argument callable to repeat; ``Cell.measure`` owns the warm-up / median /
censoring protocol.  Timings are host wall clock around the synchronous public calls (each
returns host arrays, so the device work is inside).  ``cs-exact`` (a dense joint simulation,
not on the north-star path) is not provided by this build.
"""

from __future__ import annotations

import statistics
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


def _clock(fn):
    t = time.perf_counter()
    out = fn()
    return time.perf_counter() - t, out


class Method:
    def prepare(self, model, obs, z, dims, seed, cs_draws):
        """-> (setup seconds, callable repeated by the cell)"""
        raise NotImplementedError


class Exact(Method):
    def prepare(self, model, obs, z, dims, seed, cs_draws):
        setup_s, krig = _clock(lambda: fit(model, obs, z))
        nodes = build_padded_grid((0, 1, 0, 1), dims, 1, obs).interior_nodes()
        return setup_s, lambda: predict_exact(krig, nodes)


class Rapid(Method):
    def __init__(self, L):
        self.L = L

    def prepare(self, model, obs, z, dims, seed, cs_draws):
        krig = fit(model, obs, z)   # the fit is not part of the rapid method's setup
        setup_s, setup = _clock(lambda: build_setup(model, build_padded_grid((0, 1, 0, 1), dims, self.L, obs),
                                                    self.L, obs))
        return setup_s, lambda: predict_rapid(setup, krig.c, krig.beta_hat)


class FastCS(Method):
    L = 4

    def prepare(self, model, obs, z, dims, seed, cs_draws):
        def build():
            krig = fit(model, obs, z)
            return krig, build_setup(model, build_padded_grid((0, 1, 0, 1), dims, self.L, obs), self.L, obs)
        setup_s, (krig, setup) = _clock(build)
        return setup_s, lambda: generate_ensemble(krig, setup, cs_draws, seed)


METHODS = {"exact": Exact(), "rapid-L2": Rapid(2), "rapid-L4": Rapid(4), "rapid-L8": Rapid(8), "cs-fast": FastCS()}


@dataclass
class Cell:
    reps: int
    timeout: float

    def measure(self, fn):
        """(seconds, censored): warm-up, then the median of reps calls unless censored."""
        warm, _ = _clock(fn)
        if warm > self.timeout:
            return warm, True
        return statistics.median(_clock(fn)[0] for _ in range(self.reps)), False


def _study_data(seed, n):
    """n uniform x, n uniform y, then n normals of the (seed, n) Philox stream."""
    gen = np.random.Generator(np.random.Philox(key=(int(seed) & ((1 << 64) - 1)) + (int(n) << 64)))
    xy = np.column_stack([gen.uniform(0, 1, n), gen.uniform(0, 1, n)])
    return xy, std_normals(seed, n, n, start=2 * n)


def run_timing(ns=(200, 1500), grid_ladder=((60, 60), (100, 100), (140, 140)), methods=("exact", "rapid-L4"),
               reps: int = 3, timeout_seconds: float = 60.0, seed: int = 1, nu: float = 0.5,
               corr_range: float = 0.05, sigma2: float = 1.0, tau2: float = 0.1, cs_draws: int = 10) -> list:
    bad = [m for m in methods if m not in TIMING_METHODS]
    if bad:
        raise DomainError(f"unknown timing method {bad[0]!r}; choose from {TIMING_METHODS}")
    if reps < 1:
        raise DomainError("reps must be >= 1")
    missing = [m for m in methods if m not in METHODS]
    if missing:
        raise DomainError(f"timing method {missing[0]!r} (simulate_exact_ensemble) is not provided by this build")
    model = CovarianceModel(sigma2, 1.0 / corr_range, nu, tau2)
    cell = Cell(reps, timeout_seconds)
    rows = []
    for n in ns:
        obs, z = _study_data(seed, n)
        for dims in grid_ladder:
            for name in methods:
                setup_s, call = METHODS[name].prepare(model, obs, z, dims, seed, cs_draws)
                t, censored = cell.measure(call)
                rows.append(TimingRow(name, n, tuple(dims), setup_s, float(t), reps, censored))
    return rows
