"""Seeded synthetic inputs for the BASELINE.json configurations.

The paper's NorthAmericanRainfall2 data and any benchmark suite are not
available here; these generators produce inputs with the configs' shapes,
sizes and value distributions.  Pure numpy, host side: this is input
synthesis, not part of the GPU product path.

Config table (unset seeds use the config index; cfg2 mixture centres are drawn
U[0.2,0.8]^2 with equal weights — recorded choices):

====  =====  ====  =====  ======================================================
cfg   n      L     grid   model (sigma2, alpha = 1/range, nu, tau2) and z
====  =====  ====  =====  ======================================================
1     1000   2     100^2  (1, 10, 1.5, 0.01); z = 1 + g + N(0, 0.01)
2     1368   3     350^2  (1, 1/0.15, 1.0, 0.05); 3-comp mixture sd 0.15 clipped;
                          X = [1,x,y], beta = (0.5, 1, -1); z = X beta + g + eps
3     20000  4     2048^2 (1, 20, 2.5, 0.01); z = 1 + sum_8 a_k sin(2 pi u_k.s + phi_k) + eps
4     5000   3     512^2  (1, 10, 1.5, 0.02); z = 1 + g + eps; CS R = 1024
5     50000  1-4   256^2..4096^2 (1, 20, nu in {.5,1.5,2.5}, 0.01); sinusoid z
====  =====  ====  =====  ======================================================
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

UNIT = (0.0, 1.0, 0.0, 1.0)


@dataclass
class Workload:
    name: str
    obs: np.ndarray
    z: np.ndarray
    X: np.ndarray | None
    sigma2: float
    alpha: float
    nu: float
    tau2: float
    dims: tuple
    L: int
    domain: tuple = UNIT
    grid_covariates: str | None = None   # None or "1,x,y"
    extra: dict = field(default_factory=dict)


def _matern_dense(obs, sigma2, alpha, nu):
    """Dense covariance for drawing g exactly (uses scipy.special.kv; input synthesis)."""
    from scipy.spatial.distance import cdist
    from scipy.special import gamma, kv
    d = alpha * cdist(obs, obs)
    with np.errstate(invalid="ignore", divide="ignore"):
        phi = np.where(d > 1e-12, (d ** nu) * kv(nu, d) / (2 ** (nu - 1) * gamma(nu)), 1.0)
    k = sigma2 * np.clip(phi, 0.0, 1.0)
    return 0.5 * (k + k.T)


def _exact_gp(rng, obs, sigma2, alpha, nu):
    k = _matern_dense(obs, sigma2, alpha, nu)
    k[np.diag_indices_from(k)] += 1e-10 * sigma2
    return np.linalg.cholesky(k) @ rng.standard_normal(obs.shape[0])


def _sinusoid(rng, obs):
    a = rng.normal(0.0, 0.5, size=8)          # N(0, 0.25): variance 0.25
    u = rng.uniform(-6.0, 6.0, size=(8, 2))
    ph = rng.uniform(0.0, 2 * np.pi, size=8)
    return 1.0 + (a[None, :] * np.sin(2 * np.pi * (obs @ u.T) + ph[None, :])).sum(axis=1)


def cfg1(n=1000, dims=(100, 100), seed=0):
    rng = np.random.default_rng(seed)
    obs = rng.uniform(0, 1, size=(n, 2))
    g = _exact_gp(rng, obs, 1.0, 10.0, 1.5)
    z = 1.0 + g + rng.normal(0, np.sqrt(0.01), size=n)
    return Workload("cfg1", obs, z, None, 1.0, 10.0, 1.5, 0.01, dims, 2)


def cfg2(n=1368, dims=(350, 350), seed=2):
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.2, 0.8, size=(3, 2))
    comp = rng.integers(0, 3, size=n)
    obs = np.clip(centres[comp] + rng.normal(0, 0.15, size=(n, 2)), 0.0, 1.0)
    X = np.column_stack([np.ones(n), obs[:, 0], obs[:, 1]])
    beta = np.array([0.5, 1.0, -1.0])
    g = _exact_gp(rng, obs, 1.0, 1 / 0.15, 1.0)
    z = X @ beta + g + rng.normal(0, np.sqrt(0.05), size=n)
    return Workload("cfg2", obs, z, X, 1.0, 1 / 0.15, 1.0, 0.05, dims, 3,
                    grid_covariates="1,x,y", extra={"centres": centres})


def cfg3(n=20000, dims=(2048, 2048), seed=3):
    rng = np.random.default_rng(seed)
    obs = rng.uniform(0, 1, size=(n, 2))
    z = _sinusoid(rng, obs) + rng.normal(0, 0.1, size=n)
    return Workload("cfg3", obs, z, None, 1.0, 20.0, 2.5, 0.01, dims, 4)


def cfg4(n=5000, dims=(512, 512), seed=4):
    rng = np.random.default_rng(seed)
    obs = rng.uniform(0, 1, size=(n, 2))
    g = _exact_gp(rng, obs, 1.0, 10.0, 1.5)
    z = 1.0 + g + rng.normal(0, np.sqrt(0.02), size=n)
    return Workload("cfg4", obs, z, None, 1.0, 10.0, 1.5, 0.02, dims, 3,
                    extra={"n_draws": 1024, "ens_seed": 0})


def cfg5(nu=1.5, L=4, m=4096, n=50000, seed=5):
    rng = np.random.default_rng(seed)
    obs = rng.uniform(0, 1, size=(n, 2))
    z = _sinusoid(rng, obs) + rng.normal(0, 0.1, size=n)
    return Workload(f"cfg5-nu{nu}-L{L}-{m}", obs, z, None, 1.0, 20.0, nu, 0.01, (m, m), L,
                    extra={"n_draws": 256, "ens_seed": 0})


def grid_covariates_for(interior_nodes: np.ndarray, spec: str | None):
    """Covariates at the interior nodes (x fastest), e.g. '1,x,y' -> (N, 3)."""
    if spec is None:
        return None
    cols = []
    for term in spec.split(","):
        term = term.strip()
        if term == "1":
            cols.append(np.ones(interior_nodes.shape[0]))
        elif term == "x":
            cols.append(interior_nodes[:, 0])
        elif term == "y":
            cols.append(interior_nodes[:, 1])
        elif term in ("x*y", "xy"):
            cols.append(interior_nodes[:, 0] * interior_nodes[:, 1])
        else:
            raise ValueError(f"unknown covariate term {term!r}")
    return np.column_stack(cols)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}
