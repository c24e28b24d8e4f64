"""Matern covariance model; evaluation runs on the GPU (rk_matern_cov).

Interface mirrors reference covariance.py:50-116 (``CovarianceModel`` with
``correlation``/``covariance``, ``matern_phi``, ``cov``, ``cov_matrix``): the
kernel is ``sigma2 * phi(alpha * |s - s'|)`` with alpha multiplying distance.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .errors import DomainError

__all__ = ["CovarianceModel", "matern_phi", "cov", "cov_matrix"]


@dataclass(frozen=True)
class CovarianceModel:
    """sigma2 > 0 (variance), alpha > 0 (inverse range), nu > 0 (smoothness), tau2 >= 0 (nugget)."""

    sigma2: float
    alpha: float
    nu: float
    tau2: float = 0.0

    def __post_init__(self):
        # same acceptance rules as covariance.py:80-88
        for name, bad in (("sigma2", not self.sigma2 > 0), ("alpha", not self.alpha > 0),
                          ("nu", not self.nu > 0), ("tau2", self.tau2 < 0)):
            if bad:
                raise DomainError(f"invalid {name}={getattr(self, name)!r}")

    def native(self) -> N.RkModel:
        return N.make_model(self.sigma2, self.alpha, self.nu, self.tau2)

    def covariance_device(self, dist):
        """sigma2 * phi(alpha * dist) for a CUDA tensor (returns a CUDA tensor)."""
        d = D.to_device(dist)
        out = D.empty(d.shape)
        m = self.native()
        N.call("rk_matern_cov", m, N.ptr(d), N.ptr(out), d.numel(), N.stream_ptr())
        return out

    def covariance(self, dist):
        d = np.asarray(dist, dtype=float)
        if np.any(d < 0):
            raise DomainError("distance must be nonnegative")
        out = self.covariance_device(np.atleast_1d(d)).cpu().numpy().reshape(np.atleast_1d(d).shape)
        return out[0] if d.ndim == 0 else out.reshape(d.shape)

    def correlation(self, dist):
        return self.covariance(dist) / self.sigma2


def matern_phi(d, nu: float):
    """phi(d) for dimensionless d >= 0 (reference bessel.py:258-278)."""
    if not nu > 0:
        raise DomainError(f"Matern smoothness must be positive, got nu={nu}")
    return CovarianceModel(1.0, 1.0, nu).covariance(d)


def cov(model: CovarianceModel, s, s2) -> float:
    s = np.asarray(s, dtype=float)
    s2 = np.asarray(s2, dtype=float)
    return float(model.covariance(float(np.linalg.norm(s - s2))))


def cov_matrix(model: CovarianceModel, locs_a, locs_b=None):
    """Dense covariance between location sets (reference covariance.py:100-116)."""
    t = D.torch()
    a = np.atleast_2d(np.asarray(locs_a, dtype=float))
    if a.size == 0:
        raise DomainError("cov_matrix requires at least one location")
    b = a if locs_b is None else np.atleast_2d(np.asarray(locs_b, dtype=float))
    if b.size == 0:
        raise DomainError("cov_matrix requires at least one location")
    da, db = D.to_device(a), D.to_device(b)
    dist = t.sqrt(((da[:, None, :] - db[None, :, :]) ** 2).sum(-1))
    k = model.covariance_device(dist)
    if locs_b is None:
        k = 0.5 * (k + k.T)
    return k.cpu().numpy()
