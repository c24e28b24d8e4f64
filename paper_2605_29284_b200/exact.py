"""Exact universal Kriging on the GPU: fit, batched GLS refit, prediction and its SE.

Interface of reference exact.py:40-175: ``KrigingFit`` (model, obs_locs, X,
chol_M, beta_hat, c), ``fit(model, obs_locs, z, X=None)`` (71-105),
``refit_coefficients(krig, z_new)`` (108-113), ``predict_exact(krig, targets,
target_covariates=None, chunk=20000)`` (132-147) and ``kriging_se_exact(krig, targets,
target_covariates=None, chunk=4000)`` (150-175).  The n x n factor stays on the
device; ``chol_M`` (lower, row-major like scipy) is copied out on first access.
``as_device_fit`` adopts a reference-built KrigingFit so ensembles can run on
the identical (chol_M, beta_hat, c).
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _device as D
from . import _native as N
from .covariance import CovarianceModel
from .errors import DomainError

__all__ = ["KrigingFit", "fit", "refit_coefficients", "predict_exact", "kriging_se_exact", "as_device_fit"]


class _FitHandle:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and N._lib is not None:
            N._lib.rk_fit_destroy(self.ptr)
            self.ptr = None


class KrigingFit:
    """Device-resident fit; attribute names follow exact.py:40-56."""

    def __init__(self, model, obs_locs, X, beta_hat, c, handle, chol_host=None, device=None):
        self.model = model
        self.obs_locs = obs_locs
        self.X = X
        self.beta_hat = beta_hat
        self.c = c
        self._h = handle
        self._chol = chol_host
        self.device = D.torch().cuda.current_device() if device is None else int(device)
        self._replicas = {}

    def prepare_refit(self, stream=None):
        """Build the inverse factor the batched refits use now (else on the first refit)."""
        N.call("rk_fit_prepare_refit", self.handle, N.stream_ptr(stream))

    def replica(self, device: int) -> "KrigingFit":
        """This fit on another GPU of the process: every device array copied peer to peer
        (bitwise), cached per device."""
        device = int(device)
        if device == self.device:
            return self
        if device not in self._replicas:
            h = N.C.c_void_p()
            N.call("rk_fit_replicate", self.handle, device, N.C.byref(h))
            self._replicas[device] = KrigingFit(self.model, self.obs_locs, self.X, self.beta_hat, self.c,
                                                _FitHandle(h), chol_host=self._chol, device=device)
        return self._replicas[device]

    @property
    def handle(self):
        return self._h.ptr

    @property
    def n_obs(self) -> int:
        return self.obs_locs.shape[0]

    @property
    def chol_M(self):
        if self._chol is None:
            n = self.n_obs
            ch = np.empty((n, n))
            N.call("rk_fit_copy_out", self._h.ptr, None, None, N.ptr(ch))
            self._chol = ch
        return self._chol

    def is_intercept_only(self) -> bool:
        return self.X.shape[1] == 1 and bool(np.all(self.X == self.X[0, 0]))


def _check_inputs(obs_locs, z, X):
    obs = np.ascontiguousarray(np.asarray(obs_locs, dtype=float).reshape(-1, 2))
    n = obs.shape[0]
    zz = None if z is None else np.ascontiguousarray(np.asarray(z, dtype=float).ravel())
    if zz is not None and zz.shape[0] != n:
        raise DomainError(f"z has {zz.shape[0]} entries for {n} locations")
    X = np.ones((n, 1)) if X is None else np.asarray(X, dtype=float)
    if X.ndim == 1:
        X = X[:, None]
    X = np.ascontiguousarray(X)
    p = X.shape[1]
    if X.shape[0] != n:
        raise DomainError(f"X has {X.shape[0]} rows for {n} locations")
    if not n >= p >= 1:
        raise DomainError(f"need n >= p >= 1, got n={n}, p={p}")
    if p > 8:
        raise DomainError("at most 8 covariates are supported")
    if np.linalg.matrix_rank(X) < p:
        raise DomainError("covariate matrix X is rank deficient")
    return obs, zz, X


def fit(model: CovarianceModel, obs_locs, z, X=None) -> KrigingFit:
    """Dense M = K + tau2 I, Cholesky (ridge retry 1e-10 tr(M)/n), GLS — on the GPU."""
    obs, zz, X = _check_inputs(obs_locs, z, X)
    n, p = X.shape
    h = N.C.c_void_p()
    ridge = N.C.c_int32(0)
    N.call("rk_fit_create", N.C.byref(model.native()), N.ptr(obs), n, N.ptr(zz), N.ptr(X), p,
           N.C.byref(h), N.C.byref(ridge))
    if ridge.value:
        warnings.warn("Cholesky of the observation covariance M failed; retried with ridge "
                      f"{1.0e-10 * (model.sigma2 + model.tau2):.3e}", RuntimeWarning, stacklevel=2)
    beta = np.empty(p)
    c = np.empty(n)
    N.call("rk_fit_copy_out", h, N.ptr(beta), N.ptr(c), None)
    return KrigingFit(model, obs, X, beta, c, _FitHandle(h))


def as_device_fit(krig) -> KrigingFit:
    """Our KrigingFit as is; any object with model/obs_locs/X/chol_M/beta_hat/c
    (e.g. the reference's) is uploaded once and cached on the object."""
    if isinstance(krig, KrigingFit):
        return krig
    cached = getattr(krig, "__dict__", {}).get("_b200_fit")
    if cached is not None:
        return cached
    m = krig.model
    model = m if isinstance(m, CovarianceModel) else CovarianceModel(m.sigma2, m.alpha, m.nu, m.tau2)
    obs = np.ascontiguousarray(np.asarray(krig.obs_locs, dtype=float))
    X = np.ascontiguousarray(np.asarray(krig.X, dtype=float))
    ch = np.ascontiguousarray(np.asarray(krig.chol_M, dtype=float))
    beta = np.ascontiguousarray(np.asarray(krig.beta_hat, dtype=float))
    c = np.ascontiguousarray(np.asarray(krig.c, dtype=float))
    h = N.C.c_void_p()
    N.call("rk_fit_import", N.C.byref(model.native()), N.ptr(obs), obs.shape[0], N.ptr(X), X.shape[1],
           N.ptr(ch), N.ptr(beta), N.ptr(c), N.C.byref(h))
    f = KrigingFit(model, obs, X, beta, c, _FitHandle(h), chol_host=ch)
    try:
        object.__setattr__(krig, "_b200_fit", f)
    except Exception:
        pass
    return f


def refit_coefficients(krig, z_new):
    """(beta_hat, c) for new data reusing the factorisation (exact.py:108-113).
    ``z_new`` may be (n,) or a batch (B, n); CUDA tensors stay on the device."""
    f = as_device_fit(krig)
    dev = D.is_device_tensor(z_new)
    z = D.to_device(z_new)
    batch = 1 if z.ndim == 1 else z.shape[0]
    if z.shape[-1] != f.n_obs:
        raise DomainError(f"z has {z.shape[-1]} entries for {f.n_obs} locations")
    p = f.X.shape[1]
    beta = D.empty((batch, p))
    c = D.empty((batch, f.n_obs))
    N.call("rk_refit_dev", f.handle, N.ptr(z), batch, N.ptr(beta), N.ptr(c), N.stream_ptr())
    if z.ndim == 1:
        beta, c = beta[0], c[0]
    if dev:
        return beta, c
    return beta.cpu().numpy(), c.cpu().numpy()


def _target_covariates(f: KrigingFit, targets: np.ndarray, target_covariates):
    """exact.py:116-129: None -> intercept-only fits use X[0, 0]; else (nt, p)."""
    if target_covariates is None:
        if not f.is_intercept_only():
            raise DomainError("fit uses nontrivial covariates; pass target_covariates for prediction")
        return None
    if D.is_device_tensor(target_covariates):
        xt = target_covariates.to(dtype=D.torch().float64)
        if xt.ndim == 1:
            xt = xt[:, None]
        shape = tuple(xt.shape)
    else:
        xt = np.asarray(target_covariates, dtype=float)
        if xt.ndim == 1:
            xt = xt[:, None]
        shape = xt.shape
    if shape != (targets.shape[0], f.X.shape[1]):
        raise DomainError(f"target covariates shape {shape} does not match "
                          f"({targets.shape[0]}, {f.X.shape[1]})")
    return D.to_device(xt).contiguous()


def _targets(targets):
    if D.is_device_tensor(targets):
        return targets.to(dtype=D.torch().float64).reshape(-1, 2).contiguous()
    return D.to_device(np.asarray(targets, dtype=float).reshape(-1, 2)).contiguous()


def predict_exact(krig, targets, target_covariates=None, chunk: int = 20000):
    """Exact Kriging prediction X_t beta_hat + k_t c at arbitrary targets (exact.py:132-147).
    ``chunk`` is accepted for signature compatibility: the cross covariance is never formed."""
    f = as_device_fit(krig)
    dev = D.is_device_tensor(targets)
    t = _targets(targets)
    xt = _target_covariates(f, t, target_covariates)
    out = D.empty((t.shape[0],))
    N.call("rk_predict_exact", f.handle, N.ptr(t), t.shape[0], N.ptr(xt), float(f.X[0, 0]), N.ptr(out),
           N.stream_ptr())
    return out if dev else out.cpu().numpy()


def kriging_se_exact(krig, targets, target_covariates=None, chunk: int = 4000):
    """Prediction standard error of the smooth field at each target (exact.py:150-175)."""
    f = as_device_fit(krig)
    dev = D.is_device_tensor(targets)
    t = _targets(targets)
    xt = _target_covariates(f, t, target_covariates)
    out = D.empty((t.shape[0],))
    N.call("rk_kriging_se_exact", f.handle, N.ptr(t), t.shape[0], N.ptr(xt), float(f.X[0, 0]), int(chunk),
           N.ptr(out), N.stream_ptr())
    return out if dev else out.cpu().numpy()
