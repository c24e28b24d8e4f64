"""Rapid grid prediction on the B200: device-resident setup + 3-pass FFT convolution.

Drop-in for reference rapid.py (same names and signatures):
``build_setup(model, grid, L, obs_locs) -> RapidSetup`` (rapid.py:177-230),
``predict_rapid(setup, c, beta_hat=None, grid_covariates=None)`` (252-261),
``RapidSetup.coefficients_to_grid`` (164-174), ``next_fft_len`` (46-59),
``build_filter_spectrum`` (72-86), ``convolve_filter`` (89-100),
``neighbor_cov`` (112-117) and the ``BUILD_COUNT`` instrumentation (42-43).

Host buffers in -> host arrays out (the reference semantics, H2D/D2H included);
CUDA tensors in -> CUDA tensors out (the device-resident path).  All arithmetic
runs in librapidkrig_b200.so; nothing here computes a field on the CPU.
"""

from __future__ import annotations

import warnings

import numpy as np

from . import _device as D
from . import _native as N
from .covariance import CovarianceModel
from .errors import DomainError
from .gridding import PaddedGrid

__all__ = ["RapidSetup", "build_setup", "predict_rapid", "next_fft_len",
           "build_filter_spectrum", "convolve_filter", "neighbor_cov", "FilterSpectrum"]

BUILD_COUNT = 0


def next_fft_len(n: int) -> int:
    """Smallest 2^a 3^b >= n (rapid.py:46-59)."""
    n = int(n)
    if n <= 1:
        return 1
    best = None
    pow2 = 1
    while pow2 < 4 * n:
        v = pow2
        while v < n:
            v *= 3
        best = v if best is None or v < best else best
        pow2 *= 2
    return best


class _Handle:
    """Owns an rk_setup*; destroyed with the Python object."""

    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        if self.ptr and N._lib is not None:
            N._lib.rk_setup_destroy(self.ptr)
            self.ptr = None


def _info(h):
    n = N.C.c_int64()
    L = N.C.c_int32()
    emb = (N.C.c_int32 * 2)()
    tot = (N.C.c_int32 * 2)()
    N.call("rk_setup_info", h, N.C.byref(n), N.C.byref(L), N.C.byref(emb), N.C.byref(tot))
    return int(n.value), int(L.value), (int(emb[0]), int(emb[1])), (int(tot[0]), int(tot[1]))


class FilterSpectrum:
    """Device-resident filter spectrum of one (model, grid); ``np.asarray`` gives the
    complex (p2, p1) array the reference's build_filter_spectrum returns."""

    def __init__(self, handle: _Handle, embed_dims):
        self._h = handle
        self.embed_dims = embed_dims
        self._host = None

    def __array__(self, dtype=None, copy=None):
        if self._host is None:
            p1, p2 = self.embed_dims
            re = np.empty((p2, p1))
            N.call("rk_setup_copy_spectrum", self._h.ptr, N.ptr(re))
            self._host = re.astype(np.complex128)
        return self._host if dtype is None else self._host.astype(dtype)

    @property
    def shape(self):
        return (self.embed_dims[1], self.embed_dims[0])


class RapidSetup:
    """Immutable device-resident setup (reference rapid.py:138-174)."""

    def __init__(self, model, grid, L, handle, ridge_applied=False, device=None):
        self.model = model
        self.grid = grid
        self.L = int(L)
        self._h = handle
        self.ridge_applied = bool(ridge_applied)
        n, _, emb, tot = _info(handle.ptr)
        self._n = n
        self.embed_dims = emb
        ex = (N.C.c_int32 * 2)()
        N.call("rk_setup_exec_dims", handle.ptr, N.C.byref(ex))
        self.exec_dims = (int(ex[0]), int(ex[1]))   # the torus predict_rapid runs on (see the C header)
        self._total = tot
        self._cache = {}
        self.device = D.torch().cuda.current_device() if device is None else int(device)
        self._replicas = {}

    def replica(self, device: int) -> "RapidSetup":
        """This setup on another GPU of the process: every device array (incl. the simulation
        embedding, if built) copied peer to peer, bitwise; cached per device."""
        device = int(device)
        if device == self.device:
            return self
        if device not in self._replicas:
            h = N.C.c_void_p()
            N.call("rk_setup_replicate", self.handle, device, N.C.byref(h))
            self._replicas[device] = RapidSetup(self.model, self.grid, self.L, _Handle(h), self.ridge_applied,
                                                device=device)
        return self._replicas[device]

    @property
    def handle(self):
        return self._h.ptr

    @property
    def n_obs(self) -> int:
        return self._n

    @property
    def block_size(self) -> int:
        return (2 * self.L) ** 2

    def _copy_out(self):
        if not self._cache:
            n, M = self._n, self.block_size
            idx = np.empty((n, M), dtype=np.int64)
            w = np.empty((n, M))
            cv = np.empty(n)
            kinv = np.empty((M, M))
            N.call("rk_setup_copy_out", self._h.ptr, N.ptr(idx), N.ptr(w), N.ptr(cv), N.ptr(kinv))
            self._cache.update(neighbor_indices=idx, weights=w, cond_var=cv, kn_inv=kinv)
        return self._cache

    # reference fields, materialised lazily from device memory
    @property
    def neighbor_indices(self):
        return self._copy_out()["neighbor_indices"]

    @property
    def weights(self):
        return self._copy_out()["weights"]

    @property
    def cond_var(self):
        return self._copy_out()["cond_var"]

    @property
    def kn_inv(self):
        return self._copy_out()["kn_inv"]

    @property
    def filter_spectrum(self):
        return np.asarray(FilterSpectrum(self._h, self.embed_dims))

    def coefficients_to_grid(self, c):
        """c* = A' c on the padded grid, (M2, M1); deterministic gather (no atomics)."""
        dev = D.is_device_tensor(c)
        cd = D.to_device(c).reshape(-1)
        if cd.shape[0] != self._n:
            raise DomainError(f"coefficient vector has {cd.shape[0]} entries for {self._n} observations")
        M1, M2 = self._total
        out = D.empty((M2, M1))
        N.call("rk_coefficients_to_grid", self._h.ptr, N.ptr(cd), N.ptr(out), N.stream_ptr())
        return out if dev else out.cpu().numpy()


def build_setup(model: CovarianceModel, grid: PaddedGrid, L: int, obs_locs) -> RapidSetup:
    """K_N factor, stencils, weights, conditional variances, filter spectrum — on the GPU."""
    global BUILD_COUNT
    obs = np.ascontiguousarray(np.asarray(obs_locs, dtype=float).reshape(-1, 2))
    if obs.shape[0] == 0:
        raise DomainError("build_setup requires at least one observation")
    h = N.C.c_void_p()
    ridge = N.C.c_int32(0)
    N.call("rk_build_setup", N.C.byref(model.native()), N.C.byref(grid.native()), int(L),
           N.ptr(obs), obs.shape[0], N.C.byref(h), N.C.byref(ridge))
    if ridge.value:
        r = 1.0e-12 * model.sigma2 * (2 * L) ** 2
        warnings.warn(f"neighbor covariance K_N is numerically singular; adding ridge {r:.3e} "
                      "(reduce L or roughen nu to avoid this)", RuntimeWarning, stacklevel=2)
    BUILD_COUNT += 1
    return RapidSetup(model, grid, L, _Handle(h), bool(ridge.value))


def _fixed_inputs(setup: RapidSetup, beta_hat, grid_covariates):
    """Validation of rapid.py:233-249; returns (beta f64 array | None, xg (N,p) | None)."""
    if beta_hat is None:
        return None, None
    if D.is_device_tensor(beta_hat):      # stays on the device: no host sync on the hot path
        beta = beta_hat.reshape(-1)
    else:
        beta = D.host_f64(beta_hat).ravel()
    m1, m2 = setup.grid.interior_dims
    if grid_covariates is None:
        if beta.shape[0] != 1:
            raise DomainError("grid covariates are required when beta_hat has more than one entry")
        return beta, None
    xg = grid_covariates
    if D.is_device_tensor(xg):
        if xg.ndim == 3:
            xg = xg.reshape(-1, xg.shape[2])
        shape = tuple(xg.shape)
    else:
        xg = np.asarray(xg, dtype=float)
        if xg.ndim == 3:
            xg = xg.reshape(-1, xg.shape[2])
        shape = xg.shape
    if shape != (m1 * m2, beta.shape[0]):
        raise DomainError(f"grid covariates shape {shape} does not match ({m1 * m2}, {beta.shape[0]})")
    return beta, xg


def _device_f64(t):
    """Contiguous float64 CUDA tensor on the current device (converted if needed)."""
    torch = D.torch()
    if (D.is_device_tensor(t) and t.dtype == torch.float64 and t.is_contiguous()
            and t.device.index == torch.cuda.current_device()):
        return t
    return D.to_device(t)


def _check_out(out, shape, device: bool):
    """``out`` must be a C-contiguous float64 (m2, m1) buffer: a CUDA tensor on the current
    device for device inputs, a host array otherwise."""
    torch = D.torch()
    if device:
        ok = (D.is_device_tensor(out) and out.dtype == torch.float64 and out.is_contiguous()
              and tuple(out.shape) == shape and out.device.index == torch.cuda.current_device())
    else:
        ok = (isinstance(out, np.ndarray) and out.dtype == np.float64 and out.flags.c_contiguous
              and out.shape == shape and out.flags.writeable)
    if not ok:
        kind = "CUDA tensor on the current device" if device else "writeable numpy array"
        raise DomainError(f"out must be a C-contiguous float64 {kind} of shape {shape}")


def predict_rapid(setup: RapidSetup, c, beta_hat=None, grid_covariates=None, *, out=None):
    """(m2, m1) interior field: FFT convolution of A'c with the covariance filter + X_g beta.

    ``out`` (optional) receives the result: a CUDA tensor on the device path, or a
    host float64 array (e.g. a pinned buffer) on the host path."""
    m1, m2 = setup.grid.interior_dims
    beta, xg = _fixed_inputs(setup, beta_hat, grid_covariates)
    p = 0 if beta is None else beta.shape[0]
    if D.is_device_tensor(c):
        cd = c.reshape(-1)
        if cd.dtype != D.torch().float64 or not cd.is_contiguous():
            cd = cd.to(dtype=D.torch().float64).contiguous()
        if cd.shape[0] != setup.n_obs:
            raise DomainError(f"coefficient vector has {cd.shape[0]} entries for {setup.n_obs} observations")
        # every buffer the library reads / writes as raw float64 must be contiguous float64 on
        # this device (a strided or float32 tensor would be misread / overrun)
        bd = None if beta is None else _device_f64(beta)
        xd = None if xg is None else _device_f64(xg)
        if out is None:
            res = D.empty((m2, m1))
        else:
            _check_out(out, (m2, m1), device=True)
            res = out
        N.call("rk_predict_dev", setup.handle, N.ptr(cd), N.ptr(bd), p, N.ptr(xd), N.ptr(res),
               N.stream_ptr())
        return res
    ch = D.host_f64(c).ravel()
    if ch.shape[0] != setup.n_obs:
        raise DomainError(f"coefficient vector has {ch.shape[0]} entries for {setup.n_obs} observations")
    bh = None if beta is None else D.host_f64(beta.cpu().numpy() if D.is_device_tensor(beta) else beta)
    xh = None if xg is None else D.host_f64(xg.cpu().numpy() if D.is_device_tensor(xg) else xg)
    if out is None:
        res = np.empty((m2, m1))
    else:
        _check_out(out, (m2, m1), device=False)
        res = out
    # synchronous host-buffer call: on the setup's own stream (no torch stream lookup)
    N.call("rk_predict_host", setup.handle, N.ptr(ch), N.ptr(bh), p, N.ptr(xh), N.ptr(res), None)
    return res


class _GridSetupCache:
    """Observation-free setups keyed by value (like simulate.py:82 lru_cache(maxsize=8))."""

    def __init__(self, maxsize=8):
        self.maxsize = maxsize
        self._d = {}

    def get(self, model: CovarianceModel, grid: PaddedGrid):
        key = (model, grid)
        if key in self._d:
            h = self._d.pop(key)
            self._d[key] = h
            return h
        ptr = N.C.c_void_p()
        N.call("rk_grid_setup_create", N.C.byref(model.native()), N.C.byref(grid.native()),
               N.C.byref(ptr))
        h = _Handle(ptr)
        self._d[key] = h
        while len(self._d) > self.maxsize:
            self._d.pop(next(iter(self._d)))
        return h


GRID_SETUPS = _GridSetupCache()


def build_filter_spectrum(model: CovarianceModel, grid: PaddedGrid):
    """((p1, p2), spectrum) on the (2M-1)-rounded torus; spectrum is device resident
    and converts to the reference's complex (p2, p1) array via np.asarray."""
    h = GRID_SETUPS.get(model, grid)
    _, _, emb, _ = _info(h.ptr)
    return emb, FilterSpectrum(h, emb)


def convolve_filter(spectrum, embed_dims, values):
    """Leading (M2, M1) block of the circulant convolution of ``values`` (rapid.py:89-100)."""
    p1, p2 = int(embed_dims[0]), int(embed_dims[1])
    dev = D.is_device_tensor(values)
    v = D.to_device(values)
    M2, M1 = v.shape
    out = D.empty((M2, M1))
    if isinstance(spectrum, FilterSpectrum) and _info(spectrum._h.ptr)[3] == (M1, M2):
        N.call("rk_convolve_filter", spectrum._h.ptr, N.ptr(v), N.ptr(out), N.stream_ptr())
    else:
        q = _quarter_from_full(np.asarray(spectrum), p1, p2)
        N.call("rk_convolve_spectrum", N.ptr(q), p1, p2, N.ptr(v), M1, M2, N.ptr(out),
               N.stream_ptr())
        D.torch().cuda.current_stream().synchronize()
    return out if dev else out.cpu().numpy()


def _quarter_from_full(spec, p1, p2):
    """Real part of a real-even (p2, p1) spectrum as the kernels' quarter layout,
    q[kx, ky] = Re S[ky, kx] / (p1 p2) for kx <= p1/2, ky <= p2/2 (device tensor)."""
    s = np.asarray(spec)
    if s.shape != (p2, p1):
        raise DomainError(f"spectrum shape {s.shape} does not match embed dims {(p2, p1)}")
    re = np.real(s)
    ldq = ((p2 // 2 + 1) + 1) & ~1
    q = np.zeros((p1 // 2 + 1, ldq))
    q[:, : p2 // 2 + 1] = re[: p2 // 2 + 1, : p1 // 2 + 1].T / (float(p1) * float(p2))
    return D.to_device(q)


def neighbor_cov(model: CovarianceModel, grid: PaddedGrid, L: int):
    """Shared (2L)^2 x (2L)^2 neighbour covariance (rapid.py:103-117)."""
    hx, hy = grid.spacing
    gx, gy = np.meshgrid(np.arange(2 * L) * hx, np.arange(2 * L) * hy)
    off = np.column_stack([gx.ravel(), gy.ravel()])
    d = np.hypot(off[:, None, 0] - off[None, :, 0], off[:, None, 1] - off[None, :, 1])
    k = model.covariance(d)
    return 0.5 * (k + k.T)
