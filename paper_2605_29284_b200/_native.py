"""ctypes binding of librapidkrig_b200.so (the C ABI in include/rapidkrig_b200.h).

The library is built in-tree (``python -m paper_2605_29284_b200.build``).  There
is no CPU fallback: if the library or a CUDA device is missing, every entry
point raises :class:`RapidKrigError` instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import threading

from .errors import DomainError, InternalError, NumericError, RapidKrigError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librapidkrig_b200.so")

RK_OK, RK_DOMAIN, RK_NUMERIC, RK_INTERNAL, RK_CUDA = range(5)

_EULER = 0.5772156649015329


class RkModel(C.Structure):
    _fields_ = [("sigma2", C.c_double), ("alpha", C.c_double), ("nu", C.c_double),
                ("tau2", C.c_double), ("half_n", C.c_int32), ("nl", C.c_int32),
                ("half_coef", C.c_double * 13), ("half_pref", C.c_double), ("mu", C.c_double),
                ("temme_gampl", C.c_double), ("temme_gammi", C.c_double),
                ("temme_gam1", C.c_double), ("temme_gam2", C.c_double),
                ("temme_fact", C.c_double), ("gamma_nu", C.c_double)]


class RkGrid(C.Structure):
    _fields_ = [("x0", C.c_double), ("y0", C.c_double), ("hx", C.c_double), ("hy", C.c_double),
                ("m1", C.c_int32), ("m2", C.c_int32), ("pad", C.c_int32 * 4)]


_vp = C.c_void_p
_i32 = C.c_int32
_i64 = C.c_int64
_u64 = C.c_uint64
_dp = C.c_void_p      # device or host double* (passed as an address)

_PROTOS = {
    "rk_last_error": (C.c_char_p, []),
    "rk_version": (_i32, []),
    "rk_launch_count": (_i64, []),
    "rk_matern_cov": (_i32, [C.POINTER(RkModel), _dp, _dp, _i64, _vp]),
    "rk_build_padded_grid": (_i32, [C.POINTER(C.c_double * 4), _i32, _i32, _i32, _dp, _i64,
                                    C.POINTER(RkGrid)]),
    "rk_build_setup": (_i32, [C.POINTER(RkModel), C.POINTER(RkGrid), _i32, _dp, _i64,
                              C.POINTER(_vp), C.POINTER(_i32)]),
    "rk_grid_setup_create": (_i32, [C.POINTER(RkModel), C.POINTER(RkGrid), C.POINTER(_vp)]),
    "rk_setup_destroy": (_i32, [_vp]),
    "rk_setup_info": (_i32, [_vp, C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i32 * 2),
                             C.POINTER(_i32 * 2)]),
    "rk_setup_copy_out": (_i32, [_vp, _dp, _dp, _dp, _dp]),
    "rk_setup_copy_spectrum": (_i32, [_vp, _dp]),
    "rk_setup_exec_dims": (_i32, [_vp, C.POINTER(_i32 * 2)]),
    "rk_coefficients_to_grid": (_i32, [_vp, _dp, _dp, _vp]),
    "rk_convolve_filter": (_i32, [_vp, _dp, _dp, _vp]),
    "rk_convolve_spectrum": (_i32, [_dp, _i32, _i32, _dp, _i32, _i32, _dp, _vp]),
    "rk_predict_dev": (_i32, [_vp, _dp, _dp, _i32, _dp, _dp, _vp]),
    "rk_predict_host": (_i32, [_vp, _dp, _dp, _i32, _dp, _dp, _vp]),
    "rk_predict_profile": (_i32, [_vp, _dp, _dp, _i32, _dp, _dp, _vp, C.POINTER(C.c_float * 4)]),
    "rk_predict_traffic": (_i32, [_vp, _i32, C.POINTER(C.c_double * 4)]),
    "rk_setup_time_weights": (_i32, [_vp, _vp, _i32, C.POINTER(C.c_float)]),
    "rk_setup_weights_into": (_i32, [_vp, _dp, _dp, _dp, _dp, _vp]),
    "rk_fit_create": (_i32, [C.POINTER(RkModel), _dp, _i64, _dp, _dp, _i32, C.POINTER(_vp),
                             C.POINTER(_i32)]),
    "rk_fit_import": (_i32, [C.POINTER(RkModel), _dp, _i64, _dp, _i32, _dp, _dp, _dp,
                             C.POINTER(_vp)]),
    "rk_fit_destroy": (_i32, [_vp]),
    "rk_fit_copy_out": (_i32, [_vp, _dp, _dp, _dp]),
    "rk_fit_info": (_i32, [_vp, C.POINTER(_i64), C.POINTER(_i32)]),
    "rk_refit_dev": (_i32, [_vp, _dp, _i64, _dp, _dp, _vp]),
    "rk_predict_exact": (_i32, [_vp, _dp, _i64, _dp, C.c_double, _dp, _vp]),
    "rk_kriging_se_exact": (_i32, [_vp, _dp, _i64, _dp, C.c_double, _i64, _dp, _vp]),
    "rk_draw_seed": (_u64, [_u64, _u64]),
    "rk_philox_normals": (_i32, [_u64, _u64, _u64, _i64, _dp, _vp]),
    "rk_philox_raw": (_i32, [_u64, _u64, _u64, _i64, _dp, _vp]),
    "rk_setup_embedding": (_i32, [_vp, C.POINTER(_i32 * 2), C.POINTER(_i32)]),
    "rk_sim_unconditional_dev": (_i32, [_vp, _u64, _dp, _vp]),
    "rk_sim_obs_local_dev": (_i32, [_vp, C.c_double, _dp, _u64, _dp, _vp]),
    "rk_ensemble_accumulate": (_i32, [_vp, _vp, _u64, _i64, _i64, _dp, _dp, _dp, _dp, _i32, _vp]),
    "rk_ensemble_accumulate_values": (_i32, [_dp, _i32, _i64, C.c_double, _dp, _vp]),
    "rk_ensemble_combine": (_i32, [_dp, _dp, _i64, _vp]),
    "rk_ensemble_finalize": (_i32, [_i64, _i64, C.c_double, _dp, _dp, _dp, _dp, _vp]),
    "rk_fit_prepare_refit": (_i32, [_vp, _vp]),
    "rk_setup_replicate": (_i32, [_vp, _i32, C.POINTER(_vp)]),
    "rk_fit_replicate": (_i32, [_vp, _i32, C.POINTER(_vp)]),
    "rk_setup_blob_bytes": (_i32, [_vp, C.POINTER(_i64)]),
    "rk_setup_export": (_i32, [_vp, _dp, _vp]),
    "rk_setup_import": (_i32, [_dp, _i64, C.POINTER(_vp)]),
    "rk_fit_shell": (_i32, [C.POINTER(RkModel), _i64, _i32, _i32, C.POINTER(_vp)]),
    "rk_fit_fields": (_i32, [_vp, C.POINTER(_vp * 7), C.POINTER(_i64 * 7)]),
    "rk_fit_get_gram": (_i32, [_vp, _dp, _dp]),
    "rk_fit_set_gram": (_i32, [_vp, _dp, _dp]),
    "rk_refit_profile": (_i32, [_vp, _i64, _i32, _vp, C.POINTER(C.c_float * 2)]),
}

_lock = threading.Lock()
_lib = None


def exported_symbols():
    return sorted(_PROTOS)


def load(require_gpu: bool = True):
    """Load the shared library (once).  ``require_gpu`` also checks a CUDA device."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise RapidKrigError(
                    f"CUDA library {LIB_PATH} is not built; run python -m paper_2605_29284_b200.build "
                    "(there is no CPU fallback)")
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in _PROTOS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    if require_gpu:
        import torch
        if not torch.cuda.is_available():
            raise RapidKrigError("no CUDA device visible: the rapidkrig B200 path has no CPU fallback")
    return _lib


def check(status: int):
    if status == RK_OK:
        return
    msg = (_lib.rk_last_error() or b"").decode("utf-8", "replace")
    if status == RK_DOMAIN:
        raise DomainError(msg)
    if status == RK_NUMERIC:
        raise NumericError(msg)
    if status == RK_INTERNAL:
        raise InternalError(msg)
    raise RapidKrigError(msg)


def call(name, *args):
    lib = load()
    check(getattr(lib, name)(*args))


def launch_count() -> int:
    return int(load(require_gpu=False).rk_launch_count())


# ------------------------------------------------------------------ model constants
def half_integer_order(nu: float):
    """bessel.py:216-221."""
    n = int(round(nu - 0.5))
    if 0 <= n <= 12 and abs(nu - (n + 0.5)) < 1.0e-12:
        return n
    return None


def make_model(sigma2: float, alpha: float, nu: float, tau2: float) -> RkModel:
    """rk_model with the constants computed exactly as the reference computes them:
    Horner coefficients by exact-integer true division (bessel.py:231-234), Temme
    gammas via math.gamma (bessel.py:37-47, 57), Gamma(nu) (bessel.py:255)."""
    m = RkModel()
    m.sigma2, m.alpha, m.nu, m.tau2 = float(sigma2), float(alpha), float(nu), float(tau2)
    n = half_integer_order(nu)
    m.half_n = -1 if n is None else n
    if n is not None:
        for i in range(n + 1):
            m.half_coef[i] = math.factorial(n + i) / (math.factorial(i) * math.factorial(n - i))
        m.half_pref = math.factorial(n) / math.factorial(2 * n)
    nl = int(nu + 0.5)
    mu = nu - nl
    m.nl, m.mu = nl, mu
    gampl = 1.0 / math.gamma(1.0 + mu)
    gammi = 1.0 / math.gamma(1.0 - mu)
    m.temme_gampl, m.temme_gammi = gampl, gammi
    m.temme_gam1 = -_EULER if abs(mu) < 1.0e-6 else (gammi - gampl) / (2.0 * mu)
    m.temme_gam2 = 0.5 * (gammi + gampl)
    pimu = math.pi * mu
    m.temme_fact = 1.0 if abs(pimu) < 1.0e-12 else pimu / math.sin(pimu)
    m.gamma_nu = math.gamma(nu)
    return m


def stream_ptr(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return C.c_void_p(s.cuda_stream)


def ptr(t):
    """Address of a torch tensor or numpy array (contiguous)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return C.c_void_p(t.data_ptr())
    return C.c_void_p(t.ctypes.data)
