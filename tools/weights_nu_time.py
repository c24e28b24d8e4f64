"""K1 timing for a Bessel-path smoothness: python tools/weights_nu_time.py -> cfg4 shapes with nu = 1.0"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import _native as N, workloads  # noqa: E402

wl = workloads.cfg4()
for nu in (1.0, 1.5):
    m = pk.CovarianceModel(wl.sigma2, wl.alpha, nu, wl.tau2)
    st = pk.build_setup(m, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
    ms = C.c_float(0)
    N.call("rk_setup_time_weights", st.handle, N.stream_ptr(), 20, C.byref(ms))
    print(f"cfg4 shapes, nu={nu}: {ms.value * 1000:.2f} us")
