"""K1 alone for ncu captures: python tools/profile_weights.py [cfg] [reps] (cfg5 = 4096^2 nu=2.5 L=4)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import _native as N, workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
wl = workloads.cfg5(nu=2.5, L=4, m=1024) if name == "cfg5" else workloads.CONFIGS[name]()
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
st = pk.build_setup(model, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
ms = C.c_float(0)
N.call("rk_setup_time_weights", st.handle, N.stream_ptr(), reps, C.byref(ms))
print(name, f"{ms.value * 1000:.2f} us")
