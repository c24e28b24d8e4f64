"""K1 time against n for L = 2, 3 under the current RK_WEIGHTS_* switches (threshold of the
tensor-core solve): python tools/k1_l2_probe.py"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import _native as N, workloads
out = {}
for L in (2, 3):
    for n in (1024, 2048, 4096, 8192, 16384, 50000):
        wl = workloads.cfg5(nu=1.5, L=L, m=512, n=n)
        model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
        st = pk.build_setup(model, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
        ms = C.c_float(0)
        N.call("rk_setup_time_weights", st.handle, N.stream_ptr(), 50, C.byref(ms))
        out[f"L{L}_n{n}"] = round(ms.value * 1e3, 2)
print(json.dumps(out))
