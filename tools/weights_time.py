import sys, os, ctypes as C
sys.path.insert(0, os.getcwd())
import bench, paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import workloads, _native as N
for name in sys.argv[1].split(","):
    wl = workloads.CONFIGS[name]()
    m = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    st = pk.build_setup(m, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
    ms = C.c_float(0)
    N.call("rk_setup_time_weights", st.handle, N.stream_ptr(), 20, C.byref(ms))
    print(name, os.environ.get("RK_WEIGHTS_GENERIC", "0"), f"{ms.value*1000:.2f} us")
