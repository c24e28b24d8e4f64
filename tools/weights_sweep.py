"""K1 (weights kernel) time per configuration and kernel variant (RK_WEIGHTS_MMA / RK_WEIGHTS_OB),
each variant in its own process (the switches are read once).  Prints one JSON line per variant."""
import json
import os
import subprocess
import sys

CODE = r'''
import ctypes as C, json, sys
sys.path.insert(0, ".")
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import _native as N, workloads
out = {}
for name, wl in (("cfg2", workloads.cfg2()), ("cfg3", workloads.cfg3()), ("cfg4", workloads.cfg4()),
                 ("cfg5_nu2.5_L4", workloads.cfg5(nu=2.5, L=4, m=1024)), ("cfg5_nu1.5_L3", workloads.cfg5(nu=1.5, L=3, m=1024)),
                 ("cfg5_nu0.5_L4", workloads.cfg5(nu=0.5, L=4, m=1024))):
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    st = pk.build_setup(model, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
    ms = C.c_float(0)
    N.call("rk_setup_time_weights", st.handle, N.stream_ptr(), 20, C.byref(ms))
    out[name] = round(ms.value, 5)
print(json.dumps(out))
'''
res = {}
VARIANTS = {"MMA": {"RK_WEIGHTS_MMA": "1"}, "OB0": {"RK_WEIGHTS_MMA": "0", "RK_WEIGHTS_OB": "0"},
            "OB2": {"RK_WEIGHTS_MMA": "0", "RK_WEIGHTS_OB": "2"}}
for tag, env in VARIANTS.items():
    r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, **env), capture_output=True, text=True)
    res[tag] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
    print(tag, res[tag], flush=True)
json.dump(res, open("gpurun_out/weights_sweep.json", "w"), indent=1)
