"""K1 (weights kernel) time per configuration and kernel variant (RK_WEIGHTS_OB), each variant in
its own process (the switch is read once).  Prints one JSON line per (config, variant)."""
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
for ob in ("0", "2", "4"):
    r = subprocess.run([sys.executable, "-c", CODE], env=dict(os.environ, RK_WEIGHTS_OB=ob), capture_output=True, text=True)
    res["OB" + ob] = json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else r.stderr[-500:]
    print(ob, res["OB" + ob], flush=True)
json.dump(res, open("gpurun_out/weights_sweep.json", "w"), indent=1)
