"""Time the refit's DMMA triangular panel products (rk_refit_profile) at n, S."""
import ctypes as C
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import _native as N
from paper_2605_29284_b200 import workloads

out = {}
for name, wl, S in (("cfg4", workloads.cfg4(), [64, 256, 1024]), ("cfg5", workloads.cfg5(nu=1.5, L=4, m=256), [64, 128])):
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    f = pk.fit(model, wl.obs, wl.z)
    f.prepare_refit()
    n = wl.obs.shape[0]
    for s in S:
        ms = (C.c_float * 2)()
        N.call("rk_refit_profile", f.handle, s, 3, N.stream_ptr(), C.byref(ms))
        fl = n * n * s   # one triangular product: n(n+1)/2 multiply-adds per column
        out[f"{name}_n{n}_S{s}"] = {"ms": [ms[0], ms[1]], "TF/s": [fl / (m * 1e-3) / 1e12 for m in ms]}
        print(name, n, s, out[f"{name}_n{n}_S{s}"], flush=True)
    del f
    torch.cuda.empty_cache()
json.dump(out, open("gpurun_out/refit_probe.json", "w"), indent=1)
