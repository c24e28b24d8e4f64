"""Run a few predicts of one config (for ncu captures): python tools/profile_predict.py cfg3 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import workloads

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
wl = workloads.CONFIGS[name]()
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
st = pk.build_setup(model, grid, wl.L, wl.obs)
rng = np.random.default_rng(0)
c = torch.as_tensor(rng.normal(size=wl.obs.shape[0]), device="cuda")
X = wl.X if wl.X is not None else np.ones((wl.obs.shape[0], 1))
beta = torch.as_tensor(np.ones(X.shape[1]), device="cuda")
xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
xd = None if xg is None else torch.as_tensor(xg, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(reps):
    flush.zero_()
    out = pk.predict_rapid(st, c, beta, xd)
torch.cuda.synchronize()
print("ok", name, float(out.abs().max()))
