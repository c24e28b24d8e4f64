"""One headline predict step (K1 + predict) on cfg5 4096^2 nu=2.5 L=4 for ncu captures."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import workloads

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
wl = workloads.cfg5(nu=2.5, L=4, m=4096)
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
st = pk.build_setup(model, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
c = torch.as_tensor(np.random.default_rng(1).normal(size=wl.obs.shape[0]), device="cuda")
b = torch.tensor([1.0], device="cuda", dtype=torch.float64)
out = torch.empty((4096, 4096), dtype=torch.float64, device="cuda")
for _ in range(reps):
    pk.predict_rapid(st, c, b, out=out)
torch.cuda.synchronize()
