"""Run a small cfg4 ensemble slice (for ncu launch lists): python tools/cs_probe.py [R] [batch]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402
from paper_2605_29284_b200.distributed import generate_ensemble_sharded  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 64
B = int(sys.argv[2]) if len(sys.argv) > 2 else 32
wl = workloads.cfg4()
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
f = pk.fit(model, wl.obs, wl.z)
grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
st = pk.build_setup(model, grid, wl.L, wl.obs)
generate_ensemble_sharded(f, st, R, 0, batch=B)
torch.cuda.synchronize()
t0 = time.perf_counter()
ens = generate_ensemble_sharded(f, st, R, 0, batch=B)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"R={R} batch={B}: {dt * 1e3:.2f} ms, {dt / R * 1e6:.1f} us/realization, se mean {float(ens.empirical_se.mean()):.5f}")
