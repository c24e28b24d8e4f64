"""A configs[4]-CS slice (n = 50000, 4096^2, L = 4, nu = 1.5, 8748^2 torus) for timing:
python tools/cs_probe5.py [R] [batch]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402
from paper_2605_29284_b200.distributed import generate_ensemble_sharded  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 32
B = int(sys.argv[2]) if len(sys.argv) > 2 else 16
wl = workloads.cfg5(nu=1.5, L=4, m=4096)
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
f = pk.fit(model, wl.obs, wl.z)
st = pk.build_setup(model, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
f.prepare_refit()
generate_ensemble_sharded(f, st, R, 0, batch=B)
torch.cuda.synchronize()
t0 = time.perf_counter()
ens = generate_ensemble_sharded(f, st, R, 0, batch=B)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"cfg5 CS R={R} batch={B}: {dt * 1e3:.1f} ms, {dt / R * 1e3:.3f} ms/realization, se mean {float(ens.empirical_se.mean()):.6f}")
