"""cfg5 probe (n=50000): GPU exact fit, setup, predict timing and oracle parity at the
large grids, plus a short CS run.  python tools/cfg5_probe.py [m] [nu] [L] [--cs R] [--no-oracle]"""
import argparse
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("m", type=int, nargs="?", default=4096)
ap.add_argument("nu", type=float, nargs="?", default=1.5)
ap.add_argument("L", type=int, nargs="?", default=4)
ap.add_argument("--cs", type=int, default=0)
ap.add_argument("--cs-batch", type=int, default=0)
ap.add_argument("--no-oracle", action="store_true")
a = ap.parse_args()
print(subprocess.run(["free", "-g"], capture_output=True, text=True).stdout.splitlines()[1])
wl = workloads.cfg5(nu=a.nu, L=a.L, m=a.m)
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
t0 = time.perf_counter()
f = pk.fit(model, wl.obs, wl.z, wl.X)
torch.cuda.synchronize()
print(f"fit n={wl.obs.shape[0]}: {time.perf_counter() - t0:.2f} s, beta {np.asarray(f.beta_hat)}")
t0 = time.perf_counter()
grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
st = pk.build_setup(model, grid, wl.L, wl.obs)
torch.cuda.synchronize()
print(f"setup {wl.dims} L={wl.L} nu={wl.nu}: {time.perf_counter() - t0:.3f} s, padded {grid.total_dims}, "
      f"embed {st.embed_dims}")
flush = bench.L2Flush()
case = bench.build_predict_case(pk, wl, c_variants=2)
ms, _, out = bench.time_predict_device(pk, case, 10, 3, flush)
pm, pb = bench.profile_passes(pk, case, 3, flush)
peaks, kind = bench._peaks()
rf = bench.roofline_obj(case, pm, pb, peaks, kind)
N = wl.dims[0] * wl.dims[1]
tm = sum(ms) / len(ms)
print(f"predict {tm:.3f} ms = {N / tm / 1e6:.3f} G points/s; passes {rf['passes']}")
print(f"torch max allocated {torch.cuda.max_memory_allocated() / 2**30:.1f} GiB")
if not a.no_oracle:
    from oracle import rk_oracle as ro
    t0 = time.perf_counter()
    om = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    og = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
    ost = ro.rapid_setup(om, og, wl.L, wl.obs)
    assert np.array_equal(ost.indices[:, 0], case["setup"].neighbor_indices[:, 0])
    ref = ro.predict(ost, case["cs"][0], case["beta"], None)
    got = pk.predict_rapid(case["setup"], case["cs"][0], case["beta"], None)
    print(f"oracle parity max rel {np.abs(got - ref).max() / np.abs(ref).max():.3e} "
          f"(oracle {time.perf_counter() - t0:.1f} s)")
if a.cs:
    t0 = time.perf_counter()
    kw = {} if not a.cs_batch else {"batch": a.cs_batch}
    e = pk.generate_ensemble(f, case["setup"], a.cs, 0, keep_draws=False, **kw)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    e = pk.generate_ensemble(f, case["setup"], a.cs, 0, keep_draws=False, **kw)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    se = np.asarray(e.empirical_se)
    print(f"CS R={a.cs}: first {t1 - t0:.2f} s, second {t2 - t1:.2f} s = {(t2 - t1) / a.cs * 1e3:.2f} ms/realization; "
          f"se mean {se.mean():.5f}")
