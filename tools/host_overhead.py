"""Host-side cost breakdown of one predict call (device path and host-buffer path).

python tools/host_overhead.py [cfg2]"""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import _native as N  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402


def per_call(fn, n=2000, sync=True):
    for _ in range(20):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    if sync:
        torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e6 / n


name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
case = bench.build_predict_case(pk, workloads.CONFIGS[name](), c_variants=1)
st = case["setup"]
cd = torch.as_tensor(case["cs"][0], device="cuda")
bd = torch.as_tensor(case["beta"], device="cuda")
xd = None if case["xg"] is None else torch.as_tensor(case["xg"], device="cuda").contiguous()
m1, m2 = st.grid.interior_dims
p = int(bd.numel())
out = torch.empty((m2, m1), dtype=torch.float64, device="cuda")
lib = N.load()
sp = N.stream_ptr()
args = (st.handle, N.ptr(cd), N.ptr(bd), p, N.ptr(xd), N.ptr(out), sp)
print("n", st.n_obs, "grid", (m1, m2), "p", p)
print("stream_ptr us", round(per_call(N.stream_ptr, sync=False), 2))
print("ptr us", round(per_call(lambda: N.ptr(cd), sync=False), 2))
print("raw ctypes rk_predict_dev us", round(per_call(lambda: lib.rk_predict_dev(*args)), 2))
print("predict_rapid(device) us", round(per_call(lambda: pk.predict_rapid(st, cd, bd, xd, out=out)), 2))
g = torch.cuda.CUDAGraph()
# GPU-side time of back-to-back predicts without host gaps: 20 calls per timed burst,
# launched while the GPU is held busy by a long memset
big = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for rep in range(3):
    big.zero_()
    big.zero_()
    e0.record()
    for _ in range(20):
        lib.rk_predict_dev(*args)
    e1.record()
    torch.cuda.synchronize()
    print("gpu-side b2b us/predict (host hidden behind 2 memsets)", round(e0.elapsed_time(e1) * 1e3 / 20, 2))

# host-buffer path pieces
ch = torch.from_numpy(np.ascontiguousarray(case["cs"][0])).pin_memory().numpy()
xh = None if case["xg"] is None else torch.from_numpy(np.ascontiguousarray(case["xg"])).pin_memory().numpy()
beta = np.ascontiguousarray(case["beta"])
oh = torch.empty((m2, m1), dtype=torch.float64).pin_memory().numpy()
hargs = (st.handle, N.ptr(ch), N.ptr(beta), p, N.ptr(xh), N.ptr(oh), sp)
print("raw ctypes rk_predict_host us", round(per_call(lambda: lib.rk_predict_host(*hargs), n=300), 2))
print("predict_rapid(host) us", round(per_call(lambda: pk.predict_rapid(st, ch, beta, xh, out=oh), n=300), 2))
ct, xt, ot = torch.from_numpy(ch), (None if xh is None else torch.from_numpy(xh)), torch.from_numpy(oh)
print("bytes h2d c", ch.nbytes, "xg", 0 if xh is None else xh.nbytes, "d2h", oh.nbytes)
print("torch H2D c us", round(per_call(lambda: cd.copy_(ct, non_blocking=True), n=300), 2))
if xt is not None:
    print("torch H2D xg us", round(per_call(lambda: xd.copy_(xt, non_blocking=True), n=300), 2))
print("torch D2H out us", round(per_call(lambda: ot.copy_(out, non_blocking=True), n=300), 2))
big_h = torch.empty(64 * 1024 * 1024 // 8, dtype=torch.float64).pin_memory()
big_d = torch.empty(64 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
us = per_call(lambda: big_d.copy_(big_h, non_blocking=True), n=20)
print("torch H2D 64 MB GB/s", round(64 * 1024 * 1024 / us / 1e3, 1))
us = per_call(lambda: big_h.copy_(big_d, non_blocking=True), n=20)
print("torch D2H 64 MB GB/s", round(64 * 1024 * 1024 / us / 1e3, 1))
