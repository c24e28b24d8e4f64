"""Per-CTA phase timeline of the three predict kernels (needs a RK_PHASE_TIMING=1 build:
RK_PHASE_TIMING=1 python -c 'from paper_2605_29284_b200 import build; build.build(force=True)').

python tools/phase_probe.py cfg2     -> for warm and cold-L2 runs: CTA start spread and the
median / max time (us, from the CTA's own start) at which each phase ended."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import _native as N  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

PHASES = {"row_fwd": ["gather loads", "node sums", "fft", "split+store"],
          "col": ["T loaded", "fft", "x spectrum + ifft", "bulk store"],
          "row_inv": ["U gathered", "operands ready", "ifft", "epilogue"]}
name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
case = bench.build_predict_case(pk, workloads.CONFIGS[name](), c_variants=1)
st = case["setup"]
cd = torch.as_tensor(case["cs"][0], device="cuda")
bd = torch.as_tensor(case["beta"], device="cuda")
xd = None if case["xg"] is None else torch.as_tensor(case["xg"], device="cuda").contiguous()
m1, m2 = st.grid.interior_dims
out = torch.empty((m2, m1), dtype=torch.float64, device="cuda")
lib = N.load()
big = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for mode in ["warm", "cold"]:
    for _ in range(5):
        pk.predict_rapid(st, cd, bd, xd, out=out)
    torch.cuda.synchronize()
    if mode == "cold":
        big.zero_()
    pk.predict_rapid(st, cd, bd, xd, out=out)
    torch.cuda.synchronize()
    buf = np.zeros(3 * 4096 * 8, dtype=np.uint64)
    N.check(lib.rk_phase_timestamps(buf.ctypes.data_as(C.c_void_p)))
    b = buf.reshape(3, 4096, 8).astype(np.int64)
    t0 = None
    for k, nm in enumerate(PHASES):
        v = b[k][b[k][:, 0] > 0]
        if t0 is None:
            t0 = v[:, 0].min()
        rel = (v - t0) / 1000.0
        ph = " | ".join(f"{PHASES[nm][p - 1]} {np.median(rel[:, p] - rel[:, 0]):.2f}/{(rel[:, p] - rel[:, 0]).max():.2f}"
                        for p in range(1, 5))
        if nm == "col" and (v[:, 5] > 0).all():
            print(f"   col: spectrum multiply done at {np.median((v[:, 5] - v[:, 0]) / 1000.0):.2f} us (median)")
        print(f"{mode} {nm}: {len(v)} CTAs start {rel[:, 0].min():.2f}..{rel[:, 0].max():.2f} us; {ph}; "
              f"last end {rel[:, 4].max():.2f} us")
