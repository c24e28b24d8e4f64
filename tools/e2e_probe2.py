"""Which host-path calls are slow?  Per-call times in order for the bench's e2e loop."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

case = bench.build_predict_case(pk, workloads.cfg2())
flush = bench.L2Flush()
ms, _, _ = bench.time_predict_e2e(pk, case, 40, 5, flush)
print("order:", [round(1e3 * m) for m in ms])
st = case["setup"]
m1, m2 = st.grid.interior_dims
ch = [torch.from_numpy(np.ascontiguousarray(c)).pin_memory().numpy() for c in case["cs"]]
for i, c in enumerate(ch):
    print(i, c.ctypes.data % 4096, torch.from_numpy(c).is_pinned())
xg = torch.from_numpy(np.ascontiguousarray(case["xg"])).pin_memory().numpy()
out = torch.empty((m2, m1), dtype=torch.float64).pin_memory().numpy()
print("xg pinned", torch.from_numpy(xg).is_pinned(), "out pinned", torch.from_numpy(out).is_pinned())
beta = np.ascontiguousarray(case["beta"])
for k in range(12):
    pk.predict_rapid(st, ch[k % 4], beta, xg, out=out)
ts = []
for k in range(24):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pk.predict_rapid(st, ch[k % 4], beta, xg, out=out)
    ts.append(round((time.perf_counter() - t0) * 1e6))
print("no flush:", ts)
ts = []
for k in range(24):
    flush()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pk.predict_rapid(st, ch[k % 4], beta, xg, out=out)
    ts.append(round((time.perf_counter() - t0) * 1e6))
print("flush:", ts)
