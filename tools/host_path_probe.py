"""Host-buffer predict timing under RK_HOST_CHUNKS / RK_HOST_GRAPH settings (one per process)."""
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

case = bench.build_predict_case(pk, workloads.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg2"](), c_variants=1)
st = case["setup"]
m1, m2 = st.grid.interior_dims
p = len(case["beta"])
lib = N.load()
ch = torch.from_numpy(np.ascontiguousarray(case["cs"][0])).pin_memory().numpy()
xh = torch.from_numpy(np.ascontiguousarray(case["xg"])).pin_memory().numpy()
beta = np.ascontiguousarray(case["beta"])
oh = torch.empty((m2, m1), dtype=torch.float64).pin_memory().numpy()
sp = N.stream_ptr()
args = (st.handle, N.ptr(ch), N.ptr(beta), p, N.ptr(xh), N.ptr(oh), sp)
for _ in range(10):
    lib.rk_predict_host(*args)
ts = []
for _ in range(300):
    t0 = time.perf_counter()
    lib.rk_predict_host(*args)
    ts.append((time.perf_counter() - t0) * 1e6)
ts.sort()
print(f"chunks={os.environ.get('RK_HOST_CHUNKS', 'auto')} graph={os.environ.get('RK_HOST_GRAPH', '1')}: "
      f"median {ts[150]:.1f} us  p10 {ts[30]:.1f}  p90 {ts[270]:.1f}")
