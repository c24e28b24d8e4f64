"""Probe small-config predict latency: back-to-back vs L2-flushed steps, with SM clock samples."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
case = bench.build_predict_case(pk, workloads.CONFIGS[name](), c_variants=1)
st = case["setup"]
cd = torch.as_tensor(case["cs"][0], device="cuda")
bd = torch.as_tensor(case["beta"], device="cuda")
xd = None if case["xg"] is None else torch.as_tensor(case["xg"], device="cuda").contiguous()
m1, m2 = st.grid.interior_dims
out = torch.empty((m2, m1), dtype=torch.float64, device="cuda")
flush = bench.L2Flush()
for _ in range(10):
    pk.predict_rapid(st, cd, bd, xd, out=out)
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits", "-lms", "50"],
                       stdout=subprocess.PIPE, text=True)
time.sleep(0.3)
for mode in ["b2b", "b2b_long", "flushed"]:
    n = 200 if mode != "b2b_long" else 5000
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if mode.startswith("b2b"):
        e0.record()
        for _ in range(n):
            pk.predict_rapid(st, cd, bd, xd, out=out)
        e1.record()
        torch.cuda.synchronize()
        print(mode, "us/predict", round(e0.elapsed_time(e1) * 1e3 / n, 2))
    else:
        tot = 0.0
        for _ in range(n):
            flush()
            e0.record()
            pk.predict_rapid(st, cd, bd, xd, out=out)
            e1.record()
            torch.cuda.synchronize()
            tot += e0.elapsed_time(e1)
        print(mode, "us/predict", round(tot * 1e3 / n, 2))
t0 = time.perf_counter()
for _ in range(2000):
    pk.predict_rapid(st, cd, bd, xd, out=out)
torch.cuda.synchronize()
print("host-side us/call (includes GPU if GPU-bound)", round((time.perf_counter() - t0) * 1e6 / 2000, 2))
smi.terminate()
clk = [int(x) for x in smi.stdout.read().split() if x.strip().isdigit()]
print("sm clocks sampled:", clk[:5], "...", "median", sorted(clk)[len(clk) // 2] if clk else None)
