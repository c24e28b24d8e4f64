"""Does the host fall behind the GPU between the L2 flush and the timed predict?

python tools/bubble_probe.py [cfg2]   -> per-step CUDA-event time of a flushed predict with and
without a device-side spin after the flush (the spin keeps the stream busy until the host
has enqueued the start event and the predict graph, so any host-submission gap is hidden)."""
import os
import statistics
import sys

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
for spin in [0, 20000, 100000, 0, 100000]:
    for _ in range(10):
        pk.predict_rapid(st, cd, bd, xd, out=out)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(100)]
    for a, b in ev:
        flush()
        if spin:
            torch.cuda._sleep(spin)
        a.record()
        pk.predict_rapid(st, cd, bd, xd, out=out)
        b.record()
    torch.cuda.synchronize()
    ms = [a.elapsed_time(b) * 1000 for a, b in ev]
    print(f"{name} spin {spin:6d} cycles: median {statistics.median(ms):.2f} us, min {min(ms):.2f}, "
          f"p90 {sorted(ms)[89]:.2f}")
