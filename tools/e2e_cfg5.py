"""e2e (host buffers through the public API) of the headline step, for host-path switches
(RK_HOST_ZEROCOPY, RK_HOST_CHUNKS): python tools/e2e_cfg5.py [steps]"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
flush = bench.L2Flush()
wl = workloads.cfg5(**bench.HEADLINE)
case = bench.build_predict_case(pk, wl, 1, 0, c_variants=2)
ms, h2d, d2h = bench.time_predict_e2e(pk, case, steps, 3, flush)
N = wl.dims[0] * wl.dims[1]
med = statistics.median(ms)
print(f"e2e {os.environ.get('RK_HOST_ZEROCOPY', 'd')}/{os.environ.get('RK_HOST_CHUNKS', 'd')}: median {med:.3f} ms, "
      f"{N / (med * 1e-3) / 1e9:.2f} G points/s, mean {statistics.mean(ms):.3f} ms")
