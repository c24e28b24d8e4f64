"""cfg predict time with L2 flushed before each step (the bench's protocol), many steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
case = bench.build_predict_case(pk, workloads.CONFIGS[name]())
flush = bench.L2Flush()
ms, _, _ = bench.time_predict_device(pk, case, 200, 5, flush)
ms = sorted(ms)
print(f"{name} flushed: mean {1e3 * sum(ms) / len(ms):.2f} us median {1e3 * ms[len(ms) // 2]:.2f} us")
