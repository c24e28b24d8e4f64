"""Steady-state host-buffer predict time (cfg2), many calls: python tools/e2e_ab.py"""
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
ms, _, _ = bench.time_predict_e2e(pk, case, 300, 5, flush)
ms = sorted(ms)
print(f"RK_HOST_ZEROCOPY={os.environ.get('RK_HOST_ZEROCOPY', '1')}: mean {1e3 * sum(ms) / len(ms):.1f} us, "
      f"median {1e3 * ms[len(ms) // 2]:.1f}, p10 {1e3 * ms[len(ms) // 10]:.1f}, p90 {1e3 * ms[9 * len(ms) // 10]:.1f}")
