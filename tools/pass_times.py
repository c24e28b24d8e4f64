"""Per-kernel predict times + GB/s for several configs (quick perf check):
python tools/pass_times.py cfg2 cfg3 cfg5      (cfg5 = the headline: 4096^2, L = 4, nu = 2.5)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

flush = bench.L2Flush()
peaks, kind = bench._peaks()
for name in sys.argv[1:] or ["cfg2", "cfg3"]:
    wl = workloads.cfg5(**bench.HEADLINE) if name == "cfg5" else workloads.CONFIGS[name]()
    case = bench.build_predict_case(pk, wl, 1, 0, c_variants=2)
    ms, _, _ = bench.time_predict_device(pk, case, 20, 3, flush, with_k1=True)
    ma, _, _ = bench.time_predict_device(pk, case, 20, 3, flush, with_k1=False)
    pm, pb = bench.profile_passes(pk, case, 10, flush)
    k1 = bench.weights_k1(case, reps=10)
    rf = bench.predict_roofline(case, pm, pb, k1, sum(ms) / len(ms), peaks, kind, name)
    print(name, "step ms", round(sum(ms) / len(ms), 4), "apply ms", round(sum(ma) / len(ma), 4), "K1 ms", k1["ms"],
          json.dumps(rf["passes"]), flush=True)
    del case
