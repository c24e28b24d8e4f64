"""Per-kernel predict times + GB/s for several configs (quick perf check): python tools/pass_times.py cfg2 cfg3"""
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
    wl = workloads.CONFIGS[name]()
    case = bench.build_predict_case(pk, wl, c_variants=2)
    ms, _, _ = bench.time_predict_device(pk, case, 20, 3, flush)
    pm, pb = bench.profile_passes(pk, case, 10, flush)
    rf = bench.roofline_obj(case, pm, pb, peaks, kind)
    print(name, "predict ms", round(sum(ms) / len(ms), 4), json.dumps(rf["passes"]))
