import os, sys, statistics
sys.path.insert(0, os.getcwd())
import bench, paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import workloads
flush = bench.L2Flush()
for name in ("cfg2", "cfg3"):
    wl = workloads.CONFIGS[name]()
    case = bench.build_predict_case(pk, wl, 1, 0, c_variants=2)
    ms, h2d, d2h = bench.time_predict_e2e(pk, case, 100, 3, flush)
    N = wl.dims[0] * wl.dims[1]
    print(name, "e2e median", round(statistics.median(ms), 4), "ms", round(N / (statistics.median(ms) * 1e-3) / 1e9, 3), "G points/s")
