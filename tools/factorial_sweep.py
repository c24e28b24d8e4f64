"""BASELINE configs[4]: the nu x L x grid factorial (36 cells, n = 50000) timed on one B200.

Per cell: T_predict = K1 (weights kernel) + T_apply (predict_rapid), device resident, L2 flushed
before every step, CUDA events on the launching stream (bench.time_predict_device); K1 and the
three passes alone; grid points/s; the step's algorithmic bytes and FFT + K1 flops against the
HBM / DFMA roofs.  The n x n fit is shared by the cells of one nu (the observations do not
change) and is setup, not timed.

python tools/factorial_sweep.py [out.json]      (~2 min on a B200)
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402


def main():
    import torch
    out_path = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "factorial_sweep.json")
    flush = bench.L2Flush()
    peaks, kind = bench._peaks()
    rows = []
    for nu in (0.5, 1.5, 2.5):
        wl0 = workloads.cfg5(nu=nu, L=1, m=256)
        model = pk.CovarianceModel(wl0.sigma2, wl0.alpha, wl0.nu, wl0.tau2)
        t0 = time.perf_counter()
        f = pk.fit(model, wl0.obs, wl0.z)
        torch.cuda.synchronize()
        t_fit = time.perf_counter() - t0
        c0 = np.asarray(f.c)
        rng = np.random.default_rng(123)
        cs = [c0, c0 * 1.001 + 1e-3 * rng.normal(size=c0.shape)]
        for m in (256, 1024, 4096):
            for L in (1, 2, 3, 4):
                wl = workloads.cfg5(nu=nu, L=L, m=m)
                t0 = time.perf_counter()
                grid = pk.build_padded_grid(wl.domain, wl.dims, L, wl.obs)
                st = pk.build_setup(model, grid, L, wl.obs)
                torch.cuda.synchronize()
                t_setup = time.perf_counter() - t0
                case = dict(model=model, fit=f, grid=grid, setup=st, xg=None, cs=cs,
                            beta=np.asarray(f.beta_hat))
                ms, _, _ = bench.time_predict_device(pk, case, 20, 5, flush, with_k1=True)
                ma, _, _ = bench.time_predict_device(pk, case, 20, 5, flush, with_k1=False)
                pm, pb = bench.profile_passes(pk, case, 10, flush)
                k1 = bench.weights_k1(case, reps=10)
                step = statistics.median(ms)
                rf = bench.predict_roofline(case, pm, pb, k1, step, peaks, kind, "sweep")
                rows.append({
                    "nu": nu, "L": L, "grid": m, "embed": list(st.embed_dims), "padded": list(grid.total_dims),
                    "step_ms": round(step, 5), "apply_ms": round(statistics.median(ma), 5), "k1_ms": k1["ms"],
                    "points_per_s": round(m * m / (step * 1e-3), 1),
                    "apply_points_per_s": round(m * m / (statistics.median(ma) * 1e-3), 1),
                    "k1_fp64_tflops": k1["fp64_tflops"],
                    "passes_ms": {k: v["ms"] for k, v in rf["passes"].items()},
                    "step_roofline": {k: rf["step"][k] for k in
                                      ("bytes", "flops", "hbm_roof_ms", "fp64_roof_ms", "binding",
                                       "frac_of_binding_roof")},
                    "setup_s": round(t_setup, 3),
                })
                print(json.dumps(rows[-1]), flush=True)
                del case, st
                torch.cuda.empty_cache()
        del f
        torch.cuda.empty_cache()
        print(f"# nu={nu}: fit {t_fit:.2f} s (setup, shared by its 12 cells)", flush=True)
    doc = {
        "what": "BASELINE configs[4] factorial: n = 50000 U[0,1]^2, range 0.05, sigma2 1, tau2 0.01; "
                "T_predict = K1 + predict_rapid, device resident, L2 flushed per step, median of 20 steps",
        "gpu": torch.cuda.get_device_name(0), "peaks": peaks, "peaks_kind": kind,
        "fp64_peak_tflops": bench.FP64_TFLOPS_MEASURED, "cells": rows,
    }
    os.makedirs(os.path.dirname(out_path), exist_ok=True)
    with open(out_path, "w") as fh:
        json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
