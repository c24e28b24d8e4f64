"""Per-pass predict times of factorial cells (BASELINE configs[4]) for same-box A/B runs:
python tools/cell_times.py ROOT nu:L:m [nu:L:m ...]    (ROOT: the tree to import, '.' or ab/NAME)"""
import json
import os
import sys

root = os.path.abspath(sys.argv[1])
sys.path.insert(0, root)
os.chdir(root)
import numpy as np  # noqa: E402

import bench  # noqa: E402
import paper_2605_29284_b200 as pk  # noqa: E402
from paper_2605_29284_b200 import workloads  # noqa: E402

flush = bench.L2Flush()
for spec in sys.argv[2:]:
    nu, L, m = spec.split(":")
    wl = workloads.cfg5(nu=float(nu), L=int(L), m=int(m))
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = pk.build_setup(model, grid, wl.L, wl.obs)
    rng = np.random.default_rng(1)
    c = rng.normal(size=wl.obs.shape[0])
    case = dict(model=model, grid=grid, setup=st, xg=None, cs=[c, 1.01 * c], beta=np.array([0.5]))
    ma, _, _ = bench.time_predict_device(pk, case, 30, 5, flush, with_k1=False)
    pm, _ = bench.profile_passes(pk, case, 10, flush)
    print(spec, "embed", list(st.embed_dims), "apply ms", round(float(np.median(ma)), 4),
          "passes ms", [round(float(x), 4) for x in pm], flush=True)
