"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): python tools/sanitize_cases.py {predict,split,weights,cs}"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2605_29284_b200 as pk

case = sys.argv[1] if len(sys.argv) > 1 else "predict"
rng = np.random.default_rng(7)
if case == "predict":    # spread / wide plans, fused gather, plan-block TMA, host + device paths
    for L, dims, nu in ((2, (100, 100), 1.5), (3, (350, 350), 1.0)):
        obs = rng.uniform(0, 1, size=(1200, 2))
        m = pk.CovarianceModel(1.0, 8.0, nu, 0.05)
        st = pk.build_setup(m, pk.build_padded_grid((0, 1, 0, 1), dims, L, obs), L, obs)
        f = pk.predict_rapid(st, rng.normal(size=1200), np.array([0.5]))
        print(case, L, dims, float(np.abs(f).max()))
elif case == "split":    # split-length passes (torus > 4608) incl. both column-pass variants
    obs = rng.uniform(0, 1, size=(3000, 2))
    m = pk.CovarianceModel(1.0, 12.0, 1.5, 0.01)
    st = pk.build_setup(m, pk.build_padded_grid((0, 1, 0, 1), (2600, 2500), 2, obs), 2, obs)
    f = pk.predict_rapid(st, rng.normal(size=3000), np.array([0.5]))
    print(case, st.embed_dims, float(np.abs(f).max()))
elif case == "weights":  # K1: tensor-core blocked solve (L = 3, 4) and the substitution kernels
    for L in (1, 2, 3, 4):
        obs = rng.uniform(0.05, 0.95, size=(2500, 2))
        m = pk.CovarianceModel(1.0, 9.0, 2.5 if L == 4 else 1.0)
        st = pk.build_setup(m, pk.build_padded_grid((0, 1, 0, 1), (64, 60), L, obs), L, obs)
        print(case, L, float(np.abs(st.weights).max()))
elif case == "cs":       # fit, refit, unconditional fields (row generator + column pass), ensemble
    obs = rng.uniform(0, 1, size=(400, 2))
    z = 1.0 + np.sin(5 * obs[:, 0]) + 0.1 * rng.normal(size=400)
    m = pk.CovarianceModel(1.0, 10.0, 1.5, 0.02)
    f = pk.fit(m, obs, z)
    st = pk.build_setup(m, pk.build_padded_grid((0, 1, 0, 1), (96, 80), 3, obs), 3, obs)
    ens = pk.generate_ensemble(f, st, 6, 3)
    print(case, float(np.mean(ens.empirical_se)))
