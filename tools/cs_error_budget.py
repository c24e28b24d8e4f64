"""Where does a conditional draw's deviation from the oracle come from?  cfg4, one realization:
relative (to max|ref|) errors of each stage, GPU stage fed with the ORACLE's input."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2605_29284_b200 as pk
from oracle import rk_oracle as ro
from paper_2605_29284_b200 import workloads
from paper_2605_29284_b200.simulate import draw_seed


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / np.abs(b).max())


wl = workloads.cfg4()
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
f = pk.fit(model, wl.obs, wl.z)
grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
st = pk.build_setup(model, grid, wl.L, wl.obs)
om = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
og = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
ost = ro.rapid_setup(om, og, wl.L, wl.obs)
ofit = ro.Fit(om, f.obs_locs, f.X, f.chol_M, np.asarray(f.beta_hat), np.asarray(f.c))
root = ro.embedding_root(om, og)
out = {}
for j in range(3):
    s = ro.sub_seed(0, j)
    g_ref = ro.uncond_field(om, og, ro.sub_seed(s, 101), root)
    g_gpu = pk.sim_unconditional_grid(model, st, draw_seed(s, 101))
    zs_ref = ro.obs_local(om, ost, g_ref, ro.sub_seed(s, 202))
    zs_gpu = pk.sim_obs_local(model, st, g_ref, draw_seed(s, 202))
    b_ref, c_ref = ro.refit(ofit, zs_ref)
    b_gpu, c_gpu = pk.refit_coefficients(f, zs_ref)
    p_ref = ro.predict(ost, c_ref, b_ref)
    p_gpu = pk.predict_rapid(st, c_ref, b_ref)
    p_gpu_c = pk.predict_rapid(st, c_gpu, b_gpu)
    d_ref = ro.cond_draw(ofit, ost, s, None, None, root)
    d_gpu = pk.conditional_draw(f, st, s)
    r = {"uncond_g": rel(g_gpu, g_ref), "obs_local_z": rel(zs_gpu, zs_ref), "refit_beta": rel(b_gpu, b_ref),
         "refit_c": rel(c_gpu, c_ref), "predict_same_c": rel(p_gpu, p_ref), "predict_gpu_c": rel(p_gpu_c, p_ref),
         "draw": rel(d_gpu, d_ref), "max_draw": float(np.abs(d_ref).max()),
         "abs_draw_err": float(np.abs(d_gpu - d_ref).max()),
         "abs_pred_err_from_refit": float(np.abs(p_gpu_c - p_gpu).max()),
         "abs_pred_err_same_c": float(np.abs(p_gpu - p_ref).max()),
         "abs_g_err": float(np.abs(g_gpu - g_ref).max())}
    out[j] = r
    print(j, json.dumps(r), flush=True)
json.dump(out, open("gpurun_out/cs_error_budget.json", "w"), indent=1)
