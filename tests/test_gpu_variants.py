"""Kernel variants that must agree: each run in a subprocess with its switch set, on the same
inputs, compared with the default path.

* RK_SPLIT=0: the full-length FFT passes instead of the split-length ones (for tori above the
  WIDE-plan lengths, P = 2 H with the nonzero rows / kept outputs below H): equal to 1e-13;
* RK_WEIGHTS_OB=0 / 2 (with RK_WEIGHTS_MMA=0): the one-observation-per-warp substitution
  kernels instead of the interleaved one: bitwise identical weights and fields (same
  operations, same order);
* RK_COL_PAIR=1 / 0: the split-length column pass with both halves in one CTA against the
  2-CTA cluster version: bitwise identical;
* RK_WEIGHTS_MMA=1 / 0: the FP64 tensor-core blocked solve against the substitution kernels:
  a different (backward-stable) operation order, so the weights agree to the conditioning of
  K_N and the fields to 1e-10, and the interpolation residual stays < 1e-8.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

from rk_testutil import ROOT, has_gpu, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

CODE = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2605_29284_b200 as pk
rng = np.random.default_rng(11)
n, L, dims, nu = {n}, {L}, {dims}, {nu}
obs = rng.uniform(0, 1, size=(n, 2))
model = pk.CovarianceModel(1.0, 12.0, nu, 0.01)
grid = pk.build_padded_grid((0, 1, 0, 1), dims, L, obs)
st = pk.build_setup(model, grid, L, obs)
c = rng.normal(size=n)
field = pk.predict_rapid(st, c, np.array([0.25]))
cstar = st.coefficients_to_grid(c)
conv = pk.convolve_filter(st.filter_spectrum, st.embed_dims, cstar)
np.savez({out!r}, field=field, w=st.weights, cv=st.cond_var, idx=st.neighbor_indices, conv=conv,
         embed=np.array(st.embed_dims), exe=np.array(st.exec_dims), obs=obs, h=np.array(grid.spacing),
         spec=np.asarray(st.filter_spectrum).real[:3, :3])
"""


def _run(tmp_path, tag, env_extra, **kw):
    out = str(tmp_path / f"{tag}.npz")
    code = CODE.format(root=ROOT, out=out, **kw)
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env_extra), capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(out))


@pytest.mark.parametrize("dims", [(2600, 2500), (4096, 4096)])
def test_split_length_passes_match_full_length(tmp_path, dims):
    kw = dict(n=6000, L=2, dims=dims, nu=1.5)
    a = _run(tmp_path, "split", {}, **kw)
    b = _run(tmp_path, "full", {"RK_SPLIT": "0"}, **kw)
    assert max(a["embed"]) > 4608   # a split-length torus
    assert rel_err(a["field"], b["field"]) < 1e-13
    assert rel_err(a["conv"], b["conv"]) < 1e-13


@pytest.mark.parametrize("dims", [(2600, 2500), (4096, 4096)])
def test_column_pass_one_cta_vs_cluster_bitwise(tmp_path, dims):
    """Split-length column pass: both halves in one CTA (col_pair_kernel, RK_COL_PAIR=1) vs the
    2-CTA cluster exchanging over DSMEM (col_split_kernel): same operations, bitwise equal."""
    kw = dict(n=6000, L=2, dims=dims, nu=1.5)
    a = _run(tmp_path, "pair", {"RK_COL_PAIR": "1"}, **kw)
    b = _run(tmp_path, "cluster", {"RK_COL_PAIR": "0", "RK_COL_CT": "0"}, **kw)
    assert max(a["embed"]) > 4608
    assert np.array_equal(a["field"], b["field"])
    assert np.array_equal(a["conv"], b["conv"])


@pytest.mark.parametrize("dims", [(2048, 2048), (4096, 4096)])
def test_execution_torus_matches_reference_torus(tmp_path, dims):
    """RK_EXEC_TORUS=1: along y the passes run on the shorter 2^a 3^b torus (4096 / 8192 instead
    of the reference's 4374 / 8748; the 8192 one with the split column pass folding the 6 input rows
    beyond its half), the few aliased lags corrected exactly: the predicted field equals the
    reference-torus one to 1e-12; embed_dims, filter_spectrum and convolve_filter (whole padded
    output) stay on the reference torus."""
    kw = dict(n=6000, L=2, dims=dims, nu=1.5)
    a = _run(tmp_path, "exec", {"RK_EXEC_TORUS": "1"}, **kw)
    b = _run(tmp_path, "ref", {"RK_EXEC_TORUS": "0"}, **kw)
    assert tuple(a["embed"]) == tuple(b["embed"]) and tuple(b["exe"]) == tuple(b["embed"])
    assert a["exe"][1] < a["embed"][1] and a["exe"][0] == a["embed"][0]
    assert rel_err(a["field"], b["field"]) < 1e-12
    assert np.array_equal(a["spec"], b["spec"])
    assert rel_err(a["conv"], b["conv"]) < 1e-12


@pytest.mark.parametrize("dims", [(2600, 2500), (4096, 4096)])
def test_column_pass_fused_hooks_bitwise(tmp_path, dims):
    """Split-length column pass with the odd half's twist fused into the first stage's loads and
    the spectrum product into the last forward stage's stores (RK_FUSE_PP=1) vs separate passes:
    the same arithmetic, bitwise equal."""
    kw = dict(n=6000, L=2, dims=dims, nu=1.5)
    a = _run(tmp_path, "fused", {"RK_FUSE_PP": "1"}, **kw)
    b = _run(tmp_path, "passes", {"RK_FUSE_PP": "0"}, **kw)
    assert np.array_equal(a["field"], b["field"])
    assert np.array_equal(a["conv"], b["conv"])


@pytest.mark.parametrize("dims,g", [((2600, 2500), "0"), ((4096, 4096), "0"), ((4096, 4096), "32")])
def test_column_pass_cooley_tukey_vs_stockham(tmp_path, dims, g):
    """Split-length column pass on the in-place Cooley-Tukey engine (DIF, spectrum product in
    digit-reversed order, DIT; RK_COL_CT=1, group size RK_CT_G) vs the Stockham engine: a
    different operation order, equal to 1e-13."""
    kw = dict(n=6000, L=2, dims=dims, nu=1.5)
    a = _run(tmp_path, "ct", {"RK_COL_CT": "1", "RK_CT_G": g}, **kw)
    b = _run(tmp_path, "stockham", {"RK_COL_CT": "0"}, **kw)
    assert max(a["embed"]) > 4608
    assert rel_err(a["field"], b["field"]) < 1e-13
    assert rel_err(a["conv"], b["conv"]) < 1e-13


@pytest.mark.parametrize("L,nu", [(3, 1.5), (4, 2.5), (3, 1.0)])
def test_weights_kernel_variants_bitwise(tmp_path, L, nu):
    kw = dict(n=5000, L=L, dims=(300, 280), nu=nu)
    a = _run(tmp_path, "ob4", {"RK_WEIGHTS_MMA": "0", "RK_WEIGHTS_OB": "4"}, **kw)
    for v in ("0", "2"):
        b = _run(tmp_path, "ob" + v, {"RK_WEIGHTS_MMA": "0", "RK_WEIGHTS_OB": v}, **kw)
        assert np.array_equal(a["w"], b["w"]), v
        assert np.array_equal(a["field"], b["field"]), v


@pytest.mark.parametrize("L,nu", [(2, 1.5), (3, 1.5), (3, 1.0), (4, 2.5), (4, 0.5)])
def test_weights_mma_matches_substitution(tmp_path, L, nu):
    from oracle import rk_oracle as ro
    kw = dict(n=5000, L=L, dims=(300, 280), nu=nu)
    a = _run(tmp_path, "mma", {"RK_WEIGHTS_MMA": "1"}, **kw)
    b = _run(tmp_path, "sub", {"RK_WEIGHTS_MMA": "0"}, **kw)
    assert np.array_equal(a["idx"], b["idx"])
    assert rel_err(a["field"], b["field"]) < 1e-10
    assert np.abs(a["cv"] - b["cv"]).max() < 1e-10
    # both weight sets satisfy the interpolation condition K_N w_i = k_i to the same k_i
    # (reference test_acceptance.py:98-116; the substitution kernels' residual is pinned against
    # the reference goldens in test_gpu_parity): |K_N (w_mma - w_sub)| < 1e-8
    model = ro.Model(1.0, 12.0, nu)
    hx, hy = a["h"]
    bs = 2 * L
    off = np.stack(np.meshgrid(np.arange(bs) * hx, np.arange(bs) * hy), -1).reshape(-1, 2)
    d = off[:, None, :] - off[None, :, :]
    kn = model.cov(np.hypot(d[..., 0], d[..., 1]))
    kn = 0.5 * (kn + kn.T)
    res = np.abs(kn @ (a["w"] - b["w"]).T).max()
    assert res < 1e-8, res


CFG2 = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import workloads
wl = workloads.cfg2()
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
st = pk.build_setup(model, grid, wl.L, wl.obs)
xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
c = np.random.default_rng(5).normal(size=wl.obs.shape[0])
np.save({out!r}, pk.predict_rapid(st, c, np.array([0.5, 1.0, -1.0]), xg))
"""


def test_plan_block_staging_bitwise(tmp_path):
    """Pass 1 fetching each row pair's plan by one TMA bulk copy (RK_PLAN_TMA=1, one-wave
    launches) vs the direct plan loads (0) on cfg2's clustered design: bitwise equal."""
    res = {}
    for v in ("1", "0"):
        out = str(tmp_path / f"p{v}.npy")
        r = subprocess.run([sys.executable, "-c", CFG2.format(root=ROOT, out=out)],
                           env=dict(os.environ, RK_PLAN_TMA=v), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        res[v] = np.load(out)
    assert np.array_equal(res["1"], res["0"])


def test_out_buffer_validation_and_many_streams():
    import torch
    import paper_2605_29284_b200 as pk
    from paper_2605_29284_b200.errors import DomainError
    rng = np.random.default_rng(3)
    obs = rng.uniform(0, 1, size=(200, 2))
    model = pk.CovarianceModel(1.0, 8.0, 1.5, 0.01)
    st = pk.build_setup(model, pk.build_padded_grid((0, 1, 0, 1), (40, 30), 2, obs), 2, obs)
    c = torch.as_tensor(rng.normal(size=200), device="cuda")
    ref = pk.predict_rapid(st, c, np.array([1.0]))
    for bad in (torch.empty((30, 40), dtype=torch.float32, device="cuda"),
                torch.empty((40, 30), dtype=torch.float64, device="cuda"),
                torch.empty((30, 80), dtype=torch.float64, device="cuda")[:, ::2]):
        with pytest.raises(DomainError):
            pk.predict_rapid(st, c, np.array([1.0]), out=bad)
    with pytest.raises(DomainError):
        pk.predict_rapid(st, c.cpu().numpy(), np.array([1.0]), out=np.empty((30, 40), dtype=np.float32))
    # float32 / strided beta on the device is converted, not misread
    b32 = torch.tensor([1.0, 7.0], dtype=torch.float32, device="cuda")[:1]
    assert torch.equal(pk.predict_rapid(st, c, b32), ref)
    # more streams than the workspace cap (8): oldest workspaces are evicted, results unchanged
    for k in range(12):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            out = pk.predict_rapid(st, c, torch.tensor([1.0], dtype=torch.float64, device="cuda"))
        s.synchronize()
        assert torch.equal(out, ref), k


def test_host_path_large_field_block_copies_bitwise():
    """Host-buffer predict of a field >= 16 MB (device staging, pass 3 in 4 row blocks with their
    device -> host copies on the side stream, captured into a graph from the second call) and of
    a small one (zero-copy pass 3): bitwise equal to the device-resident path, and to pageable
    buffers, on repeated calls (graph replay)."""
    import torch
    import paper_2605_29284_b200 as pk
    rng = np.random.default_rng(5)
    for dims, n in (((1600, 1500), 3000), ((120, 100), 400)):
        obs = rng.uniform(0, 1, size=(n, 2))
        model = pk.CovarianceModel(1.0, 10.0, 1.5, 0.01)
        st = pk.build_setup(model, pk.build_padded_grid((0, 1, 0, 1), dims, 2, obs), 2, obs)
        c = rng.normal(size=n)
        beta = np.array([0.5])
        ref = pk.predict_rapid(st, torch.as_tensor(c, device="cuda"), torch.as_tensor(beta, device="cuda")).cpu().numpy()
        ch = torch.from_numpy(c).pin_memory().numpy()
        out = torch.empty((dims[1], dims[0]), dtype=torch.float64).pin_memory().numpy()
        for _ in range(3):   # direct, captured, replayed
            out[:] = np.nan
            pk.predict_rapid(st, ch, beta, out=out)
            assert np.array_equal(out, ref), dims
        assert np.array_equal(pk.predict_rapid(st, c, beta), ref), dims


@pytest.mark.parametrize("dims,L", [((115, 118), 2),    # torus 243 = 3 9^2: radix-3 stage, three butterflies per thread
                                    ((124, 120), 2),    # 256 / 243
                                    ((124, 126), 1),    # 256 = 8 8 4: swizzled radix-8 pair
                                    ((250, 254), 1),    # 512 = 8^3
                                    ((200, 230), 2),    # 432 = 6 9 8 and 486 = 6 9 9: swizzled radix-6 / radix-9 pair
                                    ((180, 100), 3),    # 384 = 6 8 8 and 216 = 6 9 4
                                    ((1000, 990), 1)])  # 2048 = 8 8 8 4
def test_wide_plans_match_normal_plans(tmp_path, dims, L):
    """The WIDE FFT plans (64-register kernels: swizzled first stage pairs, fft_kmax_wide
    butterflies per thread) forced on tori of every first-stage family (RK_WIDE=3) against the
    normal plans (RK_WIDE=0): the same stage arithmetic in a different thread mapping and a
    different shared-memory layout between the first two stages -- bitwise identical fields."""
    kw = dict(n=300, L=L, dims=dims, nu=1.5)
    a = _run(tmp_path, "wide", {"RK_WIDE": "3"}, **kw)
    b = _run(tmp_path, "normal", {"RK_WIDE": "0"}, **kw)
    assert np.array_equal(a["field"], b["field"])
    assert np.array_equal(a["conv"], b["conv"])


CS_CODE = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200.simulate import embedding_dims
rng = np.random.default_rng(5)
obs = rng.uniform(0, 1, size=(50, 2))
model = pk.CovarianceModel(1.0, {alpha}, {nu}, 0.01)
grid = pk.build_padded_grid((0, 1, 0, 1), {dims}, {L}, obs)
fields = [pk.sim_unconditional_grid(model, grid, seed) for seed in (3, 2 ** 63 + 5)]
np.savez({out!r}, f0=fields[0], f1=fields[1], emb=np.array(embedding_dims(model, grid)[:2]))
"""


@pytest.mark.parametrize("dims,L,nu,alpha", [((2400, 40), 1, 1.5, 40.0),     # row torus 5184 = 2 x 2592
                                             ((4096, 24), 2, 0.5, 60.0)])    # 8748 = 2 x 4374 (configs[4])
def test_cs_row_generator_cluster_pair_bitwise(tmp_path, dims, L, nu, alpha):
    """Split-length CS row pass with one half line per CTA of a 2-CTA cluster (RK_CS_PAIR=1, the
    Philox groups dealt to both CTAs, the other parity's elements sent over DSMEM) against the
    one-CTA kernel (RK_CS_PAIR=0): bitwise identical unconditional fields."""
    outs = []
    for v in ("1", "0"):
        out = str(tmp_path / f"cs{v}.npz")
        code = CS_CODE.format(root=ROOT, out=out, dims=dims, L=L, nu=nu, alpha=alpha)
        r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, RK_CS_PAIR=v), capture_output=True,
                           text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        outs.append(dict(np.load(out)))
    assert outs[0]["emb"][0] > 4608, outs[0]["emb"]
    assert np.array_equal(outs[0]["f0"], outs[1]["f0"])
    assert np.array_equal(outs[0]["f1"], outs[1]["f1"])
    assert np.all(np.isfinite(outs[0]["f0"])) and np.abs(outs[0]["f0"]).max() > 0


def test_lean_split_kernels_bitwise(tmp_path):
    """The 6 9^a-only instantiations of the split-length passes (default on the 8748 torus) against
    the general kernels (RK_LEAN=0): the same stage bodies, bitwise identical."""
    kw = dict(n=6000, L=2, dims=(4096, 4096), nu=1.5)
    a = _run(tmp_path, "lean", {"RK_LEAN": "1"}, **kw)
    b = _run(tmp_path, "general", {"RK_LEAN": "0"}, **kw)
    assert tuple(a["embed"]) == (8748, 8748)
    assert np.array_equal(a["field"], b["field"])
    assert np.array_equal(a["conv"], b["conv"])
