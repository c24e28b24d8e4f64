"""GPU parity: CUDA path (through the C ABI) vs the reference's golden vectors and the oracle.

Tolerances (north_star / SURVEY §8(c)): stencil indices and pads bit-exact;
interpolation residual < 1e-8; fields, c* and CS draws/SE <= 1e-10 relative to
max|ref|; Philox words bit-exact; normals <= 1e-14 relative.
"""

import numpy as np
import pytest

from oracle import rk_oracle as ro
from rk_testutil import has_gpu, load_golden, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

UNIT = (0.0, 1.0, 0.0, 1.0)
FIELD_TOL = 1e-10


@pytest.fixture(scope="module")
def pk():
    import paper_2605_29284_b200 as pk
    return pk


def _model(pk, g):
    return pk.CovarianceModel(float(g["sigma2"]), float(g["alpha"]), float(g["nu"]), float(g["tau2"]))


def test_matern_against_reference(pk):
    g = load_golden("matern")
    for nu, phi in zip(g["nus"], g["phi"]):
        ours = pk.matern_phi(g["d"], float(nu))
        assert np.abs(ours - phi).max() <= 1e-13 * max(1.0, np.abs(phi).max()), nu


def test_padded_grid_and_stencils_bit_exact(pk):
    g = load_golden("grids")
    for i in range(int(g["n"])):
        dims, L, obs = tuple(int(v) for v in g[f"dims_{i}"]), int(g[f"L_{i}"]), g[f"obs_{i}"]
        grid = pk.build_padded_grid(UNIT, dims, L, obs)
        assert grid.pad == tuple(int(v) for v in g[f"pad_{i}"])
        model = pk.CovarianceModel(1.0, 3.0, 1.5)
        st = pk.build_setup(model, grid, L, obs)
        assert np.array_equal(st.neighbor_indices, g[f"indices_{i}"])


@pytest.mark.parametrize("case", ["s0", "s1", "s2", "s3", "s4", "s5"])
def test_setup_and_predict_against_reference(pk, case):
    g = load_golden("setup_" + case)
    model = _model(pk, g)
    L = int(g["L"])
    grid = pk.build_padded_grid(UNIT, tuple(int(v) for v in g["dims"]), L, g["obs"])
    assert grid.pad == tuple(int(v) for v in g["pad"])
    st = pk.build_setup(model, grid, L, g["obs"])
    assert np.array_equal(st.neighbor_indices, g["indices"])
    assert st.embed_dims == tuple(int(v) for v in g["embed_dims"])
    # interpolation condition K_N w_i = k_i (reference test_acceptance.py:98-116)
    kn = g["kn"]
    nx, ny = grid.to_coords(st.neighbor_indices)
    k_rows = ro.Model(model.sigma2, model.alpha, model.nu).cov(
        np.hypot(nx - g["obs"][:, :1], ny - g["obs"][:, 1:2]))
    assert np.abs(kn @ st.weights.T - k_rows.T).max() < 1e-8
    assert np.abs(st.cond_var - g["cond_var"]).max() < 1e-8
    spec = st.filter_spectrum
    assert np.abs(spec - g["spectrum"]).max() <= 1e-12 * np.abs(g["spectrum"]).max()
    beta = g["beta"] if g["beta"].size else None
    xg = g["xg"] if g["xg"].size else None
    assert rel_err(st.coefficients_to_grid(g["c"]), g["cstar"]) < 1e-12
    assert rel_err(pk.predict_rapid(st, g["c"], beta, xg), g["field"]) < FIELD_TOL


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_config_field_against_reference(pk, name):
    from paper_2605_29284_b200 import workloads
    g = load_golden(name)
    wl = workloads.CONFIGS[name]()
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    assert grid.pad == tuple(int(v) for v in g["pad"])
    st = pk.build_setup(model, grid, wl.L, wl.obs)
    assert st.embed_dims == tuple(int(v) for v in g["embed_dims"])
    assert np.array_equal(st.neighbor_indices[:, 0], g["base"])
    xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
    field = pk.predict_rapid(st, g["c"], g["beta"], xg)
    assert rel_err(field, g["field"]) < FIELD_TOL
    # device-resident path gives the same field
    import torch
    fd = pk.predict_rapid(st, torch.as_tensor(g["c"], device="cuda"), g["beta"],
                          None if xg is None else torch.as_tensor(xg, device="cuda"))
    assert rel_err(fd.cpu().numpy(), g["field"]) < FIELD_TOL


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_pinned_host_path_chunked_upload(pk, name):
    """Pinned host buffers take the chunked-upload path (eager call, graph capture on the
    second, replay on the third): identical to the device path bit for bit."""
    import torch
    from paper_2605_29284_b200 import workloads
    g = load_golden(name)
    wl = workloads.CONFIGS[name]()
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = pk.build_setup(model, grid, wl.L, wl.obs)
    xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
    m1, m2 = grid.interior_dims
    ch = torch.from_numpy(np.ascontiguousarray(g["c"])).pin_memory().numpy()
    xh = None if xg is None else torch.from_numpy(np.ascontiguousarray(xg)).pin_memory().numpy()
    want = pk.predict_rapid(st, torch.as_tensor(g["c"], device="cuda"), g["beta"],
                            None if xg is None else torch.as_tensor(xg, device="cuda")).cpu().numpy()
    assert rel_err(want, g["field"]) < FIELD_TOL
    out = torch.empty((m2, m1), dtype=torch.float64).pin_memory().numpy()
    for it in range(4):
        out[:] = np.nan
        ch[:] = g["c"] * (1.0 + it)     # same pointers, new values: graph replays see them
        got = pk.predict_rapid(st, ch, g["beta"], xh, out=out)
        assert got is out
        ref = want if it == 0 else pk.predict_rapid(
            st, torch.as_tensor(g["c"] * (1.0 + it), device="cuda"), g["beta"],
            None if xg is None else torch.as_tensor(xg, device="cuda")).cpu().numpy()
        assert np.array_equal(out, ref), it


@pytest.mark.parametrize("dims,L,nu", [((2, 2), 1, 1.0), ((3, 5), 1, 1.5), ((16, 11), 2, 0.5),
                                       ((37, 29), 3, 2.5), ((64, 70), 2, 1.0), ((120, 81), 4, 1.5)])
def test_convolution_and_predict_vs_oracle(pk, dims, L, nu):
    rng = np.random.default_rng(dims[0] * 1000 + dims[1])
    obs = rng.uniform(0, 1, size=(max(4, dims[0] * dims[1] // 7), 2))
    model = pk.CovarianceModel(1.2, 4.0, nu, 0.1)
    omodel = ro.Model(1.2, 4.0, nu, 0.1)
    grid = pk.build_padded_grid(UNIT, dims, L, obs)
    ogrid = ro.make_grid(UNIT, dims, L, obs)
    assert grid.pad == ogrid.pad
    st = pk.build_setup(model, grid, L, obs)
    ost = ro.rapid_setup(omodel, ogrid, L, obs)
    assert np.array_equal(st.neighbor_indices, ost.indices)
    c = rng.normal(size=obs.shape[0])
    assert rel_err(pk.predict_rapid(st, c, [0.3]), ro.predict(ost, c, [0.3])) < FIELD_TOL
    # convolve_filter against the oracle's numpy FFT convolution
    M1, M2 = grid.total_dims
    vals = rng.normal(size=(M2, M1))
    emb, spec = pk.build_filter_spectrum(model, grid)
    assert emb == ost.embed_dims
    ours = pk.convolve_filter(spec, emb, vals)
    assert rel_err(ours, ro.circ_convolve(ost.spectrum, ost.embed_dims, vals)) < 1e-12
    ours2 = pk.convolve_filter(np.asarray(spec), emb, vals)
    assert rel_err(ours2, ours) < 1e-14


def test_linearity_zero_and_reuse(pk):
    rng = np.random.default_rng(3)
    model = pk.CovarianceModel(1.0, 4.0, 1.5)
    obs = rng.uniform(0, 1, size=(10, 2))
    grid = pk.build_padded_grid(UNIT, (14, 14), 2, obs)
    st = pk.build_setup(model, grid, 2, obs)
    c1, c2 = rng.normal(size=10), rng.normal(size=10)
    lhs = pk.predict_rapid(st, 1.7 * c1 + c2)
    rhs = 1.7 * pk.predict_rapid(st, c1) + pk.predict_rapid(st, c2)
    assert np.abs(lhs - rhs).max() < 1e-10
    z = pk.predict_rapid(st, np.zeros(10), np.array([2.5]))
    assert np.abs(z - 2.5).max() < 1e-14
    st2 = pk.build_setup(model, grid, 2, obs)
    assert np.array_equal(st.filter_spectrum, st2.filter_spectrum)
    assert np.array_equal(pk.predict_rapid(st, c1), pk.predict_rapid(st2, c1))


def test_on_node_unit_rows(pk):
    model = pk.CovarianceModel(1.0, 4.0, 1.5)
    grid = pk.build_padded_grid(UNIT, (11, 11), 2, [(0.5, 0.5)])
    st = pk.build_setup(model, grid, 2, [(0.5, 0.5)])
    row = st.weights[0]
    assert np.count_nonzero(row) == 1 and row.max() == 1.0
    x, y = grid.to_coords(st.neighbor_indices[0][np.argmax(row)])
    assert (x, y) == (0.5, 0.5)
    assert st.cond_var[0] == 0.0


def test_errors_map_to_reference_exceptions(pk):
    model = pk.CovarianceModel(1.0, 4.0, 1.0)
    obs = np.array([(0.5, 0.5), (0.3, 0.7)])
    grid = pk.build_padded_grid(UNIT, (8, 8), 2, obs)
    st = pk.build_setup(model, grid, 2, obs)
    with pytest.raises(pk.DomainError):
        pk.predict_rapid(st, np.zeros(5))
    with pytest.raises(pk.DomainError):
        pk.predict_rapid(st, np.zeros(2), np.array([1.0, 2.0]))
    with pytest.raises(pk.DomainError):
        pk.build_padded_grid(UNIT, (10, 10), 2, [(1.2, 0.5)])
    with pytest.raises(pk.DomainError):
        pk.build_padded_grid(UNIT, (7, 10), 4, [(0.5, 0.5)])
    with pytest.raises(pk.DomainError):
        pk.build_setup(model, grid, 2, np.zeros((0, 2)))
    # location outside the padded coverage / stencil leaving the grid
    with pytest.raises(pk.DomainError):
        pk.build_setup(model, grid, 2, [(5.0, 5.0)])
    small = pk.build_padded_grid(UNIT, (10, 10), 2, [(0.5, 0.5)])
    with pytest.raises(pk.InternalError):
        pk.build_setup(model, small, 2, [(0.01, 0.01)])


def test_philox_bit_exact_and_normals(pk):
    import torch
    from paper_2605_29284_b200 import _native as N
    g = load_golden("rng")
    row = 0
    for s in g["seeds"]:
        for stream in (0, 1):
            raw = torch.empty(37, dtype=torch.int64, device="cuda")
            N.call("rk_philox_raw", int(s), stream, 0, 37, N.ptr(raw), N.stream_ptr())
            assert np.array_equal(raw.cpu().numpy().view(np.uint64), g["raw"][row])
            nrm = torch.empty(37, dtype=torch.float64, device="cuda")
            N.call("rk_philox_normals", int(s), stream, 0, 37, N.ptr(nrm), N.stream_ptr())
            ref = g["normals"][row]
            assert np.abs(nrm.cpu().numpy() - ref).max() <= 1e-14 * np.abs(ref).max()
            row += 1
    for si, s in enumerate(g["seeds"]):
        for ji, j in enumerate(g["js"]):
            assert N.load().rk_draw_seed(int(s), int(j)) == int(g["sub"][si, ji])
            assert pk.draw_seed(int(s), int(j)) == int(g["sub"][si, ji])


def test_philox_long_stream_vs_numpy():
    import torch
    from paper_2605_29284_b200 import _native as N
    raw = torch.empty(100_003, dtype=torch.int64, device="cuda")
    N.call("rk_philox_raw", 987654321, 0, 5, 100_003, N.ptr(raw), N.stream_ptr())
    ref = np.random.Philox(key=987654321).random_raw(100_008)[5:]
    assert np.array_equal(raw.cpu().numpy().view(np.uint64), ref)


def test_cs_chain_against_reference(pk):
    g = load_golden("cs_small")
    model = _model(pk, g)
    grid = pk.build_padded_grid(UNIT, tuple(int(v) for v in g["dims"]), int(g["L"]), g["obs"])
    st = pk.build_setup(model, grid, int(g["L"]), g["obs"])
    from paper_2605_29284_b200.simulate import embedding_dims
    assert embedding_dims(model, grid)[:2] == tuple(int(v) for v in g["embed"])
    gf = pk.sim_unconditional_grid(model, grid, 5)
    assert rel_err(gf, g["g"]) < FIELD_TOL
    zs = pk.sim_obs_local(model, st, g["g"], 6)
    assert rel_err(zs, g["zs"]) < FIELD_TOL
    # GPU fit reproduces the reference fit
    f = pk.fit(model, g["obs"], g["z"])
    assert rel_err(f.c, g["c"]) < 1e-10
    assert rel_err(f.chol_M, g["chol_M"]) < 1e-12
    bs, cs = pk.refit_coefficients(f, g["zs"])
    assert rel_err(cs, g["cs"]) < 1e-10
    assert rel_err(bs, g["bs"]) < 1e-10
    assert rel_err(pk.conditional_draw(f, st, 9), g["draw"]) < FIELD_TOL
    ens = pk.generate_ensemble(f, st, 4, 3)
    assert rel_err(ens.draws, g["ens_draws"]) < FIELD_TOL
    assert rel_err(ens.mean_field, g["ens_mean"]) < FIELD_TOL
    assert rel_err(ens.empirical_se, g["ens_se"]) < FIELD_TOL
    assert ens.rng_algorithm == "philox4x64-10"


def test_cs_with_imported_reference_fit_and_covariates(pk):
    g = load_golden("cs_cov")

    class RefFit:   # a reference-style KrigingFit (exact.py:40-56) built from the golden
        pass
    rf = RefFit()
    rf.model = _model(pk, g)
    rf.obs_locs, rf.X, rf.chol_M = g["obs"], g["X"], g["chol_M"]
    rf.beta_hat, rf.c = g["beta"], g["c"]
    grid = pk.build_padded_grid(UNIT, tuple(int(v) for v in g["dims"]), int(g["L"]), g["obs"])
    st = pk.build_setup(rf.model, grid, int(g["L"]), g["obs"])
    ens = pk.generate_ensemble(rf, st, 3, 77, grid_covariates=g["xg"])
    assert rel_err(ens.draws, g["ens_draws"]) < FIELD_TOL
    assert rel_err(ens.empirical_se, g["ens_se"]) < FIELD_TOL
    with pytest.raises(pk.DomainError):
        pk.generate_ensemble(rf, st, 3, 77)          # covariates required for p = 3
    with pytest.raises(pk.DomainError):
        pk.generate_ensemble(rf, st, 1, 77, grid_covariates=g["xg"])


def test_embedding_doubling_and_failure(pk):
    d = load_golden("cs_doubling")
    model = pk.CovarianceModel(1.0, 4.0, 1.0)
    grid = pk.build_padded_grid(UNIT, tuple(int(v) for v in d["dims"]), 2, [])
    from paper_2605_29284_b200.simulate import embedding_dims
    p1, p2, doubled = embedding_dims(model, grid)
    assert (p1, p2) == tuple(int(v) for v in d["embed"]) and doubled
    assert rel_err(pk.sim_unconditional_grid(model, grid, 3), d["g"]) < FIELD_TOL
    bad = pk.CovarianceModel(1.0, 1.0, 1.5)
    with pytest.raises(pk.NumericError, match="eigenvalue"):
        pk.sim_unconditional_grid(bad, grid, 0)


def test_ensemble_determinism_batch_independence(pk):
    rng = np.random.default_rng(4)
    model = pk.CovarianceModel(1.0, 6.0, 1.5, 0.05)
    obs = rng.uniform(0, 1, size=(40, 2))
    z = rng.normal(size=40)
    f = pk.fit(model, obs, z)
    grid = pk.build_padded_grid(UNIT, (24, 20), 2, obs)
    st = pk.build_setup(model, grid, 2, obs)
    e1 = pk.generate_ensemble(f, st, 20, 99, batch=7)
    e2 = pk.generate_ensemble(f, st, 20, 99, batch=32)
    assert np.array_equal(e1.draws, e2.draws)
    assert np.array_equal(e1.empirical_se, e2.empirical_se)
    # oracle per-draw parity
    ofit = ro.exact_fit(ro.Model(1.0, 6.0, 1.5, 0.05), obs, z)
    ost = ro.rapid_setup(ofit.model, ro.make_grid(UNIT, (24, 20), 2, obs), 2, obs)
    draws, mean, se = ro.ensemble(ofit, ost, 20, 99)
    assert rel_err(e1.draws, draws) < FIELD_TOL
    assert rel_err(e1.empirical_se, se) < FIELD_TOL
    assert rel_err(e1.mean_field, mean) < FIELD_TOL


_RECURSIVE_INV_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + '/tests')
import paper_2605_29284_b200 as pk
from oracle import rk_oracle as ro
from rk_testutil import rel_err
rng = np.random.default_rng(8)
obs = rng.uniform(0, 1, size=(1100, 2))
z = rng.normal(size=1100)
model = pk.CovarianceModel(1.0, 8.0, 1.5, 0.05)
f = pk.fit(model, obs, z)
st = pk.build_setup(model, pk.build_padded_grid((0.0, 1.0, 0.0, 1.0), (30, 26), 2, obs), 2, obs)
e = pk.generate_ensemble(f, st, 4, 5)
ofit = ro.exact_fit(ro.Model(1.0, 8.0, 1.5, 0.05), obs, z)
ost = ro.rapid_setup(ofit.model, ro.make_grid((0.0, 1.0, 0.0, 1.0), (30, 26), 2, obs), 2, obs)
draws, mean, se = ro.ensemble(ofit, ost, 4, 5)
print(rel_err(e.draws, draws), rel_err(e.empirical_se, se))
"""


def test_recursive_factor_inverse_matches_oracle():
    """Batched refit through the blocked (recursive) inverse of the Cholesky factor, forced
    at n=1100 with RK_TRTRI_BLOCK=256 (the path n > 16384 takes, e.g. cfg5's n=50000)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RK_TRTRI_BLOCK="256")
    r = subprocess.run([sys.executable, "-c", _RECURSIVE_INV_SCRIPT, root], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d, s = (float(v) for v in r.stdout.split()[-2:])
    assert d < FIELD_TOL and s < FIELD_TOL, (d, s)


_UNFUSED_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2605_29284_b200 as pk
from paper_2605_29284_b200 import workloads
wl = workloads.cfg2()
model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
st = pk.build_setup(model, grid, wl.L, wl.obs)
xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
c = np.random.default_rng(2).normal(size=wl.obs.shape[0])
np.save(sys.argv[2], pk.predict_rapid(st, c, [0.5, 1.0, -1.0], xg))
"""


def test_fused_and_standalone_scatter_identical(tmp_path):
    """Pass 1 with the fused in-smem scatter and the standalone scatter kernel (forced with
    RK_FUSED_GATHER=0) give bit-identical fields."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for flag in ("1", "0"):
        f = str(tmp_path / f"f{flag}.npy")
        r = subprocess.run([sys.executable, "-c", _UNFUSED_SCRIPT, root, f],
                           env=dict(os.environ, RK_FUSED_GATHER=flag), capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("tag", ["cov", "icpt"])
def test_predict_exact_and_se_against_reference(pk, tag):
    """GPU predict_exact / kriging_se_exact (exact.py:132-175) against the reference, on our GPU
    fit and on the reference's own fit adopted through as_device_fit; device targets stay on
    the device; intercept-only fits take target_covariates=None; bad covariates raise."""
    import torch
    g = load_golden("exact_targets")
    model = pk.CovarianceModel(float(g["sigma2"]), float(g["alpha"]), float(g[f"{tag}_nu"]), float(g["tau2"]))
    X = g[f"{tag}_X"] if g[f"{tag}_X"].size else None
    xt = g[f"{tag}_xt"] if g[f"{tag}_xt"].size else None
    f = pk.fit(model, g[f"{tag}_obs"], g[f"{tag}_z"], X)
    tg = g[f"{tag}_targets"]
    assert rel_err(pk.predict_exact(f, tg, xt), g[f"{tag}_pred"]) < FIELD_TOL
    assert rel_err(pk.kriging_se_exact(f, tg, xt, chunk=97), g[f"{tag}_se"]) < FIELD_TOL
    from types import SimpleNamespace   # the reference KrigingFit's attribute names (exact.py:40-56)
    ofit = SimpleNamespace(model=model, obs_locs=g[f"{tag}_obs"],
                           X=X if X is not None else np.ones((len(g[f"{tag}_obs"]), 1)),
                           chol_M=g[f"{tag}_chol"], beta_hat=g[f"{tag}_beta"], c=g[f"{tag}_c"])
    pd = pk.predict_exact(ofit, torch.as_tensor(tg, device="cuda"), None if xt is None else torch.as_tensor(xt, device="cuda"))
    assert pd.is_cuda and rel_err(pd.cpu().numpy(), g[f"{tag}_pred"]) < FIELD_TOL
    if tag == "cov":
        with pytest.raises(pk.DomainError):
            pk.predict_exact(f, tg)
        with pytest.raises(pk.DomainError):
            pk.kriging_se_exact(f, tg, xt[:, :2])


def test_concurrent_streams_share_one_setup(pk):
    """A setup is immutable and shareable across concurrent predicts: two CUDA
    streams, each with its own workspace / captured graph, give the sequential results."""
    import torch
    rng = np.random.default_rng(12)
    obs = rng.uniform(0, 1, size=(300, 2))
    model = pk.CovarianceModel(1.0, 7.0, 1.5, 0.02)
    grid = pk.build_padded_grid(UNIT, (90, 70), 3, obs)
    st = pk.build_setup(model, grid, 3, obs)
    cs = [torch.as_tensor(rng.normal(size=300), device="cuda") for _ in range(4)]
    beta = torch.as_tensor([0.7], device="cuda")
    want = [pk.predict_rapid(st, c, beta).cpu().numpy() for c in cs]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [torch.empty((70, 90), dtype=torch.float64, device="cuda") for _ in range(4)]
    for rep in range(3):   # first use eager, second captures, third replays
        for k in range(4):
            with torch.cuda.stream(streams[k % 2]):
                pk.predict_rapid(st, cs[k], beta, out=outs[k])
        torch.cuda.synchronize()
        for k in range(4):
            assert np.array_equal(outs[k].cpu().numpy(), want[k]), (rep, k)


@pytest.mark.parametrize("nu,alpha", [(2.5, 0.3), (3.5, 1.0)])
def test_kn_ridge_branch_against_oracle(pk, nu, alpha):
    """K_N numerically singular (smooth, long-range Matern on a fine grid, L = 4): the setup adds
    the documented ridge 1e-12 sigma2 (2L)^2 with a RuntimeWarning, exactly when the reference
    does (rapid.py:120-135, restated by the oracle's kn_factor), and the field still matches the
    oracle's ridged setup."""
    rng = np.random.default_rng(21)
    obs = rng.uniform(0, 1, size=(300, 2))
    model = pk.CovarianceModel(1.0, alpha, nu)
    om = ro.Model(1.0, alpha, nu)
    og = ro.make_grid(UNIT, (100, 100), 4, obs)
    _, ridged = ro.kn_factor(om, ro.kn_matrix(om, og, 4), 4)
    assert ridged
    grid = pk.build_padded_grid(UNIT, (100, 100), 4, obs)
    with pytest.warns(RuntimeWarning, match="ridge"):
        st = pk.build_setup(model, grid, 4, obs)
    assert st.ridge_applied
    ost = ro.rapid_setup(om, og, 4, obs)
    c = rng.normal(size=300)
    ref = ro.predict(ost, c, np.array([0.5]))
    assert rel_err(pk.predict_rapid(st, c, np.array([0.5])), ref) < FIELD_TOL
