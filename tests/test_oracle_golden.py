"""Pin the CPU oracle (oracle/rk_oracle.py) to golden vectors from the real reference.

CPU-only; these run in the build container and on the GPU box.
"""

import numpy as np
import pytest

from oracle import rk_oracle as ro
from rk_testutil import load_golden, rel_err


def test_matern_matches_reference():
    g = load_golden("matern")
    for nu, phi in zip(g["nus"], g["phi"]):
        ours = ro.matern_phi(g["d"], float(nu))
        assert np.abs(ours - phi).max() <= 1e-15, nu


def test_matern_limits():
    assert ro.matern_phi(0.0, 1.0)[0] == 1.0
    assert ro.matern_phi(1e-12, 2.5)[0] == 1.0
    with pytest.raises(ro.OracleDomainError):
        ro.matern_phi(-1.0, 1.0)


def test_fft_len_matches_reference():
    g = load_golden("fft_len")
    assert [ro.fft_len(int(k)) for k in g["n"]] == list(g["p"])


def test_grids_and_stencils_bit_exact():
    g = load_golden("grids")
    for i in range(int(g["n"])):
        dims, L, obs = tuple(g[f"dims_{i}"]), int(g[f"L_{i}"]), g[f"obs_{i}"]
        grid = ro.make_grid((0.0, 1.0, 0.0, 1.0), dims, L, obs)
        assert grid.pad == tuple(g[f"pad_{i}"])
        base, off = ro.stencils(grid, obs, L)
        idx = ro.expand_indices(base, grid.total_dims[0], L)
        assert np.array_equal(idx, g[f"indices_{i}"])
        assert np.array_equal(off, g[f"offsets_{i}"])


@pytest.mark.parametrize("case", ["s0", "s1", "s2", "s3", "s4", "s5"])
def test_setup_and_predict_match_reference(case):
    g = load_golden("setup_" + case)
    model = ro.Model(float(g["sigma2"]), float(g["alpha"]), float(g["nu"]), float(g["tau2"]))
    grid = ro.make_grid((0.0, 1.0, 0.0, 1.0), tuple(g["dims"]), int(g["L"]), g["obs"])
    assert grid.pad == tuple(g["pad"])
    st = ro.rapid_setup(model, grid, int(g["L"]), g["obs"])
    assert np.array_equal(st.indices, g["indices"])
    assert np.array_equal(np.array(st.embed_dims), g["embed_dims"])
    assert np.abs(st.spectrum - g["spectrum"]).max() <= 1e-13 * np.abs(g["spectrum"]).max()
    assert rel_err(st.weights, g["weights"]) < 1e-12
    assert np.abs(st.cond_var - g["cond_var"]).max() < 1e-13
    beta = g["beta"] if g["beta"].size else None
    xg = g["xg"] if g["xg"].size else None
    assert rel_err(ro.scatter_cstar(st, g["c"]), g["cstar"]) < 1e-14
    assert rel_err(ro.predict(st, g["c"], beta, xg), g["field"]) < 1e-13


@pytest.mark.parametrize("name", ["cfg1", "cfg2"])
def test_config_fields_match_reference(name):
    from paper_2605_29284_b200 import workloads
    g = load_golden(name)
    wl = workloads.CONFIGS[name]()
    assert np.array_equal(wl.obs, g["obs"])
    model = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    grid = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
    assert grid.pad == tuple(g["pad"])
    st = ro.rapid_setup(model, grid, wl.L, wl.obs)
    assert np.array_equal(st.base, g["base"])
    xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
    assert rel_err(ro.predict(st, g["c"], g["beta"], xg), g["field"]) < 1e-12


def test_rng_bit_exact():
    g = load_golden("rng")
    for si, s in enumerate(g["seeds"]):
        for ji, j in enumerate(g["js"]):
            assert ro.sub_seed(int(s), int(j)) == int(g["sub"][si, ji])
    row = 0
    for s in g["seeds"]:
        for stream in (0, 1):
            words = ro.philox_words(int(s), stream, 0, 37)
            assert np.array_equal(words, g["raw"][row])
            assert np.array_equal(ro.words_to_normals(words), g["normals"][row])
            row += 1


def test_philox_matches_numpy_at_offsets():
    bg = np.random.Philox(key=12345 + (1 << 64))
    raw = bg.random_raw(1000)
    assert np.array_equal(ro.philox_words(12345, 1, 993, 7), raw[993:])


def test_cs_chain_matches_reference():
    g = load_golden("cs_small")
    model = ro.Model(float(g["sigma2"]), float(g["alpha"]), float(g["nu"]), float(g["tau2"]))
    fit = ro.exact_fit(model, g["obs"], g["z"])
    assert rel_err(fit.c, g["c"]) < 1e-12
    grid = ro.make_grid((0.0, 1.0, 0.0, 1.0), tuple(g["dims"]), int(g["L"]), g["obs"])
    st = ro.rapid_setup(model, grid, int(g["L"]), g["obs"])
    p1, p2, root = ro.embedding_root(model, grid)
    assert (p1, p2) == tuple(g["embed"])
    assert rel_err(root, g["root"]) < 1e-13
    gf = ro.uncond_field(model, grid, 5)
    assert rel_err(gf, g["g"]) < 1e-13
    zs = ro.obs_local(model, st, g["g"], 6)
    assert rel_err(zs, g["zs"]) < 1e-13
    bs, cs = ro.refit(fit, g["zs"])
    assert rel_err(cs, g["cs"]) < 1e-10
    assert rel_err(ro.cond_draw(fit, st, 9), g["draw"]) < 1e-12
    draws, mean, se = ro.ensemble(fit, st, 4, 3)
    assert rel_err(draws, g["ens_draws"]) < 1e-12
    assert rel_err(se, g["ens_se"]) < 1e-11


def test_cs_covariates_and_doubling():
    g = load_golden("cs_cov")
    model = ro.Model(float(g["sigma2"]), float(g["alpha"]), float(g["nu"]), float(g["tau2"]))
    fit = ro.exact_fit(model, g["obs"], g["z"], g["X"])
    grid = ro.make_grid((0.0, 1.0, 0.0, 1.0), tuple(g["dims"]), int(g["L"]), g["obs"])
    st = ro.rapid_setup(model, grid, int(g["L"]), g["obs"])
    draws, mean, se = ro.ensemble(fit, st, 3, 77, g["xg"])
    assert rel_err(draws, g["ens_draws"]) < 1e-11
    d = load_golden("cs_doubling")
    model = ro.Model(1.0, 4.0, 1.0)
    grid = ro.make_grid((0.0, 1.0, 0.0, 1.0), tuple(d["dims"]), 2, [])
    p1, p2, _ = ro.embedding_root(model, grid)
    assert (p1, p2) == tuple(d["embed"])
    assert rel_err(ro.uncond_field(model, grid, 3), d["g"]) < 1e-13


def test_embedding_failure_raises():
    model = ro.Model(1.0, 1.0, 1.5)
    grid = ro.make_grid((0.0, 1.0, 0.0, 1.0), (24, 24), 2, [])
    with pytest.raises(ro.OracleNumericError, match="eigenvalue"):
        ro.embedding_root(model, grid)


@pytest.mark.parametrize("tag", ["cov", "icpt"])
def test_exact_targets_match_reference(tag):
    """predict_exact / kriging_se_exact (exact.py:132-175) restated in the oracle, on the
    reference's own fit (chol_M, beta_hat, c)."""
    g = load_golden("exact_targets")
    model = ro.Model(float(g["sigma2"]), float(g["alpha"]), float(g[f"{tag}_nu"]), float(g["tau2"]))
    X = g[f"{tag}_X"] if g[f"{tag}_X"].size else np.ones((g[f"{tag}_obs"].shape[0], 1))
    fit = ro.Fit(model, g[f"{tag}_obs"], X, g[f"{tag}_chol"], g[f"{tag}_beta"], g[f"{tag}_c"])
    xt = g[f"{tag}_xt"] if g[f"{tag}_xt"].size else None
    assert rel_err(ro.predict_exact(fit, g[f"{tag}_targets"], xt), g[f"{tag}_pred"]) < 1e-13
    assert rel_err(ro.kriging_se_exact(fit, g[f"{tag}_targets"], xt), g[f"{tag}_se"]) < 1e-13
    # and the oracle's own fit reproduces the reference's
    fit2 = ro.exact_fit(model, g[f"{tag}_obs"], g[f"{tag}_z"], None if tag == "icpt" else X)
    assert rel_err(fit2.c, g[f"{tag}_c"]) < 1e-10
