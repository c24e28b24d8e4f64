"""Behavioural properties the reference's own tests check (tests/test_rapid.py, test_simulate.py,
test_exact.py in the reference package), restated for the GPU path: exactness limits, invariances,
statistics, instrumentation and error behaviour."""
import warnings

import numpy as np
import pytest

from rk_testutil import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

UNIT = (0.0, 1.0, 0.0, 1.0)


@pytest.fixture(scope="module")
def pk():
    import paper_2605_29284_b200 as pk
    return pk


def _pts(n, seed):
    return np.random.default_rng(seed).uniform(0.05, 0.95, size=(n, 2))


def test_zero_variance_gives_zero_field(pk):
    model = pk.CovarianceModel(1e-300, 4.0, 1.0)
    grid = pk.build_padded_grid(UNIT, (8, 8), 1, np.zeros((0, 2)))
    assert np.abs(pk.sim_unconditional_grid(model, grid, 0)).max() < 1e-140


def test_coincident_observations_share_weights(pk):
    model = pk.CovarianceModel(1.0, 4.0, 1.0)
    obs = np.array([(0.43, 0.57), (0.43, 0.57), (0.8, 0.2)])
    st = pk.build_setup(model, pk.build_padded_grid(UNIT, (10, 10), 2, obs), 2, obs)
    assert np.array_equal(st.neighbor_indices[0], st.neighbor_indices[1])
    assert np.array_equal(st.weights[0], st.weights[1])


def test_build_count_and_ensemble_amortizes_setup(pk):
    from paper_2605_29284_b200 import rapid
    rng = np.random.default_rng(5)
    model = pk.CovarianceModel(1.0, 4.0, 1.0, 0.05)
    obs = rng.uniform(0, 1, size=(10, 2))
    grid = pk.build_padded_grid(UNIT, (10, 10), 2, obs)
    before = rapid.BUILD_COUNT
    st = pk.build_setup(model, grid, 2, obs)
    pk.build_setup(model, grid, 2, obs)
    assert rapid.BUILD_COUNT == before + 2
    f = pk.fit(model, obs, rng.normal(size=10))
    pk.generate_ensemble(f, st, 8, 1)
    assert rapid.BUILD_COUNT == before + 2


def test_exact_interpolation_and_far_field(pk):
    rng = np.random.default_rng(6)
    obs = _pts(25, 5)
    z = rng.normal(size=25)
    f = pk.fit(pk.CovarianceModel(1.5, 5.0, 1.5, 0.0), obs, z)
    assert np.abs(pk.predict_exact(f, obs) - z).max() / np.abs(z).max() < 1e-8
    assert np.abs(pk.kriging_se_exact(f, obs)).max() < 1e-5          # zero nugget: exact at the data
    f2 = pk.fit(pk.CovarianceModel(1.0, 50.0, 1.0, 0.1), _pts(10, 7), rng.normal(size=10) + 5.0)
    far = np.array([(40.0, 40.0)])
    assert pk.predict_exact(f2, far)[0] == pytest.approx(f2.beta_hat[0], abs=1e-8)
    assert pk.kriging_se_exact(f2, far)[0] >= 1.0 - 1e-12             # at least sigma far away


def test_predict_exact_linear_and_permutation_invariant(pk):
    rng = np.random.default_rng(9)
    obs = _pts(40, 9)
    model = pk.CovarianceModel(1.0, 6.0, 1.5, 0.05)
    tg = rng.uniform(0, 1, size=(50, 2))
    z1, z2 = rng.normal(size=40), rng.normal(size=40)
    p1 = pk.predict_exact(pk.fit(model, obs, z1), tg)
    p2 = pk.predict_exact(pk.fit(model, obs, z2), tg)
    p12 = pk.predict_exact(pk.fit(model, obs, 2.0 * z1 - z2), tg)
    assert np.abs(p12 - (2.0 * p1 - p2)).max() < 1e-10 * np.abs(p12).max()
    perm = rng.permutation(40)
    pp = pk.predict_exact(pk.fit(model, obs[perm], z1[perm]), tg)
    assert np.abs(pp - p1).max() < 1e-10 * np.abs(p1).max()


def test_refit_matches_fresh_fit(pk):
    rng = np.random.default_rng(11)
    obs = _pts(60, 11)
    X = np.column_stack([np.ones(60), obs[:, 0]])
    model = pk.CovarianceModel(1.0, 5.0, 1.0, 0.1)
    f = pk.fit(model, obs, rng.normal(size=60), X)
    z2 = rng.normal(size=60)
    beta, c = pk.refit_coefficients(f, z2)
    g = pk.fit(model, obs, z2, X)
    assert np.abs(beta - g.beta_hat).max() < 1e-10 and np.abs(c - g.c).max() < 1e-9 * np.abs(g.c).max()


def test_ridge_retry_warns_on_duplicate_locations(pk):
    model = pk.CovarianceModel(1.0, 2.0, 1.0, 0.0)
    obs = np.array([(0.2, 0.2), (0.2, 0.2), (0.7, 0.7)])
    with pytest.warns(RuntimeWarning):
        f = pk.fit(model, obs, np.array([1.0, 1.0, 0.0]))
    assert np.all(np.isfinite(f.c))


def test_conditional_draw_pins_data_at_zero_nugget(pk):
    """With tau2 = 0 and observations on grid nodes, every conditional draw reproduces the
    data at those nodes (simulate.py:146-159)."""
    rng = np.random.default_rng(1)
    model = pk.CovarianceModel(1.0, 5.0, 1.0, 0.0)
    nodes = pk.build_padded_grid(UNIT, (12, 12), 2, np.zeros((0, 2))).interior_nodes()
    pick = rng.choice(len(nodes), size=20, replace=False)
    obs, z = nodes[pick], rng.normal(size=20)
    f = pk.fit(model, obs, z)
    st = pk.build_setup(model, pk.build_padded_grid(UNIT, (12, 12), 2, obs), 2, obs)
    for seed in range(3):
        assert np.abs(pk.conditional_draw(f, st, seed).ravel()[pick] - z).max() < 1e-6


def test_ensemble_std_matches_exact_se(pk):
    """Monte Carlo SE of the GPU ensemble against the GPU exact SE (reference
    test_simulate.py:141-153 / test_acceptance.py:216-243 style)."""
    rng = np.random.default_rng(3)
    obs = _pts(30, 3)
    model = pk.CovarianceModel(1.0, 5.0, 1.5, 0.05)
    f = pk.fit(model, obs, rng.normal(size=30))
    grid = pk.build_padded_grid(UNIT, (24, 24), 3, obs)
    st = pk.build_setup(model, grid, 3, obs)
    ens = pk.generate_ensemble(f, st, 800, 17, keep_draws=False)
    se = pk.kriging_se_exact(f, grid.interior_nodes()).reshape(24, 24)
    rel = np.abs(ens.empirical_se - se) / se
    assert np.median(rel) < 0.05 and np.mean(rel < 0.15) > 0.95, (np.median(rel), np.mean(rel < 0.15))
    mean = pk.predict_rapid(st, f.c, f.beta_hat)
    assert np.abs(ens.mean_field - mean).max() < 5 * se.max() / np.sqrt(800)


def test_bad_inputs_raise_reference_exceptions(pk):
    model = pk.CovarianceModel(1.0, 4.0, 1.0, 0.05)
    obs = _pts(12, 4)
    f = pk.fit(model, obs, np.ones(12))
    st = pk.build_setup(model, pk.build_padded_grid(UNIT, (9, 9), 2, obs), 2, obs)
    with pytest.raises(pk.DomainError):
        pk.predict_rapid(st, np.ones(11))
    with pytest.raises(pk.DomainError):
        pk.fit(model, obs, np.ones(11))
    with pytest.raises(pk.DomainError):
        pk.fit(model, obs, np.ones(12), np.column_stack([np.ones(12), np.ones(12)]))   # rank deficient
    with pytest.raises(pk.DomainError):
        pk.generate_ensemble(f, st, 1, 0)
    with warnings.catch_warnings():
        warnings.simplefilter("error")
        pk.predict_rapid(st, f.c, f.beta_hat)   # no stray warnings on the hot path


def test_weights_kernel_timing_leaves_setup_unchanged(pk):
    import ctypes as C
    from paper_2605_29284_b200 import _native as N
    obs = _pts(300, 11)
    model = pk.CovarianceModel(1.0, 8.0, 1.0)
    st = pk.build_setup(model, pk.build_padded_grid(UNIT, (40, 40), 3, obs), 3, obs)
    w0, cv0 = st.weights.copy(), st.cond_var.copy()
    ms = C.c_float(0.0)
    N.call("rk_setup_time_weights", st.handle, N.stream_ptr(), 3, C.byref(ms))
    assert ms.value > 0.0
    st._cache.clear()
    assert np.array_equal(st.weights, w0) and np.array_equal(st.cond_var, cv0)


_WEIGHTS_CHILD = r"""
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2605_29284_b200 as pk
obs = np.random.default_rng(12).uniform(0.05, 0.95, size=(257, 2))
out = {}
for L, nu in [(1, 0.5), (2, 1.5), (3, 1.0), (4, 2.5)]:
    m = pk.CovarianceModel(1.0, 9.0, nu)
    st = pk.build_setup(m, pk.build_padded_grid((0, 1, 0, 1), (48, 40), L, obs), L, obs)
    out[f"w{L}"], out[f"c{L}"], out[f"i{L}"] = st.weights, st.cond_var, st.neighbor_indices
np.savez(sys.argv[2], **out)
"""


def test_specialised_weights_kernel_matches_generic(pk, tmp_path):
    """weights_kernel_l<L> (unrolled, reciprocal diagonal, 32/M observations per warp) against
    the runtime-M kernel (RK_WEIGHTS_GENERIC=1, per-step division) for L = 1..4: identical
    stencils; weights equal to the conditioning of K_N (the L = 4, nu = 2.5 factor is
    ill-conditioned, so two correctly rounded substitutions differ at ~1e-11); conditional
    variances (well conditioned) to 1e-12."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {}
    for gen in ("0", "1"):
        f = tmp_path / f"w{gen}.npz"
        env = dict(os.environ, RK_WEIGHTS_GENERIC=gen)
        subprocess.run([sys.executable, "-c", _WEIGHTS_CHILD, root, str(f)], env=env, check=True)
        res[gen] = np.load(f)
    for L in range(1, 5):
        a, b = res["0"], res["1"]
        assert np.array_equal(a[f"i{L}"], b[f"i{L}"])
        w_scale = np.abs(b[f"w{L}"]).max()
        assert np.abs(a[f"w{L}"] - b[f"w{L}"]).max() <= (1e-12 if L < 4 else 1e-9) * w_scale, L
        assert np.abs(a[f"c{L}"] - b[f"c{L}"]).max() <= 1e-12, L
