"""Parity at BASELINE.json's full sizes through size-independent properties (the numpy oracle
cannot run a 4374^2 torus per test in seconds):

* configs[2] (n = 20000, 2048^2 grid, L = 4, nu = 2.5, 4374^2 torus): the predicted field at
  sampled interior nodes against the DIRECT sum  sum_nodes c*[node] sigma2 phi(alpha |node - g|)
  + beta  (the reference's own FFT-path oracle, test_rapid.py:47-57 / test_acceptance.py:51-72,
  restated at full size; phi from the numpy oracle), linearity in c, and c = 0 -> exactly the
  fixed part;
* configs[3] (n = 5000, 512^2, L = 3, CS torus 2304^2): ensemble mean / SE bitwise identical
  whatever the realization batch size, and the SE finite and positive;
* configs[4]'s largest cell (n = 50000, 4096^2, 8748^2 torus): field vs the direct sum.
"""
import numpy as np
import pytest

from rk_testutil import has_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def pk():
    import paper_2605_29284_b200 as pk
    return pk


@pytest.fixture(scope="module")
def cfg3(pk):
    from paper_2605_29284_b200 import workloads
    wl = workloads.cfg3()
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = pk.build_setup(model, grid, wl.L, wl.obs)
    return wl, model, grid, st


def test_cfg3_field_matches_direct_sum(pk, cfg3):
    from oracle import rk_oracle as ro
    wl, model, grid, st = cfg3
    assert st.embed_dims == (4374, 4374)
    rng = np.random.default_rng(31)
    c = rng.normal(size=wl.obs.shape[0])
    beta = np.array([0.75])
    field = pk.predict_rapid(st, c, beta)
    cstar = st.coefficients_to_grid(c)
    iy, ix = np.nonzero(cstar)
    vals = cstar[iy, ix]
    hx, hy = grid.spacing
    l, _, b, _ = grid.pad
    m1, m2 = grid.interior_dims
    scale = np.abs(field).max()
    # corners, edges and random interior nodes
    targets = [(0, 0), (m1 - 1, m2 - 1), (0, m2 - 1), (m1 // 2, 0)]
    targets += [tuple(int(v) for v in rng.integers(0, [m1, m2])) for _ in range(6)]
    for jx, jy in targets:
        d = np.hypot((ix - (jx + l)) * hx, (iy - (jy + b)) * hy)
        ref = float(np.dot(vals, model.sigma2 * ro.matern_phi(wl.alpha * d, wl.nu))) + beta[0]
        assert abs(field[jy, jx] - ref) <= 1e-10 * scale, (jx, jy, field[jy, jx], ref)


def test_cfg3_linearity_and_zero(pk, cfg3):
    wl, model, grid, st = cfg3
    rng = np.random.default_rng(32)
    n = wl.obs.shape[0]
    c1, c2 = rng.normal(size=n), rng.normal(size=n)
    lhs = pk.predict_rapid(st, 1.7 * c1 + c2, np.array([0.0]))
    rhs = 1.7 * pk.predict_rapid(st, c1, np.array([0.0])) + pk.predict_rapid(st, c2, np.array([0.0]))
    assert np.abs(lhs - rhs).max() <= 1e-10 * np.abs(lhs).max()
    z = pk.predict_rapid(st, np.zeros(n), np.array([2.5]))
    assert np.all(z == 2.5)


def test_cfg4_ensemble_batch_independent(pk):
    from paper_2605_29284_b200 import workloads
    from paper_2605_29284_b200.distributed import generate_ensemble_sharded
    wl = workloads.cfg4()
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    f = pk.fit(model, wl.obs, wl.z)
    st = pk.build_setup(model, pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs), wl.L, wl.obs)
    a = generate_ensemble_sharded(f, st, 24, 7, batch=8, host=True)
    b = generate_ensemble_sharded(f, st, 24, 7, batch=3, host=True)
    assert np.array_equal(a.mean_field, b.mean_field)
    assert np.array_equal(a.empirical_se, b.empirical_se)
    assert np.all(np.isfinite(a.empirical_se)) and a.empirical_se.min() >= 0.0 and a.empirical_se.max() > 0.0


def test_cfg5_largest_cell_matches_direct_sum(pk):
    """configs[4]'s largest cell (n = 50000, 4096^2 grid, L = 4, nu = 1.5; an 8748^2 torus):
    random coefficients (predict does not need the n x n fit), field against the direct sum at
    sampled nodes."""
    from oracle import rk_oracle as ro
    from paper_2605_29284_b200 import workloads
    wl = workloads.cfg5(nu=1.5, L=4, m=4096)
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = pk.build_setup(model, grid, wl.L, wl.obs)
    assert max(st.embed_dims) >= 8192
    rng = np.random.default_rng(51)
    c = rng.normal(size=wl.obs.shape[0])
    field = pk.predict_rapid(st, c, np.array([-0.5]))
    cstar = st.coefficients_to_grid(c)
    iy, ix = np.nonzero(cstar)
    vals = cstar[iy, ix]
    hx, hy = grid.spacing
    l, _, b, _ = grid.pad
    m1, m2 = grid.interior_dims
    scale = np.abs(field).max()
    for jx, jy in [(0, 0), (m1 - 1, m2 - 1)] + [tuple(int(v) for v in rng.integers(0, [m1, m2])) for _ in range(4)]:
        d = np.hypot((ix - (jx + l)) * hx, (iy - (jy + b)) * hy)
        ref = float(np.dot(vals, model.sigma2 * ro.matern_phi(wl.alpha * d, wl.nu))) - 0.5
        assert abs(field[jy, jx] - ref) <= 1e-10 * scale, (jx, jy, field[jy, jx], ref)
