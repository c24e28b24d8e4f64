"""Randomised parity sweep: predict_rapid (and one CS draw) on the GPU against the oracle over
a spread of smoothness (half-integer and Bessel), neighbour orders, ragged grids, clustered
and boundary observations, and covariates — FFT lengths of every radix mix the planner makes."""
import numpy as np
import pytest

from oracle import rk_oracle as ro
from rk_testutil import has_gpu, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]

UNIT = (0.0, 1.0, 0.0, 1.0)


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    nu = float(rng.choice([0.5, 0.75, 1.0, 1.5, 2.0, 2.5]))
    L = int(rng.integers(1, 5))
    dims = (int(rng.integers(5, 140)), int(rng.integers(5, 140)))
    n = int(rng.integers(5, 400))
    if seed % 3 == 0:       # clustered
        obs = np.clip(rng.normal(0.5, 0.08, size=(n, 2)), 0, 1)
    elif seed % 3 == 1:     # touching the boundary
        obs = rng.uniform(0, 1, size=(n, 2))
        obs[: n // 5] = np.round(obs[: n // 5])
    else:
        obs = rng.uniform(0, 1, size=(n, 2))
    alpha = float(rng.uniform(3.0, 30.0))
    p = int(rng.integers(0, 4))
    return rng, nu, L, dims, obs, alpha, p


@pytest.mark.parametrize("seed", range(24))
def test_random_configs_match_oracle(seed):
    import paper_2605_29284_b200 as pk
    rng, nu, L, dims, obs, alpha, p = _case(seed)
    model = pk.CovarianceModel(1.0, alpha, nu, 0.05)
    om = ro.Model(1.0, alpha, nu, 0.05)
    grid = pk.build_padded_grid(UNIT, dims, L, obs)
    og = ro.make_grid(UNIT, dims, L, obs)
    assert grid.pad == og.pad
    st = pk.build_setup(model, grid, L, obs)
    ost = ro.rapid_setup(om, og, L, obs)
    assert np.array_equal(st.neighbor_indices, ost.indices)
    c = rng.normal(size=obs.shape[0])
    if p == 0:
        beta, xg = None, None
    elif p == 1:
        beta, xg = np.array([0.4]), None
    else:
        nodes = grid.interior_nodes()
        xg = np.column_stack([np.ones(len(nodes)), nodes[:, 0], nodes[:, 1]][:p])
        beta = rng.normal(size=p)
    ours = pk.predict_rapid(st, c, beta, xg)
    ref = ro.predict(ost, c, beta, xg)
    assert rel_err(ours, ref) < 1e-10, (seed, nu, L, dims, p)


@pytest.mark.parametrize("dims,L,nu,alpha", [((24, 26), 2, 1.0, 12.0),    # torus 54 x 54 (not 4-aligned rows)
                                             ((38, 36), 2, 0.5, 20.0),    # 81 x 81: odd rows
                                             ((30, 50), 3, 1.5, 9.0),     # mixed sizes
                                             ((60, 20), 1, 2.5, 25.0),
                                             ((25, 31), 1, 1.0, 15.0)])   # odd M1: last column unpaired
def test_unconditional_fields_any_torus_alignment(dims, L, nu, alpha):
    """The fused Philox + row-IFFT generator (rows whose first word is not Philox-block
    aligned when ps1 % 4 != 0) and the paired column pass against the oracle's field."""
    import paper_2605_29284_b200 as pk
    from paper_2605_29284_b200.simulate import embedding_dims
    rng = np.random.default_rng(dims[0] * 100 + dims[1])
    obs = rng.uniform(0, 1, size=(30, 2))
    model = pk.CovarianceModel(1.0, alpha, nu, 0.05)
    om = ro.Model(1.0, alpha, nu, 0.05)
    grid = pk.build_padded_grid(UNIT, dims, L, obs)
    og = ro.make_grid(UNIT, dims, L, obs)
    root = ro.embedding_root(om, og)
    assert embedding_dims(model, grid)[:2] == (root[0], root[1])
    for seed in (3, 2 ** 63 + 5):
        ours = pk.sim_unconditional_grid(model, grid, seed)
        ref = ro.uncond_field(om, og, seed, root)
        assert rel_err(ours, ref) < 1e-10, (dims, seed, root[:2])
