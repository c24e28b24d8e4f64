"""BASELINE configs[4]: the nu x L x grid factorial (36 cells, n = 50000) against the CPU oracle.

Every cell: stencil indices bit-exact against rapid.py:200-214 (oracle `rapid_weights`).
* 256^2 and 1024^2 grids: the full predicted field against the oracle's FFT path
  (rapid.py:252-261), <= 1e-10 relative to max|reference|;
* 4096^2 grids (tori up to 8748^2; the numpy oracle's spectrum + FFTs take ~15 s per cell): the
  field at corner / edge / random interior nodes against the DIRECT sum
  sum_nodes c*_oracle[node] sigma2 phi(alpha |node - g|) + beta, with c* scattered from the
  ORACLE's weights -- the definition the reference's FFT path is itself tested against
  (test_rapid.py:47-57), so both our weights kernel and our convolution are on the checked path.
"""
import numpy as np
import pytest

from oracle import rk_oracle as ro
from rk_testutil import has_gpu, rel_err

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not has_gpu(), reason="needs a CUDA device")]
TOL = 1e-10

CELLS = [(nu, L, m) for m in (256, 1024, 4096) for nu in (0.5, 1.5, 2.5) for L in (1, 2, 3, 4)]


@pytest.fixture(scope="module")
def pk():
    import paper_2605_29284_b200 as pk
    return pk


@pytest.mark.parametrize("nu,L,m", CELLS, ids=[f"nu{nu}-L{L}-{m}" for nu, L, m in CELLS])
def test_factorial_cell(pk, nu, L, m):
    from paper_2605_29284_b200 import workloads
    wl = workloads.cfg5(nu=nu, L=L, m=m)
    n = wl.obs.shape[0]
    model = pk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    grid = pk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = pk.build_setup(model, grid, wl.L, wl.obs)
    om = ro.Model(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    og = ro.make_grid(wl.domain, wl.dims, wl.L, wl.obs)
    rng = np.random.default_rng(1000 * m + 10 * L + int(2 * nu))
    c = rng.normal(size=n)
    beta = np.array([0.3])
    field = pk.predict_rapid(st, c, beta)
    assert field.shape == (m, m)
    if m <= 1024:
        ost = ro.rapid_setup(om, og, L, wl.obs)
        assert np.array_equal(st.neighbor_indices, ost.indices)
        assert tuple(st.embed_dims) == tuple(ost.embed_dims)
        assert rel_err(field, ro.predict(ost, c, beta)) < TOL
        return
    chol, _ = ro.kn_factor(om, ro.kn_matrix(om, og, L), L)
    _, idx, w, _ = ro.rapid_weights(om, og, L, wl.obs, chol)
    assert np.array_equal(st.neighbor_indices, idx)
    M1, M2 = og.total_dims
    cstar = np.zeros(M1 * M2)
    np.add.at(cstar, idx.ravel(), (w * c[:, None]).ravel())
    nz = np.nonzero(cstar)[0]
    vals = cstar[nz]
    iy, ix = nz // M1, nz % M1
    hx, hy = grid.spacing
    l, _, b, _ = grid.pad
    m1, m2 = grid.interior_dims
    scale = np.abs(field).max()
    targets = [(0, 0), (m1 - 1, m2 - 1), (0, m2 - 1), (m1 // 2, 0)]
    targets += [tuple(int(v) for v in rng.integers(0, [m1, m2])) for _ in range(4)]
    for jx, jy in targets:
        d = np.hypot((ix - (jx + l)) * hx, (iy - (jy + b)) * hy)
        ref = float(np.dot(vals, om.sigma2 * ro.matern_phi(wl.alpha * d, wl.nu))) + beta[0]
        assert abs(field[jy, jx] - ref) <= TOL * scale, (jx, jy, field[jy, jx], ref)
