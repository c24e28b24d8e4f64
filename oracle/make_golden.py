"""Generate tests/golden/*.npz by running the REAL reference package in this container.

Usage (build container only; /root/reference does not exist on the GPU box):
    python oracle/make_golden.py

Every fixture stores the inputs and the reference's outputs for one case of the
hot path.  tests/test_oracle_golden.py pins oracle/rk_oracle.py to these, and
the GPU parity tests compare the CUDA path against both.
"""

from __future__ import annotations

import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import rapidkrig as rk  # noqa: E402  (the reference)
from rapidkrig import bessel, rapid, simulate  # noqa: E402

from paper_2605_29284_b200 import workloads  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
UNIT = (0.0, 1.0, 0.0, 1.0)


def save(name, **arrays):
    path = os.path.join(OUT, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


def gen_matern():
    nus = np.array([0.5, 1.0, 1.5, 2.5, 0.3, 0.75, 1.25, 3.7, 5.5, 12.5, 2.0])
    d = np.concatenate([[0.0, 1e-13, 1e-12, 2e-12, 1.9999999, 2.0, 2.0000001],
                        np.logspace(-10, 2.3, 400)])
    phi = np.stack([bessel.matern_correlation(d, nu) for nu in nus])
    kv_nu = np.array([0.2, 0.5, 1.0, 1.7, 3.0])
    xk = np.logspace(-3, 2, 60)
    kv = np.stack([bessel.kv(nu, xk) for nu in kv_nu])
    save("matern", nus=nus, d=d, phi=phi, kv_nu=kv_nu, kv_x=xk, kv=kv)


def gen_grids():
    cases = []
    rng = np.random.default_rng(11)
    for k, (dims, L) in enumerate([((20, 20), 1), ((20, 20), 2), ((20, 20), 4), ((9, 9), 4),
                                   ((12, 7), 3), ((64, 64), 8), ((33, 40), 2)]):
        obs = rng.uniform(0, 1, size=(40, 2))
        obs[0] = (0.0, 0.5)
        obs[1] = (1.0, 0.5)
        obs[2] = (0.5, 0.0)
        obs[3] = (0.5, 1.0)
        obs[4] = (0.0, 0.0)
        obs[5] = (1.0, 1.0)
        hx = 1.0 / (dims[0] - 1)
        hy = 1.0 / (dims[1] - 1)
        obs[6] = (3 * hx, 2 * hy)               # on a node
        obs[7] = (3 * hx + 1e-12, 5 * hy - 1e-12)  # snapped to a node
        obs[8] = (0.5 * hx, 0.5 * hy)
        grid = rk.build_padded_grid(UNIT, dims, L, obs)
        nbs = [rk.neighborhood(grid, o, L) for o in obs]
        idx = np.stack([nb.indices for nb in nbs])
        off = np.array([nb.local_offset for nb in nbs])
        cases.append(dict(dims=np.array(dims), L=L, obs=obs, pad=np.array(grid.pad),
                          indices=idx, offsets=off))
    save("grids", n=len(cases), **{f"{k}_{i}": v for i, c in enumerate(cases) for k, v in c.items()})


def _setup_case(model, dims, L, obs, c, beta=None, xg=None):
    grid = rk.build_padded_grid(UNIT, dims, L, obs)
    st = rk.build_setup(model, grid, L, obs)
    field = rk.predict_rapid(st, c, beta, xg)
    cstar = st.coefficients_to_grid(c)
    return dict(sigma2=model.sigma2, alpha=model.alpha, nu=model.nu, tau2=model.tau2,
                dims=np.array(dims), L=L, obs=obs, pad=np.array(grid.pad),
                indices=st.neighbor_indices, weights=st.weights, cond_var=st.cond_var,
                kn=rapid.neighbor_cov(model, grid, L),
                embed_dims=np.array(st.embed_dims), spectrum=st.filter_spectrum,
                c=c, beta=(np.zeros(0) if beta is None else np.asarray(beta)),
                xg=(np.zeros((0, 0)) if xg is None else xg), cstar=cstar, field=field)


def gen_setups():
    rng = np.random.default_rng(12)
    cases = {}
    # nu=1.5, L=2, small grid, intercept
    obs = rng.uniform(0, 1, size=(50, 2))
    cases["s0"] = _setup_case(rk.CovarianceModel(1.0, 6.0, 1.5, 0.1), (20, 20), 2, obs,
                              rng.normal(size=50), np.array([0.7]))
    # nu=1.0 (Bessel), L=3, boundary points, covariates
    obs = rng.uniform(0, 1, size=(60, 2))
    obs[:4] = [(0, 0), (1, 1), (0, 1), (1, 0)]
    dims = (23, 19)
    g = rk.build_padded_grid(UNIT, dims, 3, [])
    nodes = g.interior_nodes()
    xg = np.column_stack([np.ones(len(nodes)), nodes[:, 0], nodes[:, 1]])
    cases["s1"] = _setup_case(rk.CovarianceModel(1.3, 1 / 0.15, 1.0, 0.05), dims, 3, obs,
                              rng.normal(size=60), np.array([0.5, 1.0, -1.0]), xg)
    # nu=2.5, L=4, odd torus, no beta
    obs = rng.uniform(0, 1, size=(40, 2))
    cases["s2"] = _setup_case(rk.CovarianceModel(1.0, 20.0, 2.5, 0.01), (30, 30), 4, obs,
                              rng.normal(size=40))
    # nu=0.5, L=1
    obs = rng.uniform(0, 1, size=(30, 2))
    cases["s3"] = _setup_case(rk.CovarianceModel(2.0, 4.0, 0.5, 0.0), (16, 11), 1, obs,
                              rng.normal(size=30), np.array([-1.5]))
    # on-node observations
    g0 = rk.build_padded_grid(UNIT, (15, 15), 2, [])
    nodes = g0.interior_nodes()
    obs = nodes[rng.choice(len(nodes), size=20, replace=False)]
    cases["s4"] = _setup_case(rk.CovarianceModel(1.0, 6.0, 1.5, 0.1), (15, 15), 2, obs,
                              rng.normal(size=20), np.array([0.2]))
    # non-half-integer nu = 0.75 (Bessel with mu != 0)
    obs = rng.uniform(0, 1, size=(35, 2))
    cases["s5"] = _setup_case(rk.CovarianceModel(1.0, 5.0, 0.75, 0.1), (18, 14), 2, obs,
                              rng.normal(size=35), np.array([1.0]))
    for name, cs in cases.items():
        save("setup_" + name, **cs)


def gen_config(name):
    wl = workloads.CONFIGS[name]()
    model = rk.CovarianceModel(wl.sigma2, wl.alpha, wl.nu, wl.tau2)
    krig = rk.fit(model, wl.obs, wl.z, wl.X)
    grid = rk.build_padded_grid(wl.domain, wl.dims, wl.L, wl.obs)
    st = rk.build_setup(model, grid, wl.L, wl.obs)
    xg = workloads.grid_covariates_for(grid.interior_nodes(), wl.grid_covariates)
    field = rk.predict_rapid(st, krig.c, krig.beta_hat, xg)
    save(name, obs=wl.obs, z=wl.z, c=krig.c, beta=krig.beta_hat, pad=np.array(grid.pad),
         embed_dims=np.array(st.embed_dims), base=st.neighbor_indices[:, 0],
         cond_var=st.cond_var, field=field)


def gen_rng():
    seeds = np.array([0, 1, 7, 42, 2**63, 2**64 - 1, 123456789012345], dtype=np.uint64)
    js = np.array([0, 1, 2, 101, 202, 1023, 10**9])
    sub = np.array([[simulate.draw_seed(int(s), int(j)) for j in js] for s in seeds], dtype=np.uint64)
    raw = []
    normals = []
    for s in seeds:
        for stream in (0, 1):
            gen = simulate._rng(int(s), stream)
            raw.append(np.random.Philox(key=(int(s) & ((1 << 64) - 1)) + (stream << 64)).random_raw(37))
            normals.append(simulate._std_normals(gen, 37))
    save("rng", seeds=seeds, js=js, sub=sub, raw=np.stack(raw), normals=np.stack(normals))


def gen_cs():
    rng = np.random.default_rng(13)
    model = rk.CovarianceModel(1.0, 5.0, 1.0, 0.1)
    obs = rng.uniform(0, 1, size=(30, 2))
    z = rng.normal(size=30)
    krig = rk.fit(model, obs, z)
    grid = rk.build_padded_grid(UNIT, (16, 16), 2, obs)
    st = rk.build_setup(model, grid, 2, obs)
    p1, p2, root = simulate._embedding_root(model, grid)
    g = simulate.sim_unconditional_grid(model, grid, 5)
    zs = simulate.sim_obs_local(model, st, g, 6)
    bs, cs = rk.refit_coefficients(krig, zs)
    draw = simulate.conditional_draw(krig, st, 9)
    ens = simulate.generate_ensemble(krig, st, 4, 3)
    save("cs_small", sigma2=1.0, alpha=5.0, nu=1.0, tau2=0.1, obs=obs, z=z, dims=np.array([16, 16]),
         L=2, chol_M=krig.chol_M, X=krig.X, c=krig.c, beta=krig.beta_hat,
         embed=np.array([p1, p2]), root=root, g=g, zs=zs, bs=bs, cs=cs, draw=draw,
         ens_draws=ens.draws, ens_mean=ens.mean_field, ens_se=ens.empirical_se)
    # covariates + nu = 1.5 + L = 3
    model = rk.CovarianceModel(1.0, 8.0, 1.5, 0.05)
    obs = rng.uniform(0, 1, size=(40, 2))
    X = np.column_stack([np.ones(40), obs[:, 0], obs[:, 1]])
    z = X @ np.array([0.5, 1.0, -1.0]) + rng.normal(size=40)
    krig = rk.fit(model, obs, z, X)
    dims = (20, 18)
    grid = rk.build_padded_grid(UNIT, dims, 3, obs)
    st = rk.build_setup(model, grid, 3, obs)
    nodes = grid.interior_nodes()
    xg = np.column_stack([np.ones(len(nodes)), nodes[:, 0], nodes[:, 1]])
    ens = simulate.generate_ensemble(krig, st, 3, 77, grid_covariates=xg)
    save("cs_cov", sigma2=1.0, alpha=8.0, nu=1.5, tau2=0.05, obs=obs, z=z, X=X, dims=np.array(dims),
         L=3, chol_M=krig.chol_M, c=krig.c, beta=krig.beta_hat, xg=xg,
         ens_draws=ens.draws, ens_mean=ens.mean_field, ens_se=ens.empirical_se)
    # embedding that doubles (reference test_simulate.py:188-201)
    model = rk.CovarianceModel(1.0, 4.0, 1.0)
    grid = rk.build_padded_grid(UNIT, (24, 24), 2, [])
    p1, p2, _ = simulate._embedding_root(model, grid)
    g = simulate.sim_unconditional_grid(model, grid, 3)
    save("cs_doubling", sigma2=1.0, alpha=4.0, nu=1.0, dims=np.array([24, 24]), L=2,
         embed=np.array([p1, p2]), g=g)


def gen_exact_targets():
    """predict_exact / kriging_se_exact (exact.py:132-175) at scattered targets, for a fit with
    covariates [1, x, y] (nu = 1.0, Bessel path) and an intercept-only fit (nu = 2.5); targets
    include observation locations themselves and points outside the data hull."""
    rng = np.random.default_rng(77)
    out = {}
    for tag, nu, p in (("cov", 1.0, 3), ("icpt", 2.5, 1)):
        obs = rng.uniform(0, 1, size=(160, 2))
        X = np.column_stack([np.ones(160), obs]) if p == 3 else None
        model = rk.CovarianceModel(sigma2=1.3, alpha=6.0, nu=nu, tau2=0.04)
        z = 0.5 + np.sin(5 * obs[:, 0]) * np.cos(3 * obs[:, 1]) + rng.normal(0, 0.2, 160)
        krig = rk.fit(model, obs, z, X)
        tg = np.vstack([rng.uniform(-0.1, 1.1, size=(400, 2)), obs[:20]])
        xt = np.column_stack([np.ones(len(tg)), tg]) if p == 3 else None
        out.update({f"{tag}_obs": obs, f"{tag}_z": z, f"{tag}_nu": nu, f"{tag}_targets": tg,
                    f"{tag}_xt": xt if xt is not None else np.zeros((0, 0)),
                    f"{tag}_X": X if X is not None else np.zeros((0, 0)),
                    f"{tag}_chol": krig.chol_M, f"{tag}_beta": krig.beta_hat, f"{tag}_c": krig.c,
                    f"{tag}_pred": rk.predict_exact(krig, tg, xt),
                    f"{tag}_se": rk.kriging_se_exact(krig, tg, xt)})
    save("exact_targets", sigma2=1.3, alpha=6.0, tau2=0.04, **out)


CLI_RUNS = {
    "predict_rapid": ["predict", "--grid", "32x24", "--L", "3", "--covariates", "1+x+y"],
    "predict_exact": ["predict", "--grid", "32x24", "--method", "exact", "--domain", "0,1,0,1"],
    "simulate": ["simulate", "--grid", "32x32", "--draws", "10", "--seed", "7", "--save-draws"],
}
CLI_MODEL = ["--sigma2", "1.0", "--alpha", "5.0", "--nu", "1.0", "--tau2", "0.05"]


def gen_cli():
    """The reference CLI (cli.py) on a 60-point file (test_acceptance.py:246-266 style):
    RKGRID1 outputs of predict (rapid with covariates, exact) and simulate."""
    from rapidkrig.cli import cli_main
    rng = np.random.default_rng(6)
    n = 60
    x, y = rng.uniform(0, 1, n), rng.uniform(0, 1, n)
    z = np.sin(3 * x) + np.cos(2 * y) + 0.1 * rng.normal(size=n)
    d = os.path.join(OUT, "cli")
    os.makedirs(d, exist_ok=True)
    obs = os.path.join(d, "obs.csv")
    with open(obs, "w", encoding="utf-8") as fh:
        fh.write("x,y,z\n")
        for row in zip(x, y, z):
            fh.write(",".join(f"{v:.17g}" for v in row) + "\n")
    for name, args in CLI_RUNS.items():
        out = os.path.join(d, name + ".rkg")
        assert cli_main([*args, "--obs", obs, "--out", out, *CLI_MODEL]) == 0
        print("wrote", out, os.path.getsize(out))


def gen_misc():
    ks = np.arange(1, 1200)
    save("fft_len", n=ks, p=np.array([rapid.next_fft_len(int(k)) for k in ks]))


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    gen_matern()
    gen_grids()
    gen_setups()
    gen_rng()
    gen_cs()
    gen_misc()
    gen_exact_targets()
    gen_cli()
    gen_config("cfg1")
    gen_config("cfg2")
