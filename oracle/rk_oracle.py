"""CPU oracle for the rapid-Kriging hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference package ``rapidkrig`` 0.1.0
(`/root/reference/pkg/src/rapidkrig`) for the functions on the north-star path:
Matern correlation, padded grid + stencil, rapid setup (weights, conditional
variance, filter spectrum), rapid predict (scatter + circulant FFT convolution +
fixed part), and the conditional-simulation chain (splitmix64 sub-seeds,
Philox4x64-10 normals, circulant-embedding field, local observation simulation,
GLS refit, ensemble moments).  Each function cites the reference file:line it
follows.

Who may use it: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs, as the CHECKER or the timed CPU
baseline.  The product package ``paper_2605_29284_b200`` never imports it.

Pinning: the oracle is checked against golden vectors produced by running the
real reference in the build container (``oracle/make_golden.py`` →
``tests/golden/*.npz``; test ``tests/test_oracle_golden.py``).  Third-party
arithmetic the reference delegates (numpy pocketfft FFTs, numpy ``Philox``,
``scipy.special.ndtri``, LAPACK Cholesky/triangular solves) is called here the
same way the reference calls it; the Philox4x64-10 block function is
additionally restated from Salmon et al. (SC'11) in ``philox4x64_block`` and
pinned bit-for-bit against ``numpy.random.Philox``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import scipy.linalg
from scipy.special import ndtri

# --------------------------------------------------------------------------
# errors (reference errors.py:4-17) — same class names so tests read alike
# --------------------------------------------------------------------------


class OracleError(Exception):
    pass


class OracleDomainError(OracleError):
    pass


class OracleNumericError(OracleError):
    pass


class OracleInternalError(OracleError):
    pass


SNAP = 1.0e-9          # gridding.py:35 NODE_SNAP_TOL
EPS_CONV = 1.0e-15     # bessel.py:31
EULER = 0.5772156649015329

# --------------------------------------------------------------------------
# Matern correlation  (bessel.py:37-278)
# --------------------------------------------------------------------------


def temme_constants(mu: float):
    """bessel.py:37-47 — 1/G(1+mu), 1/G(1-mu), Gamma1, Gamma2."""
    inv_gp = 1.0 / math.gamma(1.0 + mu)
    inv_gm = 1.0 / math.gamma(1.0 - mu)
    g1 = -EULER if abs(mu) < 1.0e-6 else (inv_gm - inv_gp) / (2.0 * mu)
    g2 = 0.5 * (inv_gm + inv_gp)
    return inv_gp, inv_gm, g1, g2


def _k_pair_small_x(mu: float, x: np.ndarray):
    """bessel.py:50-101 — Temme series for (K_mu, K_mu+1), 0 < x <= 2.

    Every element iterates until its own term drops below 1e-15 of its sum and
    keeps the sums of THAT iteration (per-element freeze, bessel.py:82-92).
    """
    inv_gp, inv_gm, g1, g2 = temme_constants(mu)
    hx = 0.5 * x
    ln2x = -np.log(hx)
    sg = mu * ln2x
    pm = math.pi * mu
    fct = 1.0 if abs(pm) < 1.0e-12 else pm / math.sin(pm)
    safe = np.where(sg == 0.0, 1.0, sg)
    shr = np.where(np.abs(sg) < 1.0e-12, 1.0, np.sinh(sg) / safe)
    f = fct * (g1 * np.cosh(sg) + g2 * shr * ln2x)
    ex = np.exp(sg)
    p = 0.5 * ex / inv_gp
    q = 0.5 / (ex * inv_gm)
    cc = np.ones_like(x)
    dd = hx * hx
    s0 = f.copy()
    s1 = p.copy()
    res0 = np.full_like(x, np.nan)
    res1 = np.full_like(x, np.nan)
    live = np.ones(x.shape, dtype=bool)
    mu2 = mu * mu
    for i in range(1, 501):
        f = (i * f + p + q) / (i * i - mu2)
        cc = cc * (dd / i)
        p = p / (i - mu)
        q = q / (i + mu)
        term = cc * f
        s0 = s0 + term
        s1 = s1 + cc * (p - i * f)
        hit = live & (np.abs(term) < np.abs(s0) * EPS_CONV)
        res0[hit] = s0[hit]
        res1[hit] = s1[hit]
        live &= ~hit
        if not live.any():
            break
    else:
        raise OracleNumericError("Temme series did not converge")
    return res0, res1 * (2.0 / x)


def _k_pair_large_x(mu: float, x: np.ndarray):
    """bessel.py:104-171 — Steed CF2 (Thompson-Barnett), x > 2, per-element freeze."""
    a1 = 0.25 - mu * mu
    b = 2.0 * (1.0 + x)
    d = 1.0 / b
    h = d.copy()
    dh = d.copy()
    qa = np.zeros_like(x)
    qb = np.ones_like(x)
    q = np.full_like(x, a1)
    cs = a1
    an = -a1
    s = 1.0 + q * dh
    out_h = np.full_like(x, np.nan)
    out_s = np.full_like(x, np.nan)
    live = np.ones(x.shape, dtype=bool)
    for i in range(2, 20001):
        an -= 2 * (i - 1)
        cs = -an * cs / i
        qn = (qa - b * qb) / an
        qa, qb = qb, qn
        q = q + cs * qb
        b = b + 2.0
        d = 1.0 / (d * an + b)
        dh = (b * d - 1.0) * dh
        h = h + dh
        ds = q * dh
        s = s + ds
        hit = live & (np.abs(ds) < np.abs(s) * EPS_CONV)
        out_h[hit] = h[hit]
        out_s[hit] = s[hit]
        live &= ~hit
        if not live.any():
            break
    else:
        raise OracleNumericError("CF2 did not converge")
    k0 = np.sqrt(np.pi / (2.0 * x)) * np.exp(-x) / out_s
    k1 = k0 * (mu + x + 0.5 - a1 * out_h) / x
    return k0, k1


def k_pair(mu: float, x: np.ndarray):
    """bessel.py:174-184 — split at x = 2."""
    x = np.asarray(x, dtype=float)
    k0 = np.empty_like(x)
    k1 = np.empty_like(x)
    lo = x <= 2.0
    if lo.any():
        k0[lo], k1[lo] = _k_pair_small_x(mu, x[lo])
    if (~lo).any():
        k0[~lo], k1[~lo] = _k_pair_large_x(mu, x[~lo])
    return k0, k1


def half_integer_n(nu: float):
    """bessel.py:216-221."""
    n = int(round(nu - 0.5))
    return n if (0 <= n <= 12 and abs(nu - (n + 0.5)) < 1.0e-12) else None


def half_integer_coeffs(n: int):
    """Constants of bessel.py:224-234 (computed by exact-integer true division)."""
    coef = [math.factorial(n + i) / (math.factorial(i) * math.factorial(n - i))
            for i in range(n + 1)]
    return coef, math.factorial(n) / math.factorial(2 * n)


def matern_phi(d, nu: float) -> np.ndarray:
    """bessel.py:258-278 (+ _matern_half_integer 224-234, matern_correlation_bessel 237-255)."""
    if nu <= 0:
        raise OracleDomainError("nu must be positive")
    d = np.atleast_1d(np.asarray(d, dtype=float))
    if (d < 0).any():
        raise OracleDomainError("negative distance")
    out = np.ones_like(d)
    sel = d > 1.0e-12
    if not sel.any():
        return out
    x = d[sel]
    nh = half_integer_n(nu)
    if nh is not None:
        coef, pref = half_integer_coeffs(nh)
        acc = np.zeros_like(x)
        tx = 2.0 * x
        for cf in coef:
            acc = acc * tx + cf
        phi = pref * np.exp(-x) * acc
    else:
        nl = int(nu + 0.5)
        mu = nu - nl
        k0, k1 = k_pair(mu, x)
        hx = 0.5 * x
        sc = hx ** mu
        r0 = k0 * sc
        r1 = k1 * sc * hx
        h2 = hx * hx
        for j in range(nl):
            r0, r1 = r1, h2 * r0 + (mu + j + 1) * r1
        phi = 2.0 * r0 / math.gamma(nu)
    out[sel] = np.clip(phi, 0.0, 1.0)
    return out


@dataclass(frozen=True)
class Model:
    """covariance.py:50-89 — k(d) = sigma2 * phi(alpha * d)."""
    sigma2: float
    alpha: float
    nu: float
    tau2: float = 0.0

    def cov(self, dist):
        return self.sigma2 * matern_phi(self.alpha * np.asarray(dist, dtype=float), self.nu)


# --------------------------------------------------------------------------
# padded grid and stencil  (gridding.py:38-205)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Grid:
    """gridding.py:38-111 — interior grid + (left, right, bottom, top) pads."""
    origin: tuple
    spacing: tuple
    interior_dims: tuple
    pad: tuple

    @property
    def total_dims(self):
        return (self.interior_dims[0] + self.pad[0] + self.pad[1],
                self.interior_dims[1] + self.pad[2] + self.pad[3])

    @property
    def padded_origin(self):
        return (self.origin[0] - self.pad[0] * self.spacing[0],
                self.origin[1] - self.pad[2] * self.spacing[1])

    def interior(self, field):
        m1, m2 = self.interior_dims
        return field[self.pad[2]:self.pad[2] + m2, self.pad[0]:self.pad[0] + m1]

    def interior_nodes(self):
        m1, m2 = self.interior_dims
        xs = self.origin[0] + self.spacing[0] * np.arange(m1)
        ys = self.origin[1] + self.spacing[1] * np.arange(m2)
        gx, gy = np.meshgrid(xs, ys)
        return np.column_stack([gx.ravel(), gy.ravel()])


def snap_cells(t):
    """gridding.py:123-127 — nearest node within 1e-9, else floor."""
    t = np.asarray(t, dtype=float)
    r = np.rint(t)
    return np.where(np.abs(t - r) <= SNAP, r, np.floor(t)).astype(np.int64)


def make_grid(domain, dims, L, obs) -> Grid:
    """gridding.py:130-178 — minimal data-dependent padding."""
    x0, x1, y0, y1 = (float(v) for v in domain)
    m1, m2 = int(dims[0]), int(dims[1])
    if L < 1 or m1 < max(2, 2 * L) or m2 < max(2, 2 * L) or not (x1 > x0 and y1 > y0):
        raise OracleDomainError("bad grid request")
    hx = (x1 - x0) / (m1 - 1)
    hy = (y1 - y0) / (m2 - 1)
    obs = np.asarray(obs, dtype=float).reshape(-1, 2)
    if obs.shape[0] == 0:
        return Grid((x0, y0), (hx, hy), (m1, m2), (0, 0, 0, 0))
    ok = ((obs[:, 0] >= x0 - SNAP * hx) & (obs[:, 0] <= x1 + SNAP * hx)
          & (obs[:, 1] >= y0 - SNAP * hy) & (obs[:, 1] <= y1 + SNAP * hy))
    if not ok.all():
        raise OracleDomainError(f"observation {int(np.argmin(ok))} outside the domain")
    cx = snap_cells((obs[:, 0] - x0) / hx)
    cy = snap_cells((obs[:, 1] - y0) / hy)
    pads = (max(0, int(np.max(L - 1 - cx))), max(0, int(np.max(cx + L - (m1 - 1)))),
            max(0, int(np.max(L - 1 - cy))), max(0, int(np.max(cy + L - (m2 - 1)))))
    return Grid((x0, y0), (hx, hy), (m1, m2), pads)


def stencils(grid: Grid, obs, L):
    """gridding.py:181-205, vectorised over observations.

    Returns (base, offsets): ``base`` is the flat padded index of block entry 0
    (row-major block, x fastest), ``offsets`` the (tx - cx, ty - cy) positions.
    """
    obs = np.asarray(obs, dtype=float).reshape(-1, 2)
    px0, py0 = grid.padded_origin
    hx, hy = grid.spacing
    M1, M2 = grid.total_dims
    tx = (obs[:, 0] - px0) / hx
    ty = (obs[:, 1] - py0) / hy
    inside = (tx >= -SNAP) & (tx <= M1 - 1 + SNAP) & (ty >= -SNAP) & (ty <= M2 - 1 + SNAP)
    if not inside.all():
        raise OracleDomainError("location outside padded grid coverage")
    cx = snap_cells(tx)
    cy = snap_cells(ty)
    if ((cx - (L - 1) < 0) | (cy - (L - 1) < 0) | (cx + L > M1 - 1) | (cy + L > M2 - 1)).any():
        raise OracleInternalError("stencil leaves the padded grid")
    base = (cy - (L - 1)) * M1 + (cx - (L - 1))
    return base.astype(np.int64), np.column_stack([tx - cx, ty - cy])


def expand_indices(base, M1, L):
    """Block entry m = r*2L + s sits at base + r*M1 + s (gridding.py:489-491)."""
    b = 2 * L
    r, s = np.divmod(np.arange(b * b), b)
    return base[:, None] + (r * M1 + s)[None, :]


# --------------------------------------------------------------------------
# rapid setup and predict  (rapid.py:46-261)
# --------------------------------------------------------------------------


def fft_len(n: int) -> int:
    """rapid.py:46-59 — smallest 2^a 3^b >= n."""
    if n <= 1:
        return 1
    best = None
    two = 1
    while two < 4 * n:
        v = two
        while v < n:
            v *= 3
        best = v if best is None else min(best, v)
        two *= 2
    return best


def torus_lags(grid: Grid, p1: int, p2: int):
    """rapid.py:62-69."""
    hx, hy = grid.spacing
    ix = np.arange(p1)
    iy = np.arange(p2)
    return np.hypot((np.minimum(ix, p1 - ix) * hx)[None, :],
                    (np.minimum(iy, p2 - iy) * hy)[:, None])


def filter_spectrum(model: Model, grid: Grid):
    """rapid.py:72-86 — fft2 of the wrapped lag covariance on a (2M-1)-rounded torus."""
    M1, M2 = grid.total_dims
    p1, p2 = fft_len(2 * M1 - 1), fft_len(2 * M2 - 1)
    return (p1, p2), np.fft.fft2(model.cov(torus_lags(grid, p1, p2)))


def circ_convolve(spectrum, dims, values):
    """rapid.py:89-100 — leading block of the circulant convolution."""
    p1, p2 = dims
    M2, M1 = values.shape
    buf = np.zeros((p2, p1))
    buf[:M2, :M1] = values
    return np.fft.ifft2(spectrum * np.fft.fft2(buf)).real[:M2, :M1]


def block_offsets(grid: Grid, L: int):
    """rapid.py:103-109."""
    hx, hy = grid.spacing
    gx, gy = np.meshgrid(np.arange(2 * L) * hx, np.arange(2 * L) * hy)
    return np.column_stack([gx.ravel(), gy.ravel()])


def kn_matrix(model: Model, grid: Grid, L: int):
    """rapid.py:112-117 — shared neighbour covariance, symmetrised."""
    o = block_offsets(grid, L)
    k = model.cov(np.hypot(o[:, None, 0] - o[None, :, 0], o[:, None, 1] - o[None, :, 1]))
    return 0.5 * (k + k.T)


def kn_factor(model: Model, kn, L):
    """rapid.py:120-135 — lower Cholesky, one ridge retry 1e-12 sigma2 (2L)^2.

    Returns (factor, ridge_applied)."""
    try:
        return scipy.linalg.cholesky(kn, lower=True), False
    except scipy.linalg.LinAlgError:
        ridge = 1.0e-12 * model.sigma2 * (2 * L) ** 2
        try:
            return scipy.linalg.cholesky(kn + ridge * np.eye(kn.shape[0]), lower=True), True
        except scipy.linalg.LinAlgError as err:
            raise OracleNumericError("K_N factorisation failed with ridge") from err


@dataclass
class Setup:
    """rapid.py:138-174 (fields the hot path reads)."""
    model: Model
    grid: Grid
    L: int
    chol: np.ndarray
    base: np.ndarray
    indices: np.ndarray
    weights: np.ndarray
    cond_var: np.ndarray
    embed_dims: tuple
    spectrum: np.ndarray
    ridge_applied: bool = False


def rapid_weights(model: Model, grid: Grid, L: int, obs, chol):
    """rapid.py:200-225 -- the per-observation part of build_setup (stencil indices, weights by
    cho_solve against the K_N factor, conditional variances, on-node rows, clamp)."""
    obs = np.asarray(obs, dtype=float).reshape(-1, 2)
    M1 = grid.total_dims[0]
    base, offs = stencils(grid, obs, L)
    idx = expand_indices(base, M1, L)
    px0, py0 = grid.padded_origin
    hx, hy = grid.spacing
    nx = px0 + (idx % M1) * hx
    ny = py0 + (idx // M1) * hy
    k = model.cov(np.hypot(nx - obs[:, :1], ny - obs[:, 1:2]))
    w = scipy.linalg.cho_solve((chol, True), k.T).T
    cv = model.sigma2 - np.einsum("ij,ij->i", w, k)
    node = (np.abs(offs[:, 0]) <= SNAP) & (np.abs(offs[:, 1]) <= SNAP)
    if node.any():
        w[node] = 0.0
        w[node, (L - 1) * 2 * L + (L - 1)] = 1.0
        cv[node] = 0.0
    cv = np.where((cv < 0) & (cv > -1.0e-10 * model.sigma2), 0.0, cv)
    return base, idx, w, cv


def rapid_setup(model: Model, grid: Grid, L: int, obs) -> Setup:
    """rapid.py:177-230."""
    obs = np.asarray(obs, dtype=float).reshape(-1, 2)
    if obs.shape[0] == 0:
        raise OracleDomainError("no observations")
    chol, ridged = kn_factor(model, kn_matrix(model, grid, L), L)
    base, idx, w, cv = rapid_weights(model, grid, L, obs, chol)
    dims, spec = filter_spectrum(model, grid)
    return Setup(model, grid, L, chol, base, idx, w, cv, dims, spec, ridged)


def scatter_cstar(setup: Setup, c):
    """rapid.py:164-174 — c* = A' c by np.add.at."""
    c = np.asarray(c, dtype=float).ravel()
    if c.shape[0] != setup.weights.shape[0]:
        raise OracleDomainError("coefficient length mismatch")
    M1, M2 = setup.grid.total_dims
    acc = np.zeros(M1 * M2)
    np.add.at(acc, setup.indices.ravel(), (setup.weights * c[:, None]).ravel())
    return acc.reshape(M2, M1)


def fixed_part(setup: Setup, beta, xg):
    """rapid.py:233-249."""
    if beta is None:
        return 0.0
    beta = np.asarray(beta, dtype=float).ravel()
    m1, m2 = setup.grid.interior_dims
    if xg is None:
        if beta.shape[0] != 1:
            raise OracleDomainError("grid covariates required")
        return float(beta[0])
    xg = np.asarray(xg, dtype=float)
    if xg.ndim == 3:
        xg = xg.reshape(-1, xg.shape[2])
    if xg.shape != (m1 * m2, beta.shape[0]):
        raise OracleDomainError("grid covariate shape mismatch")
    return (xg @ beta).reshape(m2, m1)


def predict(setup: Setup, c, beta=None, xg=None):
    """rapid.py:252-261."""
    conv = circ_convolve(setup.spectrum, setup.embed_dims, scatter_cstar(setup, c))
    return setup.grid.interior(conv) + fixed_part(setup, beta, xg)


# --------------------------------------------------------------------------
# exact fit / GLS  (exact.py:25-113)
# --------------------------------------------------------------------------


@dataclass(frozen=True)
class Fit:
    """exact.py:40-56."""
    model: Model
    obs: np.ndarray
    X: np.ndarray
    chol_M: np.ndarray
    beta: np.ndarray
    c: np.ndarray


def cov_dense(model: Model, a, b=None):
    """covariance.py:100-116 (cdist + symmetrise)."""
    from scipy.spatial.distance import cdist
    a = np.atleast_2d(np.asarray(a, dtype=float))
    bb = a if b is None else np.atleast_2d(np.asarray(b, dtype=float))
    k = model.cov(cdist(a, bb))
    return 0.5 * (k + k.T) if b is None else k


def gls(chol, X, z):
    """exact.py:59-68."""
    a = scipy.linalg.solve_triangular(chol, z, lower=True)
    b = scipy.linalg.solve_triangular(chol, X, lower=True)
    beta = np.linalg.solve(b.T @ b, b.T @ a)
    half = scipy.linalg.solve_triangular(chol, z - X @ beta, lower=True)
    return beta, scipy.linalg.solve_triangular(chol.T, half, lower=False)


def exact_fit(model: Model, obs, z, X=None) -> Fit:
    """exact.py:71-105 (ridge retry exact.py:25-37)."""
    obs = np.asarray(obs, dtype=float).reshape(-1, 2)
    z = np.asarray(z, dtype=float).ravel()
    n = obs.shape[0]
    X = np.ones((n, 1)) if X is None else np.asarray(X, dtype=float)
    if X.ndim == 1:
        X = X[:, None]
    m = cov_dense(model, obs)
    m[np.diag_indices_from(m)] += model.tau2
    try:
        chol = scipy.linalg.cholesky(m, lower=True)
    except scipy.linalg.LinAlgError:
        ridge = 1.0e-10 * np.trace(m) / n
        chol = scipy.linalg.cholesky(m + ridge * np.eye(n), lower=True)
    beta, c = gls(chol, X, z)
    return Fit(model, obs, X, chol, beta, c)


def refit(fit: Fit, z):
    """exact.py:108-113."""
    z = np.asarray(z, dtype=float).ravel()
    if z.shape[0] != fit.obs.shape[0]:
        raise OracleDomainError("z length mismatch")
    return gls(fit.chol_M, fit.X, z)


def target_covariates(fit: Fit, targets, xt):
    """exact.py:116-129."""
    if xt is None:
        if not (fit.X.shape[1] == 1 and np.all(fit.X == fit.X[0, 0])):
            raise OracleDomainError("fit uses nontrivial covariates")
        return np.full((targets.shape[0], 1), fit.X[0, 0])
    xt = np.asarray(xt, dtype=float)
    return xt[:, None] if xt.ndim == 1 else xt


def predict_exact(fit: Fit, targets, xt=None):
    """exact.py:132-147: X_t beta + k_t c (one block; the reference chunks only for memory)."""
    targets = np.asarray(targets, dtype=float).reshape(-1, 2)
    xt = target_covariates(fit, targets, xt)
    return cov_dense(fit.model, targets, fit.obs) @ fit.c + xt @ fit.beta


def kriging_se_exact(fit: Fit, targets, xt=None):
    """exact.py:150-175: sqrt(sigma2 - k'M^-1 k + h'(B'B)^-1 h), h = x_t - u'B, u = L^-1 k."""
    targets = np.asarray(targets, dtype=float).reshape(-1, 2)
    xt = target_covariates(fit, targets, xt)
    b = scipy.linalg.solve_triangular(fit.chol_M, fit.X, lower=True)
    g = scipy.linalg.cho_factor(b.T @ b, lower=True)
    u = scipy.linalg.solve_triangular(fit.chol_M, cov_dense(fit.model, targets, fit.obs).T, lower=True)
    var = fit.model.sigma2 - np.einsum("ij,ij->j", u, u)
    h = xt - u.T @ b
    var += np.einsum("ij,ji->i", h, scipy.linalg.cho_solve(g, h.T))
    if np.any(var < -1.0e-10):
        raise OracleNumericError(f"negative prediction variance {var.min():.3e}")
    return np.sqrt(np.clip(var, 0.0, None))


# --------------------------------------------------------------------------
# randomness  (simulate.py:52-74)
# --------------------------------------------------------------------------

MASK64 = (1 << 64) - 1
PHILOX_M = (0xD2E7470EE14C6C93, 0xCA5A826395121157)
PHILOX_W = (0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B)


def splitmix64(v: int) -> int:
    """simulate.py:52-57."""
    z = (v + 0x9E3779B97F4A7C15) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def sub_seed(seed: int, j: int) -> int:
    """simulate.py:60-62."""
    return (int(seed) ^ splitmix64(int(j))) & MASK64


def philox4x64_block(counter, key):
    """Philox4x64-10 block function (Salmon, Moraes, Dror, Shaw, SC'11).

    Restated here so the GPU kernel's bit stream can be pinned independently of
    numpy; tests check it against ``numpy.random.Philox.random_raw``."""
    c = [int(v) & MASK64 for v in counter]
    k0, k1 = int(key[0]) & MASK64, int(key[1]) & MASK64
    for rnd in range(10):
        if rnd:
            k0 = (k0 + PHILOX_W[0]) & MASK64
            k1 = (k1 + PHILOX_W[1]) & MASK64
        p0 = PHILOX_M[0] * c[0]
        p1 = PHILOX_M[1] * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k0, p1 & MASK64, (p0 >> 64) ^ c[3] ^ k1, p0 & MASK64]
    return c


def philox_words(seed: int, stream: int, start: int, count: int):
    """Words start..start+count of the stream numpy's Philox(key=seed+(stream<<64))
    emits: word w comes from block counter w//4 + 1 (pre-incremented counter)."""
    out = np.empty(count, dtype=np.uint64)
    for t in range(count):
        w = start + t
        out[t] = philox4x64_block([w // 4 + 1, 0, 0, 0], [seed, stream])[w % 4]
    return out


def rng_for(seed: int, stream: int):
    """simulate.py:65-68 — the reference's numpy generator."""
    return np.random.Generator(np.random.Philox(key=(int(seed) & MASK64) + (int(stream) << 64)))


def words_to_normals(words):
    """simulate.py:71-74 with integers(0, 2^53) == raw >> 11 (Lemire, power-of-two range)."""
    k = (np.asarray(words, dtype=np.uint64) >> np.uint64(11)).astype(float)
    return ndtri((k + 0.5) / float(1 << 53))


def normals(gen, shape):
    """simulate.py:71-74 verbatim semantics on a numpy Generator."""
    u = (gen.integers(0, 1 << 53, size=shape).astype(float) + 0.5) / float(1 << 53)
    return ndtri(u)


# --------------------------------------------------------------------------
# conditional simulation  (simulate.py:77-192)
# --------------------------------------------------------------------------


def embedding_root(model: Model, grid: Grid):
    """simulate.py:77-100 — PSD check, one doubling, sqrt of clipped eigenvalues."""
    M1, M2 = grid.total_dims
    p1, p2 = fft_len(2 * M1 - 1), fft_len(2 * M2 - 1)
    for attempt in range(2):
        lam = np.fft.fft2(model.cov(torus_lags(grid, p1, p2))).real
        if lam.min() >= -1.0e-8 * lam.max():
            return p1, p2, np.sqrt(np.clip(lam, 0.0, None))
        if attempt == 0:
            p1, p2 = fft_len(2 * p1), fft_len(2 * p2)
    raise OracleNumericError(f"circulant embedding not PSD; most negative eigenvalue {lam.min():.6e}")


def uncond_field(model: Model, grid: Grid, seed: int, root=None):
    """simulate.py:103-118."""
    M1, M2 = grid.total_dims
    p1, p2, rt = root if root is not None else embedding_root(model, grid)
    gen = rng_for(seed, 0)
    re = normals(gen, (p2, p1))
    im = normals(gen, (p2, p1))
    f = np.sqrt(p1 * p2) * np.fft.ifft2(rt * (re + 1j * im))
    return f.real[:M2, :M1]


def obs_local(model: Model, setup: Setup, g, seed: int):
    """simulate.py:121-143."""
    if g.shape != setup.grid.total_dims[::-1]:
        raise OracleDomainError("grid field shape mismatch")
    cv = setup.cond_var
    if (cv < -1.0e-10 * setup.model.sigma2).any():
        raise OracleNumericError("negative conditional variance")
    cv = np.clip(cv, 0.0, None)
    mean = np.einsum("ij,ij->i", setup.weights, g.ravel()[setup.indices])
    gen = rng_for(seed, 1)
    n = setup.weights.shape[0]
    gs = mean + np.sqrt(cv) * normals(gen, n)
    return gs + np.sqrt(model.tau2) * normals(gen, n)


def cond_draw(fit: Fit, setup: Setup, seed: int, xg=None, data_pred=None, root=None):
    """simulate.py:146-159."""
    g = uncond_field(fit.model, setup.grid, sub_seed(seed, 101), root)
    zs = obs_local(fit.model, setup, g, sub_seed(seed, 202))
    bs, cs = refit(fit, zs)
    if data_pred is None:
        data_pred = predict(setup, fit.c, fit.beta, xg)
    return data_pred + (setup.grid.interior(g) - predict(setup, cs, bs, xg))


def ensemble(fit: Fit, setup: Setup, n_draws: int, seed: int, xg=None, keep_draws=True):
    """simulate.py:174-192 — returns (draws, mean, se[ddof=1])."""
    if n_draws < 2:
        raise OracleDomainError("need at least 2 draws")
    dp = predict(setup, fit.c, fit.beta, xg)
    root = embedding_root(fit.model, setup.grid)
    draws = np.stack([cond_draw(fit, setup, sub_seed(seed, j), xg, dp, root)
                      for j in range(n_draws)])
    return draws, draws.mean(axis=0), draws.std(axis=0, ddof=1)
