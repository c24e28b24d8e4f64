// Device Matern correlation phi(x) = x^nu K_nu(x) / (2^(nu-1) Gamma(nu)), phi(0) = 1.
//
// Follows /root/reference/pkg/src/rapidkrig/bessel.py:
//   matern_correlation 258-278   (x <= 1e-12 -> 1, clip to [0, 1])
//   _matern_half_integer 224-234 (nu = n + 1/2, n <= 12: exp(-x) * Horner poly in 2x)
//   matern_correlation_bessel 237-255 (rescaled recurrence R_{m+1} = (x/2)^2 R_{m-1} + m R_m)
//   _kv_pair_series 50-101 (Temme, x <= 2) and _kv_pair_cf2 104-171 (Steed CF2, x > 2),
//   each element iterating to its own convergence (|term| < 1e-15 |sum|).
// The model-dependent constants (Horner coefficients, Temme gammas, Gamma(nu))
// are computed on the host exactly as the reference computes them (Python int
// true division / math.gamma) and passed in rk_model.
#pragma once

#include "rk_common.cuh"

namespace rk {

// reciprocals of the Temme series' per-term divisors, tabulated on the host: the series
// loop multiplies instead of dividing (a double division is a ~10-instruction dependent chain)
constexpr int kTemmeTab = 24;

struct MaternDev {
  double sigma2, alpha;
  int half_n;             // >= 0: closed form
  int ncoef;
  double coef[13];
  double pref;
  int nl;
  double mu, gampl, gammi, gam1, gam2, fact, gamma_nu;
  double rq[kTemmeTab];   // 1 / (i^2 - mu^2), i = 1 .. kTemmeTab
  double ri[kTemmeTab];   // 1 / i
  double rm[kTemmeTab];   // 1 / (i - mu)
  double rp[kTemmeTab];   // 1 / (i + mu)
};

inline MaternDev make_matern_dev(const rk_model& m) {
  MaternDev d{};
  d.sigma2 = m.sigma2;
  d.alpha = m.alpha;
  d.half_n = m.half_n;
  d.ncoef = m.half_n >= 0 ? m.half_n + 1 : 0;
  for (int i = 0; i < 13; ++i) d.coef[i] = m.half_coef[i];
  d.pref = m.half_pref;
  d.nl = m.nl;
  d.mu = m.mu;
  d.gampl = m.temme_gampl;
  d.gammi = m.temme_gammi;
  d.gam1 = m.temme_gam1;
  d.gam2 = m.temme_gam2;
  d.fact = m.temme_fact;
  d.gamma_nu = m.gamma_nu;  // divisor in 2 r0 / Gamma(nu) (bessel.py:255)
  const double mu2 = d.mu * d.mu;
  for (int i = 1; i <= kTemmeTab; ++i) {
    const double di = (double)i;
    d.rq[i - 1] = 1.0 / (di * di - mu2);
    d.ri[i - 1] = 1.0 / di;
    d.rm[i - 1] = 1.0 / (di - d.mu);
    d.rp[i - 1] = 1.0 / (di + d.mu);
  }
  return d;
}

// (K_mu(x), K_mu+1(x)) for 0 < x <= 2 (bessel.py:50-101); returns false if no convergence
__device__ inline bool kv_pair_series(const MaternDev& P, double x, double& k0, double& k1) {
  const double mu = P.mu;
  const double half_x = 0.5 * x;
  const double l2x = -log(half_x);
  const double sg = mu * l2x;
  const double shr = fabs(sg) < 1.0e-12 ? 1.0 : sinh(sg) / sg;
  double f = P.fact * (P.gam1 * cosh(sg) + P.gam2 * shr * l2x);
  const double e = exp(sg);
  double p = 0.5 * e / P.gampl;
  double q = 0.5 / (e * P.gammi);
  double c = 1.0;
  const double d = half_x * half_x;
  double s0 = f, s1 = p;
  const double mu2 = mu * mu;
  for (int i = 1; i <= 500; ++i) {
    const double di = (double)i;
    if (i <= kTemmeTab) {
      f = (di * f + p + q) * P.rq[i - 1];
      c *= d * P.ri[i - 1];
      p *= P.rm[i - 1];
      q *= P.rp[i - 1];
    } else {
      f = (di * f + p + q) / (di * di - mu2);
      c *= d / di;
      p /= di - mu;
      q /= di + mu;
    }
    const double del = c * f;
    s0 += del;
    s1 += c * (p - di * f);
    if (fabs(del) < fabs(s0) * 1.0e-15) {
      k0 = s0;
      k1 = s1 * (2.0 / x);
      return true;
    }
  }
  return false;
}

// (K_mu(x), K_mu+1(x)) for x > 2 by Steed's CF2 (bessel.py:104-171)
__device__ inline bool kv_pair_cf2(const MaternDev& P, double x, double& k0, double& k1) {
  const double mu = P.mu;
  const double a1 = 0.25 - mu * mu;
  double b = 2.0 * (1.0 + x);
  double d = 1.0 / b;
  double h = d, delh = d;
  double q1 = 0.0, q2 = 1.0;
  double q = a1, c = a1, a = -a1;
  double s = 1.0 + q * delh;
  for (int i = 2; i <= 20000; ++i) {
    a -= 2 * (i - 1);
    c = -a * c / i;
    const double qn = (q1 - b * q2) / a;
    q1 = q2;
    q2 = qn;
    q += c * q2;
    b += 2.0;
    d = 1.0 / (d * a + b);
    delh = (b * d - 1.0) * delh;
    h += delh;
    const double ds = q * delh;
    s += ds;
    if (fabs(ds) < fabs(s) * 1.0e-15) {
      const double hh = a1 * h;
      k0 = sqrt(3.14159265358979311600 / (2.0 * x)) * exp(-x) / s;
      k1 = k0 * (mu + x + 0.5 - hh) / x;
      return true;
    }
  }
  return false;
}

// phi(x) for x = alpha * distance (already scaled); *bad set on non-convergence
__device__ inline double matern_phi(const MaternDev& P, double x, int* bad) {
  if (!(x > 1.0e-12)) return 1.0;
  double phi;
  if (P.half_n >= 0) {
    double acc = 0.0;
    const double tx = 2.0 * x;
    for (int i = 0; i < P.ncoef; ++i) acc = acc * tx + P.coef[i];
    phi = P.pref * exp(-x) * acc;
  } else {
    double k0, k1;
    const bool ok = x <= 2.0 ? kv_pair_series(P, x, k0, k1) : kv_pair_cf2(P, x, k0, k1);
    if (!ok) {
      if (bad) *bad = 1;
      return nan("");
    }
    const double half = 0.5 * x;
    const double sc = pow(half, P.mu);
    double r0 = k0 * sc;
    double r1 = k1 * sc * half;
    const double h2 = half * half;
    for (int j = 0; j < P.nl; ++j) {
      const double r2 = h2 * r0 + (P.mu + j + 1) * r1;
      r0 = r1;
      r1 = r2;
    }
    phi = 2.0 * r0 / P.gamma_nu;
  }
  return fmin(fmax(phi, 0.0), 1.0);
}

// matern_phi for half-integer nu (P.half_n >= 0) only: the closed form alone, bitwise the same
// value (kernels templated on it avoid inlining the Bessel paths' code)
__device__ __forceinline__ double matern_phi_half(const MaternDev& P, double x) {
  if (!(x > 1.0e-12)) return 1.0;
  double acc = 0.0;
  const double tx = 2.0 * x;
  for (int i = 0; i < P.ncoef; ++i) acc = acc * tx + P.coef[i];
  return fmin(fmax(P.pref * exp(-x) * acc, 0.0), 1.0);
}

// sigma2 * phi(alpha * dist)  (covariance.py:83-89)
__device__ __forceinline__ double matern_cov(const MaternDev& P, double dist, int* bad) {
  return P.sigma2 * matern_phi(P, P.alpha * dist, bad);
}

}  // namespace rk
