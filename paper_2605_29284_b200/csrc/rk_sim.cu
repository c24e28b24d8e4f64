// rapidkrig B200: conditional-simulation ensemble (Philox normals, circulant-embedding field,
// local observations, batched draws, per-chunk moments).
//
// Reference mapping (/root/reference/pkg/src/rapidkrig):
//   _splitmix64 / draw_seed   simulate.py:52-62   -> splitmix64(), draw_seed()
//   _rng / _std_normals       simulate.py:65-74   -> philox4x64_10() keyed (seed, stream),
//        pre-incremented counter (block b uses counter b+1), normal = ndtri(((w>>11)+.5)/2^53)
//   _embedding_root           simulate.py:82-100  -> ensure_embedding() (PSD test, one doubling)
//   sim_unconditional_grid    simulate.py:103-118 -> cs_rowgen_kernel (Philox + normals + row IFFT;
//        cs_rng_kernel + cs_rowfft_kernel with RK_CS_FUSED=0) + cs_col_kernel (column pairs)
//   sim_obs_local             simulate.py:121-143 -> obs_local_kernel
//   refit_coefficients/_gls   exact.py:59-68,108-113 -> gls_batch (rk_exact.cu)
//   conditional_draw / generate_ensemble simulate.py:146-192 -> rk_ensemble_accumulate
//   fit / _cholesky_with_ridge exact.py:25-37,71-105 -> rk_fit_create (rk_exact.cu)
#include <cooperative_groups.h>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include <cublas_v2.h>
#include <cusolverDn.h>

#include "rk_internal.cuh"
#include "rk_ndtri.cuh"

namespace cg = cooperative_groups;

namespace rk {

// ------------------------------------------------------------- randomness
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t v) {
  uint64_t z = v + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t draw_seed(uint64_t seed, uint64_t j) {
  return seed ^ splitmix64(j);
}

// Philox4x64-10 (Salmon et al., SC'11) block for counter (ctr0, 0, 0, 0), key (k0, k1)
__device__ __forceinline__ void philox4x64_10(uint64_t ctr0, uint64_t k0, uint64_t k1, uint64_t o[4]) {
  uint64_t c0 = ctr0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t lo0 = 0xD2E7470EE14C6C93ULL * c0, hi0 = __umul64hi(0xD2E7470EE14C6C93ULL, c0);
    const uint64_t lo1 = 0xCA5A826395121157ULL * c2, hi1 = __umul64hi(0xCA5A826395121157ULL, c2);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
  }
  o[0] = c0; o[1] = c1; o[2] = c2; o[3] = c3;
}

// two Philox4x64-10 blocks of the same key in lockstep (counters ca, cb): the key schedule is
// computed once per round for both, and the two blocks' products overlap
__device__ __forceinline__ void philox4x64_10_x2(uint64_t ca, uint64_t cb, uint64_t k0, uint64_t k1, uint64_t oa[4],
                                                 uint64_t ob[4]) {
  uint64_t a0 = ca, a1 = 0, a2 = 0, a3 = 0, b0 = cb, b1 = 0, b2 = 0, b3 = 0;
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r) {
      k0 += 0x9E3779B97F4A7C15ULL;
      k1 += 0xBB67AE8584CAA73BULL;
    }
    const uint64_t la0 = 0xD2E7470EE14C6C93ULL * a0, ha0 = __umul64hi(0xD2E7470EE14C6C93ULL, a0);
    const uint64_t la1 = 0xCA5A826395121157ULL * a2, ha1 = __umul64hi(0xCA5A826395121157ULL, a2);
    const uint64_t lb0 = 0xD2E7470EE14C6C93ULL * b0, hb0 = __umul64hi(0xD2E7470EE14C6C93ULL, b0);
    const uint64_t lb1 = 0xCA5A826395121157ULL * b2, hb1 = __umul64hi(0xCA5A826395121157ULL, b2);
    a0 = ha1 ^ a1 ^ k0;
    a1 = la1;
    a2 = ha0 ^ a3 ^ k1;
    a3 = la0;
    b0 = hb1 ^ b1 ^ k0;
    b1 = lb1;
    b2 = hb0 ^ b3 ^ k1;
    b3 = lb0;
  }
  oa[0] = a0; oa[1] = a1; oa[2] = a2; oa[3] = a3;
  ob[0] = b0; ob[1] = b1; ob[2] = b2; ob[3] = b3;
}

__device__ __forceinline__ uint64_t philox_word(uint64_t seed, uint64_t stream, uint64_t w) {
  uint64_t o[4];
  philox4x64_10(w / 4 + 1, seed, stream, o);
  const int q = (int)(w & 3);
  return q == 0 ? o[0] : q == 1 ? o[1] : q == 2 ? o[2] : o[3];
}

// integers(0, 2^53) == w >> 11 (Lemire, power-of-two range); u = (k + 0.5) / 2^53; ndtri(u)
__device__ __forceinline__ double word_uniform(uint64_t w) { return ((double)(w >> 11) + 0.5) * 0x1.0p-53; }
__device__ __forceinline__ double word_normal(uint64_t w) { return ndtri_b200(word_uniform(w)); }

__global__ void philox_kernel(uint64_t seed, uint64_t stream, uint64_t start, int64_t count,
                              double* out_n, uint64_t* out_raw) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < count;
       t += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t w = philox_word(seed, stream, start + (uint64_t)t);
    if (out_raw) out_raw[t] = w;
    if (out_n) out_n[t] = word_normal(w);
  }
}

// ------------------------------------------------------------- CS field
struct CsColArgs {
  FftPlan pl;
  int lpc;
  int ncols;                 // M1
  int keep;                  // M2
  const double2* V;
  int64_t ldV, V_bstride;
  double* g;                 // (batch, M2, M1)
  int64_t g_bstride;
  int tw_off;                // smem offset (double2 units) of the staged twiddle table
  SplitTw sw;                // split-length kernel: w_P^n tables
};

template <bool TWS, int FM>
__global__ void __launch_bounds__(FM == 1 ? kFftWideThreads : FM == 2 ? kFftSplitThreads : 512, 1) cs_col_kernel(const CsColArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  // two columns per line: only Re(IFFT(V)) is kept, which is the IFFT of V's Hermitian part
  // H[k] = (V[k] + conj V[-k]) / 2; the IFFT of H_a + i H_b is Re IFFT V_a + i Re IFFT V_b
  const int ca = 2 * (blockIdx.x * a.lpc + line), cb = ca + 1;
  double2* buf = smem + (size_t)line * n;
  const double2* Va = a.V + (int64_t)b * a.V_bstride + (int64_t)ca * a.ldV;
  const double2* Vb = Va + a.ldV;
  const bool va = ca < a.ncols, vb = cb < a.ncols;
  const FftPlan pls = TWS ? fft_twiddles_to_smem(a.pl, smem + a.tw_off) : a.pl;
  pdl_wait();   // V is the predecessor's output
  for (int y = tl; y < n; y += nthr) {
    const int m = y ? n - y : 0;
    const double2 A = va ? Va[y] : make_double2(0.0, 0.0), Am = va ? Va[m] : make_double2(0.0, 0.0);
    const double2 B = vb ? Vb[y] : make_double2(0.0, 0.0), Bm = vb ? Vb[m] : make_double2(0.0, 0.0);
    buf[y] = make_double2(0.5 * ((A.x + Am.x) - (B.y - Bm.y)), 0.5 * ((A.y - Am.y) + (B.x + Bm.x)));
  }
  __syncthreads();
  fft_line<true, TWS, FM>(buf, pls, tl, a.lpc > 1 ? 1 + line : 0);
  if (a.lpc > 1) __syncthreads();   // the stores below read every line
  double* g = a.g + (int64_t)b * a.g_bstride;
  for (int idx = threadIdx.x; idx < a.lpc * a.keep; idx += blockDim.x) {
    const int l = idx % a.lpc, y = idx / a.lpc;
    const int c0 = 2 * (blockIdx.x * a.lpc + l);
    const double2 v = smem[(size_t)l * n + y];
    if (c0 < a.ncols) g[(int64_t)y * a.ncols + c0] = v.x;
    if (c0 + 1 < a.ncols) g[(int64_t)y * a.ncols + c0 + 1] = v.y;
  }
}

struct ObsArgs {
  const int32_t* base;
  const double* weights;
  const double* cond_var;
  int64_t n;
  int M, bs, M1;
  const double* g;
  int64_t g_bstride;
  double sqrt_tau2;
  uint64_t seed;
  int64_t j0;
  int direct;
  double* z;                 // (batch, n)
};

__global__ void obs_local_kernel(const ObsArgs a) {
  const int b = blockIdx.y;
  const uint64_t os = a.direct ? a.seed : draw_seed(draw_seed(a.seed, (uint64_t)(a.j0 + b)), 202);
  const double* g = a.g + (int64_t)b * a.g_bstride;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t base = a.base[i];
    const double* w = a.weights + i * a.M;
    double mean = 0.0;
    for (int m = 0; m < a.M; ++m) mean = fma(w[m], g[base + (int64_t)(m / a.bs) * a.M1 + (m % a.bs)], mean);
    const double eta = word_normal(philox_word(os, 1, (uint64_t)i));
    const double eps = word_normal(philox_word(os, 1, (uint64_t)(a.n + i)));
    const double cv = fmax(a.cond_var[i], 0.0);
    const double gs = mean + sqrt(cv) * eta;
    a.z[(int64_t)b * a.n + i] = gs + a.sqrt_tau2 * eps;
  }
}

// ----------------------------------------------------- exact (order-free) ensemble moments
// Per pixel, the moments s1 = sum e_j and s2 = sum e_j^2 of e_j = draw_j - data_pred are kept
// as fixed-point INTEGERS: each term v (scaled by the power of two 2^-k nearest sigma, exact) is
// converted to trunc(v 2^64) and added as three signed 42-bit digits into three int64 limbs.
// Integer addition is associative, so the moments -- and mean / SE -- are bitwise the same
// whatever the order, batching, chunking or GPU count (one all-reduce of int64 limbs combines
// ranks), and they are the exactly rounded sums of the terms (the reference's two-pass
// std(ddof=1), simulate.py:191-192, is matched to ~1e-16 instead of one-pass roundoff).
// Range: |v| < 2^20 sigma per term and < 2^21 terms per limb (checked; RK_NUMERIC beyond).
constexpr int kFxFrac = 64;
constexpr double kFxMaxTerm = 1048576.0;   // 2^20

__device__ __forceinline__ void fx_digits(double v, long long d[3]) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
  const int ex = (int)((bits >> 52) & 0x7ff);
  unsigned long long m = bits & ((1ULL << 52) - 1);
  if (ex) m |= 1ULL << 52;
  const int sh = (ex ? ex : 1) - 1075 + kFxFrac;   // |v| 2^64 = m 2^sh
  unsigned __int128 M = 0;
  if (sh >= 0) M = (unsigned __int128)m << sh;       // sh <= 72 under the range check
  else if (sh > -64) M = m >> (-sh);                  // truncation toward zero
  const unsigned long long mask = (1ULL << 42) - 1;
  long long d0 = (long long)((unsigned long long)M & mask);
  long long d1 = (long long)((unsigned long long)(M >> 42) & mask);
  long long d2 = (long long)(unsigned long long)(M >> 84);
  if (bits >> 63) { d0 = -d0; d1 = -d1; d2 = -d2; }
  d[0] = d0; d[1] = d1; d[2] = d2;
}

__global__ void accumulate_fx_kernel(const double* __restrict__ E, int batch, int64_t npix,
                                     const double* __restrict__ dp, double inv_scale,
                                     long long* __restrict__ acc, double* __restrict__ draws,
                                     int* __restrict__ bad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
       p += (int64_t)gridDim.x * blockDim.x) {
    long long a[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) a[q] = acc[q * npix + p];
    const double d = dp[p];
    bool oob = false;
    for (int b = 0; b < batch; ++b) {
      const double e = E[(int64_t)b * npix + p];
      const double v = e * inv_scale;   // exact: a power of two
      if (!(fabs(v) < kFxMaxTerm)) oob = true;   // also NaN / inf
      long long t[3];
      fx_digits(oob ? 0.0 : v, t);
      a[0] += t[0]; a[1] += t[1]; a[2] += t[2];
      fx_digits(oob ? 0.0 : v * v, t);
      a[3] += t[0]; a[4] += t[1]; a[5] += t[2];
      if (draws) draws[(int64_t)b * npix + p] = d + e;
    }
#pragma unroll
    for (int q = 0; q < 6; ++q) acc[q * npix + p] = a[q];
    if (oob) atomicOr(bad, 1);
  }
}

__global__ void acc_add_kernel(long long* __restrict__ dst, const long long* __restrict__ src, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] += src[i];
}

__device__ __forceinline__ double fx_value(long long d0, long long d1, long long d2) {
  const __int128 S = ((__int128)d2 << 84) + ((__int128)d1 << 42) + (__int128)d0;
  const long long hi = (long long)(S >> 64);
  const unsigned long long lo = (unsigned long long)S;
  return fma((double)hi, 18446744073709551616.0, (double)lo) * 0x1.0p-64;
}

__global__ void finalize_fx_kernel(int64_t npix, double R, double scale, const double* dp,
                                   const long long* __restrict__ acc, double* mean, double* se) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npix;
       p += (int64_t)gridDim.x * blockDim.x) {
    const double s1 = fx_value(acc[p], acc[npix + p], acc[2 * npix + p]) * scale;
    const double s2 = fx_value(acc[3 * npix + p], acc[4 * npix + p], acc[5 * npix + p]) * (scale * scale);
    const double m = s1 / R;
    if (mean) mean[p] = dp[p] + m;
    if (se) se[p] = sqrt(fmax((s2 - s1 * m) / (R - 1.0), 0.0));
  }
}

// the power of two nearest sigma (exact rescaling of the moments)
static double fx_scale(double sigma2) {
  if (!(sigma2 > 0.0) || !std::isfinite(sigma2)) return 1.0;
  return std::ldexp(1.0, (int)std::floor(0.5 * std::log2(sigma2)));
}

__global__ void root_q_kernel(const double* __restrict__ lam_q, int hs1, int qs2, double scale,
                              double* __restrict__ root_q) {
  const int64_t tot = (int64_t)hs1 * qs2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / hs1), bc = (int)(e % hs1);   // root_q[a][b] <- lam_q[b][a]
    root_q[e] = sqrt(fmax(lam_q[(int64_t)bc * qs2 + a], 0.0)) * scale;
  }
}

Status spectrum_quarter(const MaternDev& P, double hx, double hy, int p1, int p2, double scale,
                        double* out_q, int ldq, cudaStream_t st);

static int64_t next_fft_len(int64_t m) {
  if (m <= 1) return 1;
  int64_t best = -1;
  for (int64_t two = 1; two < 4 * m; two *= 2) {
    int64_t v = two;
    while (v < m) v *= 3;
    if (best < 0 || v < best) best = v;
  }
  return best;
}

Status ensure_embedding(rk_setup* s, cudaStream_t st) {
  if (s->emb.ready) return Status::ok();
  int64_t p1 = next_fft_len(2 * (int64_t)s->M1 - 1), p2 = next_fft_len(2 * (int64_t)s->M2 - 1);
  double lmin = 0, lmax = 0;
  for (int attempt = 0; attempt < 2; ++attempt) {
    const int hs1 = (int)(p1 / 2 + 1), qs2 = (int)(p2 / 2 + 1);
    double* lam = nullptr;
    RK_CUDA_TRY(cudaMalloc(&lam, sizeof(double) * (size_t)hs1 * qs2));
    Status sp = spectrum_quarter(s->mat, s->grid.hx, s->grid.hy, (int)p1, (int)p2, 1.0, lam, qs2, st);
    if (!sp.good()) { cudaFree(lam); return sp; }
    std::vector<double> h((size_t)hs1 * qs2);
    RK_CUDA_TRY(cudaMemcpy(h.data(), lam, sizeof(double) * h.size(), cudaMemcpyDeviceToHost));
    lmin = *std::min_element(h.begin(), h.end());
    lmax = *std::max_element(h.begin(), h.end());
    if (!(lmin < -1.0e-8 * lmax)) {
      Embedding& e = s->emb;
      e.ps1 = (int)p1;
      e.ps2 = (int)p2;
      e.doubled = attempt;
      e.hs1 = hs1;
      e.qs2 = qs2;
      RK_TRY(embedding_plans(s));
      RK_CUDA_TRY(cudaMalloc(&e.root_q, sizeof(double) * (size_t)hs1 * qs2));
      const double P = (double)p1 * (double)p2;
      root_q_kernel<<<(int)std::min<int64_t>(ceil_div((int64_t)hs1 * qs2, 256), 148 * 32), 256, 0, st>>>(
          lam, hs1, qs2, std::sqrt(P) / P, e.root_q);
      count_launch();
      RK_LAUNCH_CHECK();
      RK_CUDA_TRY(cudaStreamSynchronize(st));
      cudaFree(lam);
      e.ready = true;
      return Status::ok();
    }
    cudaFree(lam);
    p1 = next_fft_len(2 * p1);
    p2 = next_fft_len(2 * p2);
  }
  char b[256];
  snprintf(b, sizeof b,
           "circulant embedding is not positive semidefinite even after doubling; most negative "
           "eigenvalue %.6e",
           lmin);
  return Status::err(RK_NUMERIC, b);
}

// CS pass A, part 1 (high occupancy): the 2 Ps normals of each realization (Philox words
// [0, Ps) real, [Ps, 2 Ps) imaginary, row-major over (ps2, ps1); simulate.py:113-116) scaled by
// sqrt(lambda) sqrt(P)/P, written as complex Z[p] (64-byte coalesced stores per thread).
struct CsRngArgs {
  uint64_t seed;
  int64_t j0;
  int direct;
  int ps1, ps2;
  const double* root_q;
  int rq_ld;
  double2* Z;                // (batch, ps2, ps1)
  int64_t Z_bstride;
};

// Inverse normal with warp-level tail compaction: every lane evaluates the central rational
// for its 8 normals; the ~8% tail values (log + sqrt + a second rational) are queued per warp
// in shared memory and evaluated by all lanes together, so a warp pays one tail round per
// iteration instead of running both branches for every lane.
constexpr int kRngThreads = 256;
#ifndef RK_RNG_MINB
#define RK_RNG_MINB 4
#endif

__global__ void __launch_bounds__(kRngThreads, RK_RNG_MINB) cs_rng_kernel(const CsRngArgs a) {
  __shared__ double tq[kRngThreads / 32][8 * 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double* wq = tq[wid];
  const int b = blockIdx.y;
  const uint64_t fs = a.direct ? a.seed : draw_seed(draw_seed(a.seed, (uint64_t)(a.j0 + b)), 101);
  // 32-bit indexing (the host checks Ps < 2^31); (iy, ix) of word 4t advance incrementally
  const uint32_t Ps = (uint32_t)a.ps1 * (uint32_t)a.ps2;
  const uint32_t nblk = (Ps + 3) / 4, ps4 = Ps / 4;
  const int imoff = (int)(Ps & 3);
  double2* Z = a.Z + (int64_t)b * a.Z_bstride;
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t dstep = 4 * stride;
  const int dy = (int)(dstep / (uint32_t)a.ps1), dx = (int)(dstep % (uint32_t)a.ps1);
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  int iy = (int)(4 * t / (uint32_t)a.ps1), ix = (int)(4 * t - (uint32_t)iy * a.ps1);
  const bool quad_rows = (a.ps1 & 3) == 0;
  // warp-uniform grid-stride loop (the compaction uses full-warp shuffles)
  for (uint32_t t0 = t - lane; t0 < nblk; t0 += stride, t += stride) {
    const bool valid = t < nblk;
    uint64_t re[4], im[8];
    philox4x64_10((uint64_t)t + 1, fs, 0, re);
    const uint64_t ib = (uint64_t)ps4 + t;          // first block holding imaginary words
    philox4x64_10(ib + 1, fs, 0, im);
    if (imoff) philox4x64_10(ib + 2, fs, 0, im + 4);
    double uu[8], z[8];
    unsigned tmask = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      // im[imoff + q - 4] with compile-time indices only (a runtime index would put im in
      // local memory)
      const int k = q - 4;
      const uint64_t w = q < 4 ? re[q]
                       : imoff == 0 ? im[k] : imoff == 1 ? im[k + 1] : imoff == 2 ? im[k + 2] : im[k + 3];
      uu[q] = word_uniform(w);
      if (valid && ndtri_is_tail(uu[q])) tmask |= 1u << q;
    }
    ndtri_central_n<8>(uu, z);   // tails are replaced below
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (tmask >> q & 1) z[q] = uu[q];
    // exclusive prefix of the tail counts across the warp
    const int cnt = __popc(tmask);
    int off = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += v;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= cnt;
    if (total) {
      int o = off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) wq[o++] = z[q];
      __syncwarp();
      for (int k = lane; k < total; k += 32) wq[k] = ndtri_tail(wq[k]);
      __syncwarp();
      o = off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) z[q] = wq[o++];
      __syncwarp();
    }
    if (valid && quad_rows) {   // the 4 words lie in one row, all in range (ps1 % 4 == 0)
      const double* rq = a.root_q + min(iy, a.ps2 - iy) * a.rq_ld;
      double2* zp = Z + 4 * t;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double r = __ldg(&rq[min(ix + q, a.ps1 - ix - q)]);
        zp[q] = make_double2(r * z[q], r * z[4 + q]);
      }
    } else if (valid) {
      uint32_t p = 4 * t;
      int jy = iy, jx = ix;
#pragma unroll
      for (int q = 0; q < 4; ++q, ++p) {
        if (p < Ps) {
          const double r = __ldg(&a.root_q[min(jy, a.ps2 - jy) * a.rq_ld + min(jx, a.ps1 - jx)]);
          Z[p] = make_double2(r * z[q], r * z[4 + q]);
        }
        if (++jx == a.ps1) {
          jx = 0;
          ++jy;
        }
      }
    }
    ix += dx;
    iy += dy;
    if (ix >= a.ps1) {
      ix -= a.ps1;
      ++iy;
    }
  }
}

// CS pass A, part 2: TMA bulk load of each row of Z, inverse FFT along x, keep the M1
// columns, write V[ix][iy] (transposed for the column pass).
struct CsFftArgs {
  FftPlan pl;
  int lpc;
  int ps2;
  int keep;                  // M1
  const double2* Z;
  int64_t Z_bstride;
  double2* V;
  int64_t ldV, V_bstride;
  int tw_off;
};

template <bool TWS, int FM>
__global__ void __launch_bounds__(FM == 1 ? kFftWideThreads : FM == 2 ? kFftSplitThreads : 512, 1) cs_rowfft_kernel(const CsFftArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  double2* buf = smem + (size_t)line * n;
  uint64_t* bar = (uint64_t*)(smem + (size_t)a.lpc * n);
  const FftPlan pls = TWS ? fft_twiddles_to_smem(a.pl, smem + a.tw_off) : a.pl;
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  pdl_wait();   // Z is the predecessor's output
  if (threadIdx.x == 0) {
    int nv = 0;
    for (int l = 0; l < a.lpc; ++l) nv += (blockIdx.x * a.lpc + l) < a.ps2;
    mbar_expect_tx(bar, (uint32_t)nv * (uint32_t)n * 16u);
    const double2* Zb = a.Z + (int64_t)b * a.Z_bstride;
    for (int l = 0; l < a.lpc; ++l) {
      const int iy = blockIdx.x * a.lpc + l;
      if (iy < a.ps2) bulk_g2s(smem + (size_t)l * n, Zb + (int64_t)iy * n, (uint32_t)n * 16u, bar);
    }
  }
  if (blockIdx.x * a.lpc + line >= a.ps2)
    for (int x = tl; x < n; x += nthr) buf[x] = make_double2(0.0, 0.0);
  mbar_wait(bar, 0);
  __syncthreads();
  fft_line<true, TWS, FM>(buf, pls, tl, a.lpc > 1 ? 1 + line : 0);
  if (a.lpc > 1) __syncthreads();   // the stores below read every line
  double2* V = a.V + (int64_t)b * a.V_bstride;
  for (int idx = threadIdx.x; idx < a.lpc * a.keep; idx += blockDim.x) {
    const int l = idx % a.lpc, ix = idx / a.lpc;
    const int row = blockIdx.x * a.lpc + l;
    if (row < a.ps2) V[(int64_t)ix * a.ldV + row] = smem[(size_t)l * n + ix];
  }
}

// Fused CS pass A: each line's threads generate its row of Z = sqrt(lambda) (re + i im) straight
// into shared memory (Philox words, inverse normals with warp-level tail compaction), then run
// the inverse row FFT and store the kept columns transposed.  No Z round trip through HBM, and
// CTAs of one SM in different phases overlap integer (Philox) and FP64 / smem (FFT) work.
struct CsGenArgs {
  FftPlan pl;
  int lpc;
  uint64_t seed;
  int64_t j0;
  int direct;
  int ps1, ps2;
  const double* root_q;
  int rq_ld;
  int keep;                  // M1
  double2* V;
  int64_t ldV, V_bstride;
  int tw_off, q_off;         // smem offsets (double2 units): twiddles, tail queues
  int qcap;                  // tail-queue entries per warp actually used (<= the kernel's QCAP;
                             // smaller only to exercise the overflow path: RK_CS_QCAP)
  SplitTw sw;                // split-length kernel: w_P^n tables
};

// words w .. w+3 of the (fs, 0) Philox stream; two blocks when w is not block aligned
__device__ __forceinline__ void philox_words4(uint64_t w, uint64_t fs, uint64_t o[4]) {
  uint64_t a[4], c[4];
  const uint64_t blk = w >> 2;
  const int off = (int)(w & 3);
  philox4x64_10(blk + 1, fs, 0, a);
  if (off == 0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = a[q];
    return;
  }
  philox4x64_10(blk + 2, fs, 0, c);
#pragma unroll
  for (int q = 0; q < 4; ++q) {   // compile-time indices only
    const uint64_t x1 = q + 1 < 4 ? a[q + 1] : c[q - 3];
    const uint64_t x2 = q + 2 < 4 ? a[q + 2] : c[q - 2];
    const uint64_t x3 = q + 3 < 4 ? a[q + 3] : c[q - 1];
    o[q] = off == 1 ? x1 : off == 2 ? x2 : x3;
  }
}

// MAXT / MINB: the occupancy variant used for WIDE plans of one line of <= 288 threads per CTA
// (e.g. cfg4's 2304-point rows): twiddles from L1 instead of smem and 128-entry tail queues, so
// four CTAs fit an SM (56 registers) instead of three; CS 138.7 -> 135.4 us per realization.
// RK_CS_GEN4=0 keeps the 3-per-SM kernel.
// AL (aligned): ps1 % 4 == 0, so every row starts on a Philox block for both the real and the
// imaginary words (Ps = ps1 ps2 is then a multiple of 4 too) and every 4-point group lies inside
// the row: one block per 4 words and no range checks (the doubled tori, e.g. cfg4's 2304).
template <bool TWS, int FM, int MAXT = (FM == 1 ? kFftWideThreads : FM == 2 ? kFftSplitThreads : 512), int MINB = 1,
          bool AL = false>
__global__ void __launch_bounds__(MAXT, MINB) cs_rowgen_kernel(const CsGenArgs a) {
  constexpr int QCAP = MINB > 1 ? 128 : 256;   // tail-queue entries per warp
  extern __shared__ __align__(16) double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int iy = blockIdx.x * a.lpc + line;
  double2* buf = smem + (size_t)line * n;
  double* wq = (double*)(smem + a.q_off) + (size_t)(threadIdx.x >> 5) * QCAP;
  const FftPlan pls = TWS ? fft_twiddles_to_smem(a.pl, smem + a.tw_off) : a.pl;
  const uint64_t fs = a.direct ? a.seed : draw_seed(draw_seed(a.seed, (uint64_t)(a.j0 + b)), 101);
  if (iy < a.ps2) {
    const uint64_t Ps = (uint64_t)a.ps1 * (uint64_t)a.ps2;
    const uint64_t wre = (uint64_t)iy * a.ps1, wim = Ps + wre;   // simulate.py:114-115
    const double* rq = a.root_q + (int64_t)min(iy, a.ps2 - iy) * a.rq_ld;
    const int ng = (a.ps1 + 3) / 4;
    for (int g0 = tl - lane; g0 < ng; g0 += nthr) {   // warp-uniform (nthr % 32 == 0)
      const int g = g0 + lane;
      const int x0 = 4 * g;
      uint64_t re[4], im[4];
      if (AL) {
        // the key is re-read per group (an opaque copy): hoisted out of the loop, its 10-round
        // schedule stays live across the transform and spills at this kernel's 56 registers
        uint64_t fk;
        asm volatile("mov.b64 %0, %1;" : "=l"(fk) : "l"(fs));
        philox4x64_10_x2(((wre + x0) >> 2) + 1, ((wim + x0) >> 2) + 1, fk, 0, re, im);
      } else {
        philox_words4(wre + x0, fs, re);
        philox_words4(wim + x0, fs, im);
      }
      double uu[8], z[8];
      unsigned tmask = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        uu[q] = word_uniform(q < 4 ? re[q] : im[q - 4]);
        if (g < ng && (AL || x0 + (q & 3) < a.ps1) && ndtri_is_tail(uu[q])) tmask |= 1u << q;
      }
      ndtri_central_n<8>(uu, z);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) z[q] = uu[q];
      const int cnt = __popc(tmask);
      int off = cnt;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, off, d);
        if (lane >= d) off += v;
      }
      const int total = __shfl_sync(0xffffffffu, off, 31);
      off -= cnt;
      if (total > min(QCAP, a.qcap)) {   // queue overflow (rare): each lane evaluates its own
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (tmask >> q & 1) z[q] = ndtri_tail(uu[q]);
      } else if (total) {
        int o = off;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (tmask >> q & 1) wq[o++] = z[q];
        __syncwarp();
        for (int k = lane; k < total; k += 32) wq[k] = ndtri_tail(wq[k]);
        __syncwarp();
        o = off;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (tmask >> q & 1) z[q] = wq[o++];
        __syncwarp();
      }
      if (g < ng) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int x = x0 + q;
          if (AL || x < a.ps1) {
            const double r = __ldg(&rq[min(x, a.ps1 - x)]);
            buf[x] = make_double2(r * z[q], r * z[4 + q]);
          }
        }
      }
    }
  } else {
    for (int x = tl; x < n; x += nthr) buf[x] = make_double2(0.0, 0.0);
  }
  __syncthreads();
  fft_line<true, TWS, FM, false>(buf, pls, tl, a.lpc > 1 ? 1 + line : 0);
  if (a.lpc > 1) __syncthreads();   // the stores below read every line
  double2* V = a.V + (int64_t)b * a.V_bstride;
  for (int idx = threadIdx.x; idx < a.lpc * a.keep; idx += blockDim.x) {
    const int l = idx % a.lpc, ix = idx / a.lpc;
    const int row = blockIdx.x * a.lpc + l;
    if (row < a.ps2) V[(int64_t)ix * a.ldV + row] = smem[(size_t)l * n + ix];
  }
}

// Split-length versions of the two field passes for the large tori (ps = 2 H above the
// WIDE-plan lengths; rk_predict.cu explains the identity).  Only the OUTPUT is pruned here (kept
// columns / rows < H; the random input fills the whole torus), so each length-ps inverse
// transform is the two length-H inverse transforms of its even- and odd-indexed inputs,
// combined as y[n] = e[n] + w^-n o[n] for the kept n.
constexpr int kSplitQcap = 128;   // tail-queue entries per warp

template <bool AL = false>   // AL: ps1 % 4 == 0, as cs_rowgen_kernel
__global__ void __launch_bounds__(kFftWideThreads, 1) cs_rowgen_split_kernel(const CsGenArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int H = a.pl.n;
  const int nthr = a.pl.nthr;
  const int half = threadIdx.x / nthr;
  const int tl = threadIdx.x - half * nthr;
  const int t2 = threadIdx.x, n2 = 2 * nthr;
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.y;
  const int iy = blockIdx.x;
  double2* be = smem;
  double2* bo = smem + H;
  double* wq = (double*)(smem + a.q_off) + (size_t)(threadIdx.x >> 5) * kSplitQcap;
  const FftPlan pls = fft_twiddles_to_smem(a.pl, smem + a.tw_off);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  const uint64_t fs = a.direct ? a.seed : draw_seed(draw_seed(a.seed, (uint64_t)(a.j0 + b)), 101);
  const uint64_t Ps = (uint64_t)a.ps1 * (uint64_t)a.ps2;
  const uint64_t wre = (uint64_t)iy * a.ps1, wim = Ps + wre;   // simulate.py:114-115
  const double* rq = a.root_q + (int64_t)min(iy, a.ps2 - iy) * a.rq_ld;
  const int ng = (a.ps1 + 3) / 4;
  for (int g0 = t2 - lane; g0 < ng; g0 += n2) {   // warp-uniform
    const int g = g0 + lane;
    const int x0 = 4 * g;
    uint64_t re[4], im[4];
    if (AL) {
      uint64_t fk;   // opaque per group (see cs_rowgen_kernel)
      asm volatile("mov.b64 %0, %1;" : "=l"(fk) : "l"(fs));
      philox4x64_10_x2(((wre + x0) >> 2) + 1, ((wim + x0) >> 2) + 1, fk, 0, re, im);
    } else {
      philox_words4(wre + x0, fs, re);
      philox_words4(wim + x0, fs, im);
    }
    double uu[8], z[8];
    unsigned tmask = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uu[q] = word_uniform(q < 4 ? re[q] : im[q - 4]);
      if (g < ng && (AL || x0 + (q & 3) < a.ps1) && ndtri_is_tail(uu[q])) tmask |= 1u << q;
    }
    ndtri_central_n<8>(uu, z);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (tmask >> q & 1) z[q] = uu[q];
    const int cnt = __popc(tmask);
    int off = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += v;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= cnt;
    if (total > min(kSplitQcap, a.qcap)) {   // queue overflow (rare): each lane evaluates its own
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) z[q] = ndtri_tail(uu[q]);
    } else if (total) {
      int o = off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) wq[o++] = z[q];
      __syncwarp();
      for (int k = lane; k < total; k += 32) wq[k] = ndtri_tail(wq[k]);
      __syncwarp();
      o = off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) z[q] = wq[o++];
      __syncwarp();
    }
    if (g < ng) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int x = x0 + q;
        if (x < a.ps1) {
          const double r = __ldg(&rq[min(x, a.ps1 - x)]);
          (x & 1 ? bo : be)[x >> 1] = make_double2(r * z[q], r * z[4 + q]);
        }
      }
    }
  }
  __syncthreads();
  fft_line<true, true, 1, true, 2>(half ? bo : be, pls, tl, 1 + half);
  __syncthreads();   // both halves
  double2* V = a.V + (int64_t)b * a.V_bstride;
  for (int ix = threadIdx.x; ix < a.keep; ix += blockDim.x)
    V[(int64_t)ix * a.ldV + iy] = cadd(be[ix], cmulc(bo[ix], split_w(wt, ix)));
}

// The same row pass with ONE half line per CTA of a 2-CTA cluster (two CTAs, i.e. two rows' worth of
// half lines, per SM, where cs_rowgen_split_kernel's single 140 KB CTA per SM cannot overlap its
// generation, transform and store phases).  A measured alternative (RK_CS_PAIR=1): no faster.  The row's Philox
// groups are dealt to the two CTAs warp by warp; each group's four elements alternate between
// the even and the odd half line, so every CTA stores two of them locally and two into its
// partner's line over DSMEM.  After the transforms the halves are combined as in the predict
// passes, each CTA finishing half the kept columns.  Same arithmetic per element as
// cs_rowgen_split_kernel: bitwise the same field.
constexpr int kCsPairThreads = 512;

template <bool AL = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCsPairThreads, 2) cs_rowgen_pair_kernel(const CsGenArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int half = (int)cl.block_rank();
  const int H = a.pl.n;
  const int tl = threadIdx.x;
  const int nthr = blockDim.x;   // == a.pl.nthr
  const int lane = tl & 31, warp = tl >> 5, nwarps = nthr >> 5;
  const int b = blockIdx.y;
  const int iy = blockIdx.x >> 1;
  double2* buf = smem;                                        // this CTA's half line (x % 2 == half)
  double2* remote = cl.map_shared_rank(buf, half ^ 1);
  double* wq = (double*)(smem + a.q_off) + (size_t)warp * kSplitQcap;
  uint64_t* xb = (uint64_t*)(smem + a.sw.off + 128 + a.sw.nhi);   // exit protection
  if (tl == 0) mbar_init(xb, 1);
  const FftPlan pls = fft_twiddles_to_smem(a.pl, smem + a.tw_off);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  const uint64_t fs = a.direct ? a.seed : draw_seed(draw_seed(a.seed, (uint64_t)(a.j0 + b)), 101);
  const uint64_t Ps = (uint64_t)a.ps1 * (uint64_t)a.ps2;
  const uint64_t wre = (uint64_t)iy * a.ps1, wim = Ps + wre;   // simulate.py:114-115
  const double* rq = a.root_q + (int64_t)min(iy, a.ps2 - iy) * a.rq_ld;
  const int ng = (a.ps1 + 3) / 4;
  cl.sync();   // the partner runs (remote stores may follow); publishes xb
  for (int c = 2 * warp + half; 32 * c < ng; c += 2 * nwarps) {   // warp-uniform: 32 groups per turn
    const int g = 32 * c + lane;
    const int x0 = 4 * g;
    uint64_t re[4], im[4];
    if (AL) {
      uint64_t fk;   // opaque per group (see cs_rowgen_kernel)
      asm volatile("mov.b64 %0, %1;" : "=l"(fk) : "l"(fs));
      philox4x64_10_x2(((wre + x0) >> 2) + 1, ((wim + x0) >> 2) + 1, fk, 0, re, im);
    } else {
      philox_words4(wre + x0, fs, re);
      philox_words4(wim + x0, fs, im);
    }
    double uu[8], z[8];
    unsigned tmask = 0;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      uu[q] = word_uniform(q < 4 ? re[q] : im[q - 4]);
      if (g < ng && (AL || x0 + (q & 3) < a.ps1) && ndtri_is_tail(uu[q])) tmask |= 1u << q;
    }
    ndtri_central_n<8>(uu, z);
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (tmask >> q & 1) z[q] = uu[q];
    const int cnt = __popc(tmask);
    int off = cnt;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, off, d);
      if (lane >= d) off += v;
    }
    const int total = __shfl_sync(0xffffffffu, off, 31);
    off -= cnt;
    if (total > min(kSplitQcap, a.qcap)) {   // queue overflow (rare): each lane evaluates its own
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) z[q] = ndtri_tail(uu[q]);
    } else if (total) {
      int o = off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) wq[o++] = z[q];
      __syncwarp();
      for (int k = lane; k < total; k += 32) wq[k] = ndtri_tail(wq[k]);
      __syncwarp();
      o = off;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (tmask >> q & 1) z[q] = wq[o++];
      __syncwarp();
    }
    if (g < ng) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int x = x0 + q;
        if (x < a.ps1) {
          const double r = __ldg(&rq[min(x, a.ps1 - x)]);
          ((q & 1) == half ? buf : remote)[x >> 1] = make_double2(r * z[q], r * z[4 + q]);   // x0 is even
        }
      }
    }
  }
  cl.sync();   // both CTAs' elements are in both half lines
  fft_line<true, true, 1, true, 2>(buf, pls, tl);
  cl.sync();   // both halves transformed
  const double2* other = cl.map_shared_rank(buf, half ^ 1);
  double2* V = a.V + (int64_t)b * a.V_bstride;
  const int km = (a.keep + 1) >> 1;
  const int i0 = half ? km : 0, i1 = half ? a.keep : km;
  for (int ix = i0 + tl; ix < i1; ix += nthr) {
    const double2 e = half ? other[ix] : buf[ix];
    const double2 o = half ? buf[ix] : other[ix];
    V[(int64_t)ix * a.ldV + iy] = cadd(e, cmulc(o, split_w(wt, ix)));
  }
  __syncthreads();   // this CTA's remote reads are done
  if (tl == 0) cluster_arrive_partner(xb, (uint32_t)(half ^ 1));
  cluster_wait_partner(xb);   // ... and the partner's, before this CTA's shared memory goes away
}

__global__ void __launch_bounds__(kFftWideThreads, 1) cs_col_split_kernel(const CsColArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int H = a.pl.n, P = 2 * H;
  const int nthr = a.pl.nthr;
  const int half = threadIdx.x / nthr;
  const int tl = threadIdx.x - half * nthr;
  const int b = blockIdx.y;
  const int ca = 2 * blockIdx.x, cb = ca + 1;
  double2* be = smem;
  double2* bo = smem + H;
  const double2* Va = a.V + (int64_t)b * a.V_bstride + (int64_t)ca * a.ldV;
  const double2* Vb = Va + a.ldV;
  const bool va = ca < a.ncols, vb = cb < a.ncols;
  const FftPlan pls = fft_twiddles_to_smem(a.pl, smem + a.tw_off);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  pdl_wait();
  for (int y = threadIdx.x; y < P; y += blockDim.x) {   // Hermitian parts, as cs_col_kernel
    const int m = y ? P - y : 0;
    const double2 A = va ? Va[y] : make_double2(0.0, 0.0), Am = va ? Va[m] : make_double2(0.0, 0.0);
    const double2 B = vb ? Vb[y] : make_double2(0.0, 0.0), Bm = vb ? Vb[m] : make_double2(0.0, 0.0);
    (y & 1 ? bo : be)[y >> 1] =
        make_double2(0.5 * ((A.x + Am.x) - (B.y - Bm.y)), 0.5 * ((A.y - Am.y) + (B.x + Bm.x)));
  }
  __syncthreads();
  fft_line<true, true, 1, true, 2>(half ? bo : be, pls, tl, 1 + half);
  __syncthreads();   // both halves
  double* g = a.g + (int64_t)b * a.g_bstride;
  for (int y = threadIdx.x; y < a.keep; y += blockDim.x) {
    const double2 v = cadd(be[y], cmulc(bo[y], split_w(wt, y)));
    if (va) g[(int64_t)y * a.ncols + ca] = v.x;
    if (vb) g[(int64_t)y * a.ncols + cb] = v.y;
  }
}

static Status uncond_fields(rk_setup* s, uint64_t seed, int64_t j0, int direct, int batch,
                            double* g, cudaStream_t st) {
  RK_TRY(ensure_embedding(s, st));
  const Embedding& e = s->emb;
  const int64_t ldV = (e.ps2 + 1) & ~1;
  double2* V = nullptr;
  RK_TRY(scratch_alloc((void**)&V, sizeof(double2) * (size_t)s->M1 * ldV * batch, st));
  double2* Zs = nullptr;   // freed after the column pass so the two FFT kernels stay adjacent
  static const bool fused = !(getenv("RK_CS_FUSED") && atoi(getenv("RK_CS_FUSED")) == 0);
  bool gen_done = false;
  if (fused && e.hs1v.v[2].n && 2 * e.hs1v.v[2].nthr <= kFftWideThreads) {   // split-length row pass
    CsGenArgs ga{};
    ga.pl = e.hs1v.v[2];
    ga.lpc = 1;
    ga.seed = seed;
    ga.j0 = j0;
    ga.direct = direct;
    ga.ps1 = e.ps1;
    ga.ps2 = e.ps2;
    ga.root_q = e.root_q;
    ga.rq_ld = e.hs1;
    ga.keep = s->M1;
    ga.V = V;
    ga.ldV = ldV;
    ga.V_bstride = (int64_t)s->M1 * ldV;
    static const int qcap_env2 = getenv("RK_CS_QCAP") ? atoi(getenv("RK_CS_QCAP")) : 1 << 30;
    ga.qcap = std::max(0, qcap_env2);
    ga.sw = e.sws1;
    const int threads = 2 * ga.pl.nthr;
    size_t by = sizeof(double2) * 2 * (size_t)ga.pl.n;
    ga.q_off = (int)((by + 15) / 16);
    by = (size_t)ga.q_off * 16 + sizeof(double) * (size_t)(threads / 32) * kSplitQcap;
    ga.tw_off = (int)((by + 15) / 16);
    by = (size_t)ga.tw_off * 16 + sizeof(double2) * (size_t)ga.pl.ntw;
    ga.sw.off = (int)((by + 15) / 16);
    by = (size_t)ga.sw.off * 16 + sizeof(double2) * (size_t)(128 + ga.sw.nhi);
    // RK_CS_PAIR=1: one half line per CTA of a 2-CTA cluster (two CTAs per SM) where it fits.
    // Bitwise the same field (test_gpu_variants) and measured no faster than the one-CTA kernel
    // (configs[4] CS 3.95 vs 3.94 ms per realization), so off by default.
    static const bool pair_env = getenv("RK_CS_PAIR") && atoi(getenv("RK_CS_PAIR")) != 0;
    if (pair_env && ga.pl.nthr <= kCsPairThreads) {
      CsGenArgs pa = ga;
      size_t pb = sizeof(double2) * (size_t)pa.pl.n;
      pa.q_off = (int)((pb + 15) / 16);
      pb = (size_t)pa.q_off * 16 + sizeof(double) * (size_t)(pa.pl.nthr / 32) * kSplitQcap;
      pa.tw_off = (int)((pb + 15) / 16);
      pb = (size_t)pa.tw_off * 16 + sizeof(double2) * (size_t)pa.pl.ntw;
      pa.sw.off = (int)((pb + 15) / 16);
      pb = (size_t)pa.sw.off * 16 + sizeof(double2) * (size_t)(128 + pa.sw.nhi) + 16;   // + the exit mbarrier
      if (pb <= 113 * 1024) {
        static const bool al_env = !(getenv("RK_CS_ALIGNED") && atoi(getenv("RK_CS_ALIGNED")) == 0);
        auto pkern = al_env && e.ps1 % 4 == 0 ? cs_rowgen_pair_kernel<true> : cs_rowgen_pair_kernel<false>;
        RK_TRY(set_smem_attr((const void*)pkern, pb));
        pkern<<<dim3((unsigned)(2 * e.ps2), (unsigned)batch), pa.pl.nthr, pb, st>>>(pa);
        count_launch();
        RK_LAUNCH_CHECK();
        gen_done = true;
      }
    }
    if (!gen_done && by <= 227 * 1024) {
      static const bool al_env = !(getenv("RK_CS_ALIGNED") && atoi(getenv("RK_CS_ALIGNED")) == 0);
      auto gkern = al_env && e.ps1 % 4 == 0 ? cs_rowgen_split_kernel<true> : cs_rowgen_split_kernel<false>;
      RK_TRY(set_smem_attr((const void*)gkern, by));
      gkern<<<dim3((unsigned)e.ps2, (unsigned)batch), threads, by, st>>>(ga);
      count_launch();
      RK_LAUNCH_CHECK();
      gen_done = true;
    }
  }
  if (gen_done) {
  } else if (fused) {
    CsGenArgs ga{};
    ga.pl = plan_pick(e.ps1v, (int64_t)e.ps2 * batch);
    ga.lpc = pick_lpc(ga.pl, 4, (int64_t)e.ps2 * batch);
    ga.seed = seed;
    ga.j0 = j0;
    ga.direct = direct;
    ga.ps1 = e.ps1;
    ga.ps2 = e.ps2;
    ga.root_q = e.root_q;
    ga.rq_ld = e.hs1;
    ga.keep = s->M1;
    ga.V = V;
    ga.ldV = ldV;
    ga.V_bstride = (int64_t)s->M1 * ldV;
    static const int qcap_env = getenv("RK_CS_QCAP") ? atoi(getenv("RK_CS_QCAP")) : 1 << 30;
    ga.qcap = std::max(0, qcap_env);
    const int warps = ga.lpc * ga.pl.nthr / 32;
    static const bool gen4 = !(getenv("RK_CS_GEN4") && atoi(getenv("RK_CS_GEN4")) == 0);
    const bool occ4 = gen4 && ga.pl.wide == 2 && ga.lpc == 1 && ga.pl.nthr <= 288;
    ga.q_off = (int)(ga.lpc * (size_t)e.ps1);
    ga.tw_off = ga.q_off + warps * (occ4 ? 64 : 128);   // 128 / 256 doubles per warp
    size_t smem = sizeof(double2) * ((size_t)ga.tw_off + ga.pl.ntw);
    const bool tws = !occ4 && smem <= 227 * 1024;
    if (!tws) smem = sizeof(double2) * (size_t)ga.tw_off;
    if (ga.pl.wide >= 2 && !tws && !occ4) return Status::err(RK_INTERNAL, "wide FFT plan without room for its twiddle table");
    static const bool al_env = !(getenv("RK_CS_ALIGNED") && atoi(getenv("RK_CS_ALIGNED")) == 0);
    const bool al = al_env && e.ps1 % 4 == 0;
    auto kern = occ4 ? (al ? cs_rowgen_kernel<false, 1, 288, 4, true> : cs_rowgen_kernel<false, 1, 288, 4>)
                : ga.pl.wide == 2 ? (al ? cs_rowgen_kernel<true, 1, kFftWideThreads, 1, true> : cs_rowgen_kernel<true, 1>)
                : ga.pl.wide == 3 ? cs_rowgen_kernel<true, 2>
                : tws ? cs_rowgen_kernel<true, 0> : cs_rowgen_kernel<false, 0>;
    RK_TRY(set_smem_attr((const void*)kern, smem));
    const dim3 grid((unsigned)ceil_div(e.ps2, ga.lpc), (unsigned)batch);
    kern<<<grid, ga.lpc * ga.pl.nthr, smem, st>>>(ga);
    count_launch();
    RK_LAUNCH_CHECK();
  } else {
    const int64_t Ps = (int64_t)e.ps1 * e.ps2;
    if (Ps >= (int64_t)1 << 31) return Status::err(RK_DOMAIN, "simulation torus larger than 2^31 nodes");
    double2* Z = nullptr;
    RK_TRY(scratch_alloc((void**)&Z, sizeof(double2) * (size_t)Ps * batch, st));
    CsRngArgs ga{};
    ga.seed = seed;
    ga.j0 = j0;
    ga.direct = direct;
    ga.ps1 = e.ps1;
    ga.ps2 = e.ps2;
    ga.root_q = e.root_q;
    ga.rq_ld = e.hs1;
    ga.Z = Z;
    ga.Z_bstride = Ps;
    const dim3 rgrid((unsigned)std::min<int64_t>(ceil_div(ceil_div(Ps, 4), kRngThreads), 148 * 8), (unsigned)batch);
    cs_rng_kernel<<<rgrid, kRngThreads, 0, st>>>(ga);
    count_launch();
    RK_LAUNCH_CHECK();
    CsFftArgs fa{};
    fa.pl = plan_pick(e.ps1v, (int64_t)e.ps2 * batch);
    fa.lpc = pick_lpc(fa.pl, 4, (int64_t)e.ps2 * batch);
    fa.ps2 = e.ps2;
    fa.keep = s->M1;
    fa.Z = Z;
    fa.Z_bstride = Ps;
    fa.V = V;
    fa.ldV = ldV;
    fa.V_bstride = (int64_t)s->M1 * ldV;
    const dim3 grid((unsigned)ceil_div(e.ps2, fa.lpc), (unsigned)batch);
    fa.tw_off = (int)(fa.lpc * (size_t)e.ps1) + 1;
    size_t smem = sizeof(double2) * (e.ps1 * (size_t)fa.lpc + 1 + fa.pl.ntw);
    const bool tws = smem <= 227 * 1024;   // else twiddles are read through L1/L2
    if (!tws) smem = sizeof(double2) * (e.ps1 * (size_t)fa.lpc + 1);
    if (fa.pl.wide >= 2 && !tws) return Status::err(RK_INTERNAL, "wide FFT plan without room for its twiddle table");
    auto kern = fa.pl.wide == 2 ? cs_rowfft_kernel<true, 1> : fa.pl.wide == 3 ? cs_rowfft_kernel<true, 2>
                : tws ? cs_rowfft_kernel<true, 0> : cs_rowfft_kernel<false, 0>;
    RK_TRY(set_smem_attr((const void*)kern, smem));
    RK_CUDA_TRY(launch_pdl(kern, grid, dim3(fa.lpc * fa.pl.nthr), smem, st, fa));
    count_launch();
    Zs = Z;
  }
  const int64_t cpairs = (s->M1 + 1) / 2;   // two columns per line
  if (e.hs2v.v[2].n && 2 * e.hs2v.v[2].nthr <= kFftWideThreads) {   // split-length column pass
    CsColArgs cs{};
    cs.pl = e.hs2v.v[2];
    cs.lpc = 1;
    cs.ncols = s->M1;
    cs.keep = s->M2;
    cs.V = V;
    cs.ldV = ldV;
    cs.V_bstride = (int64_t)s->M1 * ldV;
    cs.g = g;
    cs.g_bstride = (int64_t)s->M1 * s->M2;
    cs.sw = e.sws2;
    size_t by = sizeof(double2) * 2 * (size_t)cs.pl.n;
    cs.tw_off = (int)((by + 15) / 16);
    by = (size_t)cs.tw_off * 16 + sizeof(double2) * (size_t)cs.pl.ntw;
    cs.sw.off = (int)((by + 15) / 16);
    by = (size_t)cs.sw.off * 16 + sizeof(double2) * (size_t)(128 + cs.sw.nhi);
    if (by <= 227 * 1024) {
      RK_TRY(set_smem_attr((const void*)cs_col_split_kernel, by));
      RK_CUDA_TRY(launch_pdl(cs_col_split_kernel, dim3((unsigned)cpairs, (unsigned)batch), dim3(2 * cs.pl.nthr), by,
                             st, cs));
      count_launch();
      scratch_free(Zs, st);
      scratch_free(V, st);
      return Status::ok();
    }
  }
  CsColArgs ca{};
  ca.pl = plan_pick(e.ps2v, cpairs * batch);
  ca.lpc = pick_lpc(ca.pl, 4, cpairs * batch);
  ca.ncols = s->M1;
  ca.keep = s->M2;
  ca.V = V;
  ca.ldV = ldV;
  ca.V_bstride = (int64_t)s->M1 * ldV;
  ca.g = g;
  ca.g_bstride = (int64_t)s->M1 * s->M2;
  {
    const dim3 grid((unsigned)ceil_div(cpairs, ca.lpc), (unsigned)batch);
    ca.tw_off = (int)(ca.lpc * (size_t)e.ps2);
    size_t smem = sizeof(double2) * (e.ps2 * (size_t)ca.lpc + ca.pl.ntw);
    const bool tws = smem <= 227 * 1024;
    if (!tws) smem = sizeof(double2) * e.ps2 * (size_t)ca.lpc;
    if (ca.pl.wide >= 2 && !tws) return Status::err(RK_INTERNAL, "wide FFT plan without room for its twiddle table");
    auto kern = ca.pl.wide == 2 ? cs_col_kernel<true, 1> : ca.pl.wide == 3 ? cs_col_kernel<true, 2>
                : tws ? cs_col_kernel<true, 0> : cs_col_kernel<false, 0>;
    RK_TRY(set_smem_attr((const void*)kern, smem));
    RK_CUDA_TRY(launch_pdl(kern, grid, dim3(ca.lpc * ca.pl.nthr), smem, st, ca));
    count_launch();
  }
  scratch_free(Zs, st);
  scratch_free(V, st);
  return Status::ok();
}

static Status obs_local(const rk_setup* s, double tau2, const double* g, uint64_t seed, int64_t j0,
                        int direct, int batch, double* z, cudaStream_t st) {
  if (s->cond_var_min < -1.0e-10 * s->model.sigma2) {
    char b[160];
    snprintf(b, sizeof b, "negative conditional variance %.3e; K_N solve inconsistent",
             s->cond_var_min);
    return Status::err(RK_NUMERIC, b);
  }
  ObsArgs a;
  a.base = s->base;
  a.weights = s->weights;
  a.cond_var = s->cond_var;
  a.n = s->n;
  a.M = s->M;
  a.bs = s->bs;
  a.M1 = s->M1;
  a.g = g;
  a.g_bstride = (int64_t)s->M1 * s->M2;
  a.sqrt_tau2 = std::sqrt(tau2);
  a.seed = seed;
  a.j0 = j0;
  a.direct = direct;
  a.z = z;
  const dim3 grid((unsigned)std::min<int64_t>(ceil_div(s->n, 128), 4096), (unsigned)batch);
  obs_local_kernel<<<grid, 128, 0, st>>>(a);
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

}  // namespace rk

using namespace rk;

static int finish_sim(const Status& s) {
  if (!s.good()) rk::set_error(s.code, s.msg);
  return s.code;
}

extern "C" {

uint64_t rk_draw_seed(uint64_t seed, uint64_t j) { return draw_seed(seed, j); }

rk_status rk_philox_normals(uint64_t seed, uint64_t stream_id, uint64_t start, int64_t count,
                            double* out_dev, void* stream) {
  auto run = [&]() -> Status {
    if (count <= 0) return Status::ok();
    philox_kernel<<<(int)std::min<int64_t>(ceil_div(count, 256), 148 * 32), 256, 0,
                    (cudaStream_t)stream>>>(seed, stream_id, start, count, out_dev, nullptr);
    count_launch();
    RK_LAUNCH_CHECK();
    return Status::ok();
  };
  return (rk_status)finish_sim(run());
}

rk_status rk_philox_raw(uint64_t seed, uint64_t stream_id, uint64_t start, int64_t count,
                        uint64_t* out_dev, void* stream) {
  auto run = [&]() -> Status {
    if (count <= 0) return Status::ok();
    philox_kernel<<<(int)std::min<int64_t>(ceil_div(count, 256), 148 * 32), 256, 0,
                    (cudaStream_t)stream>>>(seed, stream_id, start, count, nullptr, out_dev);
    count_launch();
    RK_LAUNCH_CHECK();
    return Status::ok();
  };
  return (rk_status)finish_sim(run());
}

rk_status rk_setup_embedding(rk_setup* s, int32_t embed_out[2], int32_t* doubled) {
  Status st = ensure_embedding(s, 0);
  if (st.good()) {
    if (embed_out) { embed_out[0] = s->emb.ps1; embed_out[1] = s->emb.ps2; }
    if (doubled) *doubled = s->emb.doubled;
  }
  return (rk_status)finish_sim(st);
}

rk_status rk_sim_unconditional_dev(rk_setup* s, uint64_t seed, double* field_dev, void* stream) {
  return (rk_status)finish_sim(uncond_fields(s, seed, 0, 1, 1, field_dev, (cudaStream_t)stream));
}

rk_status rk_sim_obs_local_dev(const rk_setup* s, double tau2, const double* field_dev, uint64_t seed,
                               double* z_dev, void* stream) {
  return (rk_status)finish_sim(obs_local(s, tau2, field_dev, seed, 0, 1, 1, z_dev, (cudaStream_t)stream));
}

rk_status rk_ensemble_accumulate(rk_setup* s, const rk_fit* f, uint64_t seed, int64_t j0, int64_t count,
                                 const double* xg_dev, const double* data_pred_dev, long long* acc_dev,
                                 double* draws_dev, int32_t batch, void* stream) {
  auto run = [&]() -> Status {
    cudaStream_t st = (cudaStream_t)stream;
    if (f->n != s->n) return Status::err(RK_DOMAIN, "fit and setup disagree on the number of observations");
    if (!xg_dev && f->p != 1)
      return Status::err(RK_DOMAIN, "grid covariates are required when beta_hat has more than one entry");
    if (count <= 0) return Status::ok();
    if (count > (int64_t)1 << 21)
      return Status::err(RK_DOMAIN, "at most 2^21 realizations per accumulator");
    RK_TRY(ensure_embedding(s, st));
    RK_TRY(ensure_uinv(const_cast<rk_fit*>(f), st));
    // Realizations per field pass (B) are capped so the per-pass FFT scratch (V, T, U, e)
    // stays within ~8 GB.  The refit, whose cost is reading the n x n inverse factor twice,
    // runs once per super-batch of up to `count` realizations: their unconditional fields
    // are kept (up to ~16 GB) between the simulation passes and the prediction passes.
    const double per_real = 16.0 * ((double)s->M1 * s->emb.ps2 + 2.0 * s->H1 * s->M2) + 8.0 * (double)s->m1 * s->m2;
    const int B = std::max(1, std::min((int)batch, (int)(8.0e9 / per_real)));
    const int64_t gsz = (int64_t)s->M1 * s->M2;
    const int64_t S = std::max<int64_t>(B, std::min<int64_t>(count, (int64_t)(16.0e9 / (8.0 * gsz))));
    const int64_t npix = (int64_t)s->m1 * s->m2;
    const double scale = fx_scale(f->model.sigma2);
    double *G = nullptr, *Z = nullptr, *C = nullptr, *BT = nullptr, *E = nullptr;
    int* bad = nullptr;
    RK_TRY(scratch_alloc((void**)&G, sizeof(double) * (size_t)gsz * S, st));
    RK_TRY(scratch_alloc((void**)&Z, sizeof(double) * (size_t)s->n * S, st));
    RK_TRY(scratch_alloc((void**)&C, sizeof(double) * (size_t)s->n * S, st));
    RK_TRY(scratch_alloc((void**)&BT, sizeof(double) * (size_t)f->p * S, st));
    RK_TRY(scratch_alloc((void**)&E, sizeof(double) * (size_t)npix * B, st));
    RK_TRY(scratch_alloc((void**)&bad, sizeof(int), st));
    RK_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
    for (int64_t js = j0; js < j0 + count; js += S) {
      const int64_t sc = std::min<int64_t>(S, j0 + count - js);
      for (int64_t k = 0; k < sc; k += B) {   // unconditional fields + simulated observations
        const int bc = (int)std::min<int64_t>(B, sc - k);
        RK_TRY(uncond_fields(s, seed, js + k, 0, bc, G + k * gsz, st));
        RK_TRY(obs_local(s, f->model.tau2, G + k * gsz, seed, js + k, 0, bc, Z + k * s->n, st));
      }
      RK_TRY(gls_batch(f, Z, sc, BT, C, st));
      for (int64_t k = 0; k < sc; k += B) {   // e = interior(g) - predict(c_sim, beta_sim)
        const int bc = (int)std::min<int64_t>(B, sc - k);
        PredictBatch pb;
        pb.batch = bc;
        pb.c = C + k * s->n;
        pb.c_stride = s->n;
        pb.beta = BT + k * f->p;
        pb.p = f->p;
        pb.xg = xg_dev;
        pb.g = G + k * gsz;
        pb.out = E;
        RK_TRY(predict_batch(s, pb, st));
        accumulate_fx_kernel<<<(int)std::min<int64_t>(ceil_div(npix, 256), 148 * 16), 256, 0, st>>>(
            E, bc, npix, data_pred_dev, 1.0 / scale, acc_dev,
            draws_dev ? draws_dev + (js + k - j0) * npix : nullptr, bad);
        count_launch();
        RK_LAUNCH_CHECK();
      }
    }
    int hb = 0;
    RK_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    scratch_free(G, st);
    scratch_free(Z, st);
    scratch_free(C, st);
    scratch_free(BT, st);
    scratch_free(E, st);
    scratch_free(bad, st);
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    if (hb)
      return Status::err(RK_NUMERIC, "conditional draw deviates from the data prediction by more than 2^20 sigma "
                                     "(or is not finite)");
    return Status::ok();
  };
  return (rk_status)finish_sim(run());
}

// the fixed-point accumulation alone, on caller values: acc += moments of e_dev (count, n_pix)
// (tests pin the integer arithmetic against exact host sums)
rk_status rk_ensemble_accumulate_values(const double* e_dev, int32_t count, int64_t n_pix, double sigma2,
                                        long long* acc_dev, void* stream) {
  auto run = [&]() -> Status {
    cudaStream_t st = (cudaStream_t)stream;
    int* bad = nullptr;
    RK_TRY(scratch_alloc((void**)&bad, sizeof(int), st));
    RK_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
    accumulate_fx_kernel<<<(int)std::min<int64_t>(ceil_div(n_pix, 256), 148 * 16), 256, 0, st>>>(
        e_dev, count, n_pix, e_dev, 1.0 / fx_scale(sigma2), acc_dev, nullptr, bad);
    count_launch();
    RK_LAUNCH_CHECK();
    int hb = 0;
    RK_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    scratch_free(bad, st);
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    if (hb) return Status::err(RK_NUMERIC, "value outside the fixed-point range (>= 2^20 sigma or not finite)");
    return Status::ok();
  };
  return (rk_status)finish_sim(run());
}

rk_status rk_ensemble_combine(long long* dst_dev, const long long* src_dev, int64_t n_pix, void* stream) {
  auto run = [&]() -> Status {
    const int64_t n = 6 * n_pix;
    acc_add_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 148 * 16), 256, 0, (cudaStream_t)stream>>>(
        dst_dev, src_dev, n);
    count_launch();
    RK_LAUNCH_CHECK();
    return Status::ok();
  };
  return (rk_status)finish_sim(run());
}

rk_status rk_ensemble_finalize(int64_t n_pix, int64_t n_draws, double sigma2, const double* data_pred_dev,
                               const long long* acc_dev, double* mean_dev, double* se_dev, void* stream) {
  auto run = [&]() -> Status {
    if (n_draws < 2) return Status::err(RK_DOMAIN, "need at least 2 draws, got " + std::to_string(n_draws));
    finalize_fx_kernel<<<(int)std::min<int64_t>(ceil_div(n_pix, 256), 148 * 16), 256, 0,
                         (cudaStream_t)stream>>>(n_pix, (double)n_draws, fx_scale(sigma2), data_pred_dev, acc_dev,
                                                 mean_dev, se_dev);
    count_launch();
    RK_LAUNCH_CHECK();
    return Status::ok();
  };
  return (rk_status)finish_sim(run());
}

}  // extern "C"
