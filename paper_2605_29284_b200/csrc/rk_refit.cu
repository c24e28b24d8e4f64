// rapidkrig B200: the batched GLS refit of the conditional-simulation path on FP64 tensor cores.
//
// Reference mapping (/root/reference/pkg/src/rapidkrig/exact.py):
//   refit_coefficients 108-113 -> _gls 59-68:  a = L^-1 z ; b = L^-1 X ; beta = (b'b)^-1 b'a ;
//                                             half = L^-1 (z - X beta) ; c = L^-T half
//
// The n x n factor is shared by every realization of an ensemble, so a batch of S right-hand
// sides is refit with the inverse factor L^-1 (built once per fit, ensure_uinv) as two
// triangular-matrix x panel products -- both read the SAME n x n triangle:
//   A = L^-1 Z                         (trmm_panel_kernel<false>)
//   beta = (B'B)^-1 B'A                (bta_kernel + gram_solve_kernel; B = L^-1 X from the fit)
//   H = A - B beta   (= L^-1 (Z - X beta), the reference's third solve, by linearity)
//   C = L^-T H                         (trmm_panel_kernel<true>)
//
// trmm_panel_kernel: 128 x 64 output tiles (rows x right-hand sides), 8 warps of 32 x 32, each
// a 4 x 4 grid of mma.sync.m8n8k4 f64 (DMMA) tiles; K in steps of 16 through a 3-stage
// cp.async ring.  Only the k range the triangle touches is visited (the other triangle of
// the stored inverse holds exact zeros, so a tile straddling the diagonal needs no masking).
// Every output column is a function of its own right-hand side only, accumulated in the same
// k order whatever the batch size: a realization's refit is bitwise independent of how many
// realizations share the launch (and of which GPU runs it).
#include <algorithm>
#include <cmath>
#include <mutex>

#include "rk_internal.cuh"

namespace rk {

constexpr int TR_BM = 128, TR_BN = 64, TR_BK = 16, TR_STAGES = 3, TR_THREADS = 256;
constexpr int TR_LDA = TR_BK + 4;    // row-major A tile [BM][BK + 4]  (A = L^-1 rows)
constexpr int TR_LDAT = TR_BM + 4;   // k-major A tile  [BK][BM + 4]   (A = L^-T: columns of L^-1)
constexpr int TR_LDB = TR_BK + 4;    // panel tile      [BN][BK + 4]
constexpr int TR_A_ELEMS = TR_BM * TR_LDA > TR_BK * TR_LDAT ? TR_BM * TR_LDA : TR_BK * TR_LDAT;
constexpr int TR_B_ELEMS = TR_BN * TR_LDB;
constexpr size_t TR_SMEM = sizeof(double) * (size_t)TR_STAGES * (TR_A_ELEMS + TR_B_ELEMS);

struct TrmmArgs {
  const double* Li;   // L^-1, row-major lower (element (i, k) at Li[i * ld + k]); exact zeros above
  int64_t ld, n;
  const double* X;    // (n, S) column-major, leading dimension ldx
  int64_t ldx;
  int S;
  double* out;        // (n, S) column-major, leading dimension ldo
  int64_t ldo;
};

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// asynchronous copies with zero fill (src_bytes = 0 -> the destination is zeroed)
__device__ __forceinline__ void cp_async16z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async8z(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 8 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// TRANS = false: out = L^-1 X  (row band i0: k in [0, i0 + BM))
// TRANS = true:  out = L^-T X  (row band j0: k in [j0, n)), out[j] = sum_k Li[k][j] X[k]
// V16: 16-byte copies (ld, ldx even and both bases 16-byte aligned), else 8-byte copies
template <bool TRANS, bool V16>
__global__ void __launch_bounds__(TR_THREADS, 2) trmm_panel_kernel(const TrmmArgs a) {
  extern __shared__ __align__(16) double tsm[];
  double* As = tsm;                                   // [STAGES][A_ELEMS]
  double* Bs = tsm + (size_t)TR_STAGES * TR_A_ELEMS;  // [STAGES][B_ELEMS]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;            // 4 x 2 warps of 32 x 32
  const int nb = (int)((a.n + TR_BM - 1) / TR_BM);
  // heaviest row bands first: they have the longest k range
  const int band = TRANS ? (int)blockIdx.y : nb - 1 - (int)blockIdx.y;
  const int64_t r0 = (int64_t)band * TR_BM;
  const int b0 = blockIdx.x * TR_BN;
  const int64_t kbeg = TRANS ? r0 / TR_BK * TR_BK : 0;
  const int64_t kend = TRANS ? a.n : (a.n < r0 + TR_BM ? a.n : r0 + TR_BM);
  const int nk = (int)((kend - kbeg + TR_BK - 1) / TR_BK);

  auto load = [&](int kt, int stage) {
    const int64_t k0 = kbeg + (int64_t)kt * TR_BK;
    double* as = As + (size_t)stage * TR_A_ELEMS;
    double* bs = Bs + (size_t)stage * TR_B_ELEMS;
    if (V16) {
      if (!TRANS) {   // 128 rows x 8 pairs
#pragma unroll
        for (int q = 0; q < TR_BM * (TR_BK / 2) / TR_THREADS; ++q) {
          const int e = tid + q * TR_THREADS;
          const int r = e >> 3, c = (e & 7) * 2;
          const int64_t gi = r0 + r, gk = k0 + c;
          const bool ok = gi < a.n && gk < a.n;
          cp_async16z(as + r * TR_LDA + c, ok ? a.Li + gi * a.ld + gk : a.Li, ok);
        }
      } else {        // 16 k-rows x 64 pairs
#pragma unroll
        for (int q = 0; q < TR_BK * (TR_BM / 2) / TR_THREADS; ++q) {
          const int e = tid + q * TR_THREADS;
          const int kk = e >> 6, c = (e & 63) * 2;
          const int64_t gk = k0 + kk, gj = r0 + c;
          const bool ok = gk < a.n && gj < a.n;
          cp_async16z(as + kk * TR_LDAT + c, ok ? a.Li + gk * a.ld + gj : a.Li, ok);
        }
      }
#pragma unroll
      for (int q = 0; q < TR_BN * (TR_BK / 2) / TR_THREADS; ++q) {   // 64 columns x 8 pairs
        const int e = tid + q * TR_THREADS;
        const int bb = e >> 3, c = (e & 7) * 2;
        const int64_t gk = k0 + c;
        const bool ok = b0 + bb < a.S && gk < a.n;
        cp_async16z(bs + bb * TR_LDB + c, ok ? a.X + (int64_t)(b0 + bb) * a.ldx + gk : a.X, ok);
      }
    } else {
      if (!TRANS) {
#pragma unroll 4
        for (int q = 0; q < TR_BM * TR_BK / TR_THREADS; ++q) {
          const int e = tid + q * TR_THREADS;
          const int r = e >> 4, c = e & 15;
          const int64_t gi = r0 + r, gk = k0 + c;
          const bool ok = gi < a.n && gk < a.n;
          cp_async8z(as + r * TR_LDA + c, ok ? a.Li + gi * a.ld + gk : a.Li, ok);
        }
      } else {
#pragma unroll 4
        for (int q = 0; q < TR_BK * TR_BM / TR_THREADS; ++q) {
          const int e = tid + q * TR_THREADS;
          const int kk = e >> 7, c = e & 127;
          const int64_t gk = k0 + kk, gj = r0 + c;
          const bool ok = gk < a.n && gj < a.n;
          cp_async8z(as + kk * TR_LDAT + c, ok ? a.Li + gk * a.ld + gj : a.Li, ok);
        }
      }
#pragma unroll
      for (int q = 0; q < TR_BN * TR_BK / TR_THREADS; ++q) {
        const int e = tid + q * TR_THREADS;
        const int bb = e >> 4, c = e & 15;
        const int64_t gk = k0 + c;
        const bool ok = b0 + bb < a.S && gk < a.n;
        cp_async8z(bs + bb * TR_LDB + c, ok ? a.X + (int64_t)(b0 + bb) * a.ldx + gk : a.X, ok);
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int s = 0; s < TR_STAGES - 1; ++s) {
    if (s < nk) load(s, s);
    cp_async_commit();
  }
  const int g = lane >> 2, t4 = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<TR_STAGES - 2>();
    __syncthreads();
    if (kt + TR_STAGES - 1 < nk) load(kt + TR_STAGES - 1, (kt + TR_STAGES - 1) % TR_STAGES);
    cp_async_commit();
    const int stage = kt % TR_STAGES;
    const double* as = As + (size_t)stage * TR_A_ELEMS;
    const double* bs = Bs + (size_t)stage * TR_B_ELEMS;
#pragma unroll
    for (int k4 = 0; k4 < TR_BK / 4; ++k4) {
      double af[4], bf[4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) {
        const int r = wm * 32 + mi * 8 + g, k = k4 * 4 + t4;
        af[mi] = TRANS ? as[k * TR_LDAT + r] : as[r * TR_LDA + k];
      }
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = bs[(wn * 32 + ni * 8 + g) * TR_LDB + k4 * 4 + t4];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma884(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  cp_async_wait<0>();
  // epilogue: C fragment element (g, 2 t4 + e) of each 8 x 8 tile
#pragma unroll
  for (int mi = 0; mi < 4; ++mi) {
    const int64_t row = r0 + wm * 32 + mi * 8 + g;
    if (row >= a.n) continue;
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = b0 + wn * 32 + ni * 8 + 2 * t4 + e;
        if (col < a.S) a.out[(int64_t)col * a.ldo + row] = acc[mi][ni][e];
      }
  }
}

// rhs[b, q] = sum_i B[i, q] A[i, b]  (p <= 8) -- one CTA per right-hand side, fixed order:
// thread-strided partial sums, then a fixed shared-memory tree
constexpr int kBtaThreads = 256;
__global__ void __launch_bounds__(kBtaThreads) bta_kernel(const double* __restrict__ B, int64_t n, int p,
                                                          const double* __restrict__ A, int64_t lda,
                                                          double* __restrict__ rhs) {
  __shared__ double red[8][kBtaThreads];
  const int b = blockIdx.x;
  const double* col = A + (int64_t)b * lda;
  double s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = threadIdx.x; i < n; i += kBtaThreads) {
    const double v = col[i];
#pragma unroll
    for (int q = 0; q < 8; ++q)
      if (q < p) s[q] = fma(B[(int64_t)q * n + i], v, s[q]);
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) red[q][threadIdx.x] = s[q];
  __syncthreads();
  for (int h = kBtaThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h)
#pragma unroll
      for (int q = 0; q < 8; ++q) red[q][threadIdx.x] += red[q][threadIdx.x + h];
    __syncthreads();
  }
  if (threadIdx.x < p) rhs[(int64_t)b * p + threadIdx.x] = red[threadIdx.x][0];
}

static Status launch_trmm(bool trans, const TrmmArgs& a, cudaStream_t st) {
  if (a.n <= 0 || a.S <= 0) return Status::ok();
  const bool v16 = (a.ld % 2 == 0) && (a.ldx % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.Li) & 15) == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.X) & 15) == 0);
  auto kern = trans ? (v16 ? trmm_panel_kernel<true, true> : trmm_panel_kernel<true, false>)
                    : (v16 ? trmm_panel_kernel<false, true> : trmm_panel_kernel<false, false>);
  RK_TRY(set_smem_attr((const void*)kern, TR_SMEM));
  const dim3 grid((unsigned)ceil_div(a.S, TR_BN), (unsigned)ceil_div(a.n, TR_BM));
  kern<<<grid, TR_THREADS, TR_SMEM, st>>>(a);
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

// out (n x S) = L^-1 X  or  L^-T X with the fit's inverse factor (U^-1 column-major upper is
// L^-1 row-major lower)
Status trmm_linv(const rk_fit* f, bool trans, const double* X, int64_t ldx, int64_t S, double* out, int64_t ldo,
                 cudaStream_t st) {
  for (int64_t s0 = 0; s0 < S; s0 += 65535LL * TR_BN) {   // grid.x limit
    TrmmArgs a;
    a.Li = f->Uinv;
    a.ld = f->n;
    a.n = f->n;
    a.X = X + s0 * ldx;
    a.ldx = ldx;
    a.S = (int)std::min<int64_t>(S - s0, 65535LL * TR_BN);
    a.out = out + s0 * ldo;
    a.ldo = ldo;
    RK_TRY(launch_trmm(trans, a, st));
  }
  return Status::ok();
}

Status bta(const rk_fit* f, const double* A, int64_t lda, int64_t S, double* rhs, cudaStream_t st) {
  for (int64_t s0 = 0; s0 < S; s0 += 1 << 30) {
    const int64_t m = std::min<int64_t>(S - s0, 1 << 30);
    bta_kernel<<<(unsigned)m, kBtaThreads, 0, st>>>(f->B, f->n, f->p, A + s0 * lda, lda, rhs + s0 * f->p);
    count_launch();
    RK_LAUNCH_CHECK();
  }
  return Status::ok();
}

}  // namespace rk

using namespace rk;

namespace {
__global__ void fill_panel_kernel(double* z, int64_t tot) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x)
    z[i] = 1.0 + (double)(i % 1013) * 1.0e-3;
}
int finish_refit(const Status& s) {
  if (!s.good()) rk::set_error(s.code, s.msg);
  return s.code;
}
}  // namespace

extern "C" {

// Kernel timing for the refit roofline: the two triangular panel products (L^-1 Z, L^-T H) of
// a refit of S right-hand sides, CUDA events on `stream`, average over reps (ms_out[0], [1]).
rk_status rk_refit_profile(rk_fit* f, int64_t S, int32_t reps, void* stream, float* ms_out) {
  auto run = [&]() -> Status {
    cudaStream_t st = (cudaStream_t)stream;
    RK_TRY(ensure_uinv(f, st));
    const int64_t n = f->n;
    double *Z = nullptr, *A = nullptr;
    RK_TRY(scratch_alloc((void**)&Z, sizeof(double) * (size_t)n * S, st));
    RK_TRY(scratch_alloc((void**)&A, sizeof(double) * (size_t)n * S, st));
    fill_panel_kernel<<<148 * 8, 256, 0, st>>>(Z, n * S);
    count_launch();
    cudaEvent_t e[3];
    for (auto& x : e) RK_CUDA_TRY(cudaEventCreate(&x));
    RK_TRY(trmm_linv(f, false, Z, n, S, A, n, st));   // warm-up
    RK_TRY(trmm_linv(f, true, A, n, S, Z, n, st));
    RK_CUDA_TRY(cudaEventRecord(e[0], st));
    for (int r = 0; r < reps; ++r) RK_TRY(trmm_linv(f, false, Z, n, S, A, n, st));
    RK_CUDA_TRY(cudaEventRecord(e[1], st));
    for (int r = 0; r < reps; ++r) RK_TRY(trmm_linv(f, true, A, n, S, Z, n, st));
    RK_CUDA_TRY(cudaEventRecord(e[2], st));
    RK_CUDA_TRY(cudaEventSynchronize(e[2]));
    RK_CUDA_TRY(cudaEventElapsedTime(&ms_out[0], e[0], e[1]));
    RK_CUDA_TRY(cudaEventElapsedTime(&ms_out[1], e[1], e[2]));
    ms_out[0] /= reps;
    ms_out[1] /= reps;
    for (auto& x : e) cudaEventDestroy(x);
    scratch_free(Z, st);
    scratch_free(A, st);
    return Status::ok();
  };
  return (rk_status)finish_refit(run());
}

}  // extern "C"
