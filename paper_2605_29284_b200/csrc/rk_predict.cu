// rapidkrig B200: rapid predict = deterministic scatter + circulant FFT convolution.
//
// Reference mapping (/root/reference/pkg/src/rapidkrig/rapid.py):
//   coefficients_to_grid 164-174 (np.add.at)  -> cstar_at(): per-node GATHER over the
//       cell-sorted observations (fixed order, no atomics), fused into pass 1
//   convolve_filter 89-100 (fft2 * spectrum, ifft2, crop) -> 3 passes:
//       pass 1 row_fwd_kernel : two real padded rows per complex FFT (length p1),
//                               split into two half spectra, written transposed T[kx][y]
//       pass 2 col_kernel     : column kx: FFT(p2) of the M2 nonzero rows, x real even
//                               spectrum (quarter stored, 1/(p1 p2) folded in), IFFT,
//                               keep only the m2 interior rows -> U[kx][y']
//       pass 3 row_inv_kernel : Hermitian-combined pair of interior rows, IFFT(p1),
//                               keep the m1 interior columns, fused epilogue
//   _fixed_part 233-249 / predict_rapid 252-261 -> epilogue of pass 3
//   build_filter_spectrum 72-86 -> spectrum_quarter(): lag table on the quarter torus,
//       pass 1 (lag mode) + pass 2 (spectrum mode, real part of ky <= p2/2)
#include <algorithm>

#include "rk_internal.cuh"

namespace rk {

// ----------------------------------------------------------------- gather
struct GatherSrc {
  const int32_t* cell_start;
  const int32_t* bsort;
  const int32_t* perm;
  const double* wsort;
  const double* c;
  int64_t c_stride;
  int M1, M2, bs, M;
};

// c*[y, x] = sum over observations whose 2L x 2L block covers (y, x) of w * c,
// visiting base rows by = y .. y-2L+1 and, inside each, the contiguous sorted
// range of bases bx in [x-2L+1, x].
__device__ __forceinline__ double cstar_at(const GatherSrc& g, const double* __restrict__ c, int y,
                                           int x) {
  double acc = 0.0;
  const int xlo = max(0, x - g.bs + 1);
  const int xhi = min(x, g.M1 - g.bs);
  if (xlo > xhi) return 0.0;
  for (int dy = 0; dy < g.bs; ++dy) {
    const int by = y - dy;
    if (by < 0 || by > g.M2 - g.bs) continue;
    const int rowb = by * g.M1;
    const int j0 = __ldg(&g.cell_start[rowb + xlo]);
    const int j1 = __ldg(&g.cell_start[rowb + xhi + 1]);
    for (int j = j0; j < j1; ++j) {
      const int bx = __ldg(&g.bsort[j]) - rowb;
      const double w = __ldg(&g.wsort[(int64_t)j * g.M + dy * g.bs + (x - bx)]);
      const double cj = __ldg(&c[__ldg(&g.perm[j])]);
      acc = __dadd_rn(acc, __dmul_rn(w, cj));   // (w * c) then add, as np.add.at
    }
  }
  return acc;
}

__global__ void cstar_kernel(GatherSrc g, double* __restrict__ out) {
  const int64_t tot = (int64_t)g.M1 * g.M2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int y = (int)(e / g.M1), x = (int)(e % g.M1);
    out[e] = cstar_at(g, g.c, y, x);
  }
}

// ----------------------------------------------------------------- pass 1
enum RowSrc { SRC_GATHER = 0, SRC_REAL = 1, SRC_LAG = 2 };

struct RowFwdArgs {
  FftPlan pl;
  int lpc;
  int nrows;                 // input rows
  int ncols;                 // nonzero input columns
  double2* T;                // (H, ldT) per batch
  int64_t ldT, T_bstride;
  GatherSrc g;               // SRC_GATHER
  const double* real_in;     // SRC_REAL: (nrows, ncols) row-major
  const double* lagq;        // SRC_LAG: quarter lag table (p2/2+1, p1/2+1)
  int lag_ld, p2;
};

template <int SRC>
__global__ void __launch_bounds__(512, 1) row_fwd_kernel(const RowFwdArgs a) {
  extern __shared__ double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  double2* buf = smem + (size_t)line * n;
  const int ya = 2 * (blockIdx.x * a.lpc + line);
  const int yb = ya + 1;
  const bool va = ya < a.nrows, vb = yb < a.nrows;
  const double* cb = (SRC == SRC_GATHER) ? a.g.c + (int64_t)b * a.g.c_stride : nullptr;
  for (int x = tl; x < n; x += nthr) {
    double u = 0.0, v = 0.0;
    if (x < a.ncols) {
      if (SRC == SRC_GATHER) {
        if (va) u = cstar_at(a.g, cb, ya, x);
        if (vb) v = cstar_at(a.g, cb, yb, x);
      } else if (SRC == SRC_REAL) {
        if (va) u = a.real_in[(int64_t)ya * a.ncols + x];
        if (vb) v = a.real_in[(int64_t)yb * a.ncols + x];
      } else {
        const int bx = min(x, n - x);
        if (va) u = __ldg(&a.lagq[(int64_t)min(ya, a.p2 - ya) * a.lag_ld + bx]);
        if (vb) v = __ldg(&a.lagq[(int64_t)min(yb, a.p2 - yb) * a.lag_ld + bx]);
      }
    }
    buf[x] = make_double2(u, v);
  }
  __syncthreads();
  fft_line<false>(buf, a.pl, tl);
  // split Z = FFT(u + i v) into U = (Z + conj Z[-k]) / 2, V = (Z - conj Z[-k]) / 2i
  const int nr = 2 * a.lpc;
  const int H = n / 2 + 1;
  double2* T = a.T + (int64_t)b * a.T_bstride;
  for (int idx = threadIdx.x; idx < H * nr; idx += blockDim.x) {
    const int r = idx % nr, kx = idx / nr;
    const int l = r >> 1;
    const int row = 2 * (blockIdx.x * a.lpc + l) + (r & 1);
    if (row >= a.nrows) continue;
    const double2* bl = smem + (size_t)l * n;
    const double2 z = bl[kx];
    const double2 zc = bl[kx == 0 ? 0 : n - kx];
    double2 o;
    if ((r & 1) == 0) o = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
    else o = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
    T[(int64_t)kx * a.ldT + row] = o;
  }
}

// ----------------------------------------------------------------- pass 2
struct ColArgs {
  FftPlan pl;
  int lpc;
  int ncols;                 // number of columns (kx)
  int nin;                   // nonzero input rows
  const double2* T;
  int64_t ldT, T_bstride;
  const double* spec_q;      // filter mode: (ncols, Q2)
  int Q2;
  int row0, nout;            // filter mode: keep rows [row0, row0 + nout)
  double2* U;
  int64_t ldU, U_bstride;
  double* out_q;             // spectrum mode: out_q[kx * Q2 + ky] = Re * scale
  double scale;
};

template <int MODE>  // 0 = filter (fwd, x spectrum, inv, crop), 1 = spectrum (fwd, real part)
__global__ void __launch_bounds__(512, 1) col_kernel(const ColArgs a) {
  extern __shared__ double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  const int kx = blockIdx.x * a.lpc + line;
  const bool valid = kx < a.ncols;
  double2* buf = smem + (size_t)line * n;
  const double2* T = a.T + (int64_t)b * a.T_bstride + (int64_t)kx * a.ldT;
  for (int y = tl; y < n; y += nthr)
    buf[y] = (valid && y < a.nin) ? T[y] : make_double2(0.0, 0.0);
  __syncthreads();
  fft_line<false>(buf, a.pl, tl);
  if (MODE == 0) {
    if (valid) {
      const double* S = a.spec_q + (int64_t)kx * a.Q2;
      for (int ky = tl; ky < n; ky += nthr) buf[ky] = cscale(buf[ky], __ldg(&S[min(ky, n - ky)]));
    }
    __syncthreads();
    fft_line<true>(buf, a.pl, tl);
    if (valid) {
      double2* U = a.U + (int64_t)b * a.U_bstride + (int64_t)kx * a.ldU;
      for (int y = tl; y < a.nout; y += nthr) U[y] = buf[a.row0 + y];
    }
  } else {
    if (valid)
      for (int ky = tl; ky < a.Q2; ky += nthr) a.out_q[(int64_t)kx * a.Q2 + ky] = buf[ky].x * a.scale;
  }
}

// ----------------------------------------------------------------- pass 3
struct RowInvArgs {
  FftPlan pl;
  int lpc;
  int nrows;                 // output rows (rows of U)
  const double2* U;
  int64_t ldU, U_bstride;
  int col0, ncols;           // output columns [col0, col0 + ncols) of the padded row
  double* out;
  int64_t ldo, out_bstride;
  int epi;                   // EpiMode
  const double* beta;        // (batch, p)
  int p;
  const double* xg;          // (nrows * ncols, p)
  const double* g;           // CS: unconditional fields (batch, M2, M1), or null
  int64_t g_bstride;
  int g_ld, g_row0, g_col0;
};

__global__ void __launch_bounds__(512, 1) row_inv_kernel(const RowInvArgs a) {
  extern __shared__ double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  const int H = n / 2 + 1;
  const double2* U = a.U + (int64_t)b * a.U_bstride;
  // coalesced load of both rows of every line: Z[k] = A[k] + i B[k], Hermitian upper half
  for (int idx = threadIdx.x; idx < a.lpc * H; idx += blockDim.x) {
    const int l = idx % a.lpc, k = idx / a.lpc;
    const int ya = 2 * (blockIdx.x * a.lpc + l);
    const double2 A = ya < a.nrows ? U[(int64_t)k * a.ldU + ya] : make_double2(0.0, 0.0);
    const double2 B = ya + 1 < a.nrows ? U[(int64_t)k * a.ldU + ya + 1] : make_double2(0.0, 0.0);
    double2* bl = smem + (size_t)l * n;
    bl[k] = make_double2(A.x - B.y, A.y + B.x);
    if (k >= 1 && k <= n - H) bl[n - k] = make_double2(A.x + B.y, B.x - A.y);
  }
  __syncthreads();
  double2* buf = smem + (size_t)line * n;
  fft_line<true>(buf, a.pl, tl);
  const int ya = 2 * (blockIdx.x * a.lpc + line);
  const double* beta = a.beta ? a.beta + (int64_t)b * a.p : nullptr;
  double* out = a.out + (int64_t)b * a.out_bstride;
  const double* gb = a.g ? a.g + (int64_t)b * a.g_bstride : nullptr;
  for (int e = tl; e < 2 * a.ncols; e += nthr) {
    const int which = e >= a.ncols;
    const int x = e - which * a.ncols;
    const int y = ya + which;
    if (y >= a.nrows) continue;
    const double2 z = buf[a.col0 + x];
    double v = which ? z.y : z.x;
    if (a.epi == EPI_SCALAR) {
      v = v + beta[0];
    } else if (a.epi == EPI_COV) {
      const double* xr = a.xg + ((int64_t)y * a.ncols + x) * a.p;
      double fx = 0.0;
      for (int q = 0; q < a.p; ++q) fx = fma(xr[q], beta[q], fx);
      v = v + fx;
    }
    if (gb) v = gb[(int64_t)(a.g_row0 + y) * a.g_ld + a.g_col0 + x] - v;
    out[(int64_t)y * a.ldo + x] = v;
  }
}

// ----------------------------------------------------------------- launches
static Status launch_row_fwd(int src, const RowFwdArgs& a0, int batch, cudaStream_t st) {
  RowFwdArgs a = a0;
  const int pairs = (a.nrows + 1) / 2;
  const dim3 grid((unsigned)ceil_div(pairs, a.lpc), (unsigned)batch);
  const size_t smem = sizeof(double2) * a.pl.n * a.lpc;
  const int threads = a.lpc * a.pl.nthr;
  if (src == SRC_GATHER) {
    RK_TRY(set_smem_attr((const void*)row_fwd_kernel<SRC_GATHER>, smem));
    row_fwd_kernel<SRC_GATHER><<<grid, threads, smem, st>>>(a);
  } else if (src == SRC_REAL) {
    RK_TRY(set_smem_attr((const void*)row_fwd_kernel<SRC_REAL>, smem));
    row_fwd_kernel<SRC_REAL><<<grid, threads, smem, st>>>(a);
  } else {
    RK_TRY(set_smem_attr((const void*)row_fwd_kernel<SRC_LAG>, smem));
    row_fwd_kernel<SRC_LAG><<<grid, threads, smem, st>>>(a);
  }
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

static Status launch_col(int mode, const ColArgs& a, int batch, cudaStream_t st) {
  const dim3 grid((unsigned)ceil_div(a.ncols, a.lpc), (unsigned)batch);
  const size_t smem = sizeof(double2) * a.pl.n * a.lpc;
  const int threads = a.lpc * a.pl.nthr;
  if (mode == 0) {
    RK_TRY(set_smem_attr((const void*)col_kernel<0>, smem));
    col_kernel<0><<<grid, threads, smem, st>>>(a);
  } else {
    RK_TRY(set_smem_attr((const void*)col_kernel<1>, smem));
    col_kernel<1><<<grid, threads, smem, st>>>(a);
  }
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

static Status launch_row_inv(const RowInvArgs& a, int batch, cudaStream_t st) {
  const int pairs = (a.nrows + 1) / 2;
  const dim3 grid((unsigned)ceil_div(pairs, a.lpc), (unsigned)batch);
  const size_t smem = sizeof(double2) * a.pl.n * a.lpc;
  RK_TRY(set_smem_attr((const void*)row_inv_kernel, smem));
  row_inv_kernel<<<grid, a.lpc * a.pl.nthr, smem, st>>>(a);
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

__global__ void lagq_kernel(MaternDev P, double hx, double hy, int H1, int Q2, double* out, int* bad) {
  const int64_t tot = (int64_t)H1 * Q2;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int a = (int)(e / H1), bcol = (int)(e % H1);
    // rapid.py:62-69: min(i, p - i) * h per axis, then hypot
    const double d = hypot((double)bcol * hx, (double)a * hy);
    out[e] = matern_cov(P, d, bad);
  }
}

// Re(fft2(lag filter))[ky, kx] * scale for kx <= p1/2, ky <= p2/2, stored out_q[kx * Q2 + ky]
Status spectrum_quarter(const MaternDev& P, double hx, double hy, int p1, int p2, double scale,
                        double* out_q, cudaStream_t st) {
  FftPlan pl1, pl2;
  RK_TRY(plan_for(p1, &pl1));
  RK_TRY(plan_for(p2, &pl2));
  const int H1 = p1 / 2 + 1, Q2 = p2 / 2 + 1;
  double* lagq = nullptr;
  double2* T = nullptr;
  int* bad = nullptr;
  RK_TRY(scratch_alloc((void**)&lagq, sizeof(double) * (size_t)H1 * Q2, st));
  RK_TRY(scratch_alloc((void**)&T, sizeof(double2) * (size_t)H1 * p2, st));
  RK_TRY(scratch_alloc((void**)&bad, sizeof(int), st));
  RK_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
  lagq_kernel<<<(int)std::min<int64_t>(ceil_div((int64_t)H1 * Q2, 256), 148 * 64), 256, 0, st>>>(
      P, hx, hy, H1, Q2, lagq, bad);
  count_launch();
  RK_LAUNCH_CHECK();
  RowFwdArgs ra{};
  ra.pl = pl1;
  ra.lpc = pick_lpc(pl1, 4);
  ra.nrows = p2;
  ra.ncols = p1;
  ra.T = T;
  ra.ldT = p2;
  ra.T_bstride = 0;
  ra.lagq = lagq;
  ra.lag_ld = H1;
  ra.p2 = p2;
  RK_TRY(launch_row_fwd(SRC_LAG, ra, 1, st));
  ColArgs ca{};
  ca.pl = pl2;
  ca.lpc = pick_lpc(pl2, 4);
  ca.ncols = H1;
  ca.nin = p2;
  ca.T = T;
  ca.ldT = p2;
  ca.Q2 = Q2;
  ca.out_q = out_q;
  ca.scale = scale;
  RK_TRY(launch_col(1, ca, 1, st));
  int hb = 0;
  RK_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
  scratch_free(lagq, st);
  scratch_free(T, st);
  scratch_free(bad, st);
  RK_CUDA_TRY(cudaStreamSynchronize(st));
  if (hb) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");
  return Status::ok();
}

static GatherSrc gather_src(const rk_setup* s, const double* c, int64_t c_stride) {
  GatherSrc g;
  g.cell_start = s->cell_start;
  g.bsort = s->bsort;
  g.perm = s->perm;
  g.wsort = s->wsort;
  g.c = c;
  g.c_stride = c_stride;
  g.M1 = s->M1;
  g.M2 = s->M2;
  g.bs = s->bs;
  g.M = s->M;
  return g;
}

static inline int64_t round_even(int64_t v) { return (v + 1) & ~int64_t(1); }

// Shared 3-pass pipeline. src: SRC_GATHER (coefficients) or SRC_REAL (padded field).
static Status conv_pipeline(const rk_setup* s, int src, const double* c, int64_t c_stride,
                            const double* real_in, int batch, int row0, int nout, int col0,
                            int ncols, const RowInvArgs& epi, cudaStream_t st,
                            cudaEvent_t* ev = nullptr) {
  const int64_t ldT = round_even(s->M2);
  const int64_t ldU = round_even(nout);
  double2 *T = nullptr, *U = nullptr;
  RK_TRY(scratch_alloc((void**)&T, sizeof(double2) * (size_t)s->H1 * ldT * batch, st));
  RK_TRY(scratch_alloc((void**)&U, sizeof(double2) * (size_t)s->H1 * ldU * batch, st));
  RowFwdArgs ra{};
  ra.pl = s->pl1;
  ra.lpc = pick_lpc(s->pl1, 4);
  ra.nrows = s->M2;
  ra.ncols = s->M1;
  ra.T = T;
  ra.ldT = ldT;
  ra.T_bstride = (int64_t)s->H1 * ldT;
  ra.g = gather_src(s, c, c_stride);
  ra.real_in = real_in;
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[0], st));
  RK_TRY(launch_row_fwd(src, ra, batch, st));
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[1], st));
  ColArgs ca{};
  ca.pl = s->pl2;
  ca.lpc = pick_lpc(s->pl2, 4);
  ca.ncols = s->H1;
  ca.nin = s->M2;
  ca.T = T;
  ca.ldT = ldT;
  ca.T_bstride = ra.T_bstride;
  ca.spec_q = s->spec_q;
  ca.Q2 = s->Q2;
  ca.row0 = row0;
  ca.nout = nout;
  ca.U = U;
  ca.ldU = ldU;
  ca.U_bstride = (int64_t)s->H1 * ldU;
  RK_TRY(launch_col(0, ca, batch, st));
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[2], st));
  RowInvArgs ia = epi;
  ia.pl = s->pl1;
  ia.lpc = pick_lpc(s->pl1, 4);
  ia.nrows = nout;
  ia.U = U;
  ia.ldU = ldU;
  ia.U_bstride = ca.U_bstride;
  ia.col0 = col0;
  ia.ncols = ncols;
  RK_TRY(launch_row_inv(ia, batch, st));
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[3], st));
  scratch_free(T, st);
  scratch_free(U, st);
  return Status::ok();
}

Status predict_batch(const rk_setup* s, const PredictBatch& pb, cudaStream_t st, cudaEvent_t* ev) {
  RowInvArgs e{};
  e.out = pb.out;
  e.ldo = s->m1;
  e.out_bstride = (int64_t)s->m1 * s->m2;
  e.epi = pb.beta == nullptr ? EPI_PLAIN : (pb.xg == nullptr ? EPI_SCALAR : EPI_COV);
  e.beta = pb.beta;
  e.p = pb.p;
  e.xg = pb.xg;
  e.g = pb.g;
  e.g_bstride = (int64_t)s->M1 * s->M2;
  e.g_ld = s->M1;
  e.g_row0 = s->grid.pad[2];
  e.g_col0 = s->grid.pad[0];
  return conv_pipeline(s, SRC_GATHER, pb.c, pb.c_stride, nullptr, pb.batch, s->grid.pad[2], s->m2,
                       s->grid.pad[0], s->m1, e, st, ev);
}

}  // namespace rk

using namespace rk;

static int finish_status(const Status& s) {
  if (!s.good()) rk::set_error(s.code, s.msg);
  return s.code;
}

extern "C" {

rk_status rk_coefficients_to_grid(const rk_setup* s, const double* c_dev, double* cstar_dev,
                                  void* stream) {
  auto run = [&]() -> Status {
    GatherSrc g = gather_src(s, c_dev, 0);
    const int64_t tot = (int64_t)s->M1 * s->M2;
    cstar_kernel<<<(int)std::min<int64_t>(ceil_div(tot, 256), 148 * 16), 256, 0,
                   (cudaStream_t)stream>>>(g, cstar_dev);
    count_launch();
    RK_LAUNCH_CHECK();
    return Status::ok();
  };
  return (rk_status)finish_status(run());
}

rk_status rk_convolve_filter(const rk_setup* s, const double* values_dev, double* out_dev,
                             void* stream) {
  auto run = [&]() -> Status {
    RowInvArgs e{};
    e.out = out_dev;
    e.ldo = s->M1;
    e.epi = EPI_PLAIN;
    return conv_pipeline(s, SRC_REAL, nullptr, 0, values_dev, 1, 0, s->M2, 0, s->M1, e,
                         (cudaStream_t)stream);
  };
  return (rk_status)finish_status(run());
}

rk_status rk_convolve_spectrum(const double* spec_q_dev, int32_t p1, int32_t p2,
                               const double* values_dev, int32_t M1, int32_t M2, double* out_dev,
                               void* stream) {
  auto run = [&]() -> Status {
    if (p1 < 2 * M1 - 2 || p2 < 2 * M2 - 2)
      return Status::err(RK_DOMAIN, "embedding dims too small for the padded grid");
    rk_setup t;   // descriptor only: the pipeline reads plans, dims and the spectrum
    t.M1 = M1;
    t.M2 = M2;
    t.p1 = p1;
    t.p2 = p2;
    t.H1 = p1 / 2 + 1;
    t.Q2 = p2 / 2 + 1;
    t.spec_q = const_cast<double*>(spec_q_dev);
    RK_TRY(plan_for(p1, &t.pl1));
    RK_TRY(plan_for(p2, &t.pl2));
    RowInvArgs e{};
    e.out = out_dev;
    e.ldo = M1;
    e.epi = EPI_PLAIN;
    Status st = conv_pipeline(&t, SRC_REAL, nullptr, 0, values_dev, 1, 0, M2, 0, M1, e,
                              (cudaStream_t)stream);
    t.spec_q = nullptr;
    return st;
  };
  return (rk_status)finish_status(run());
}

rk_status rk_predict_dev(const rk_setup* s, const double* c_dev, const double* beta_dev, int32_t p,
                         const double* xg_dev, double* out_dev, void* stream) {
  auto run = [&]() -> Status {
    if (beta_dev && !xg_dev && p != 1)
      return Status::err(RK_DOMAIN, "grid covariates are required when beta_hat has more than one entry");
    PredictBatch pb;
    pb.batch = 1;
    pb.c = c_dev;
    pb.c_stride = s->n;
    pb.beta = beta_dev;
    pb.p = p;
    pb.xg = xg_dev;
    pb.out = out_dev;
    return predict_batch(s, pb, (cudaStream_t)stream);
  };
  return (rk_status)finish_status(run());
}

rk_status rk_predict_profile(const rk_setup* s, const double* c_dev, const double* beta_dev,
                             int32_t p, const double* xg_dev, double* out_dev, void* stream,
                             float* ms_out) {
  auto run = [&]() -> Status {
    cudaStream_t st = (cudaStream_t)stream;
    cudaEvent_t ev[4];
    for (int i = 0; i < 4; ++i) RK_CUDA_TRY(cudaEventCreate(&ev[i]));
    PredictBatch pb;
    pb.batch = 1;
    pb.c = c_dev;
    pb.c_stride = s->n;
    pb.beta = beta_dev;
    pb.p = p;
    pb.xg = xg_dev;
    pb.out = out_dev;
    Status r = predict_batch(s, pb, st, ev);
    if (r.good()) {
      RK_CUDA_TRY(cudaEventSynchronize(ev[3]));
      for (int i = 0; i < 3; ++i) RK_CUDA_TRY(cudaEventElapsedTime(&ms_out[i], ev[i], ev[i + 1]));
    }
    for (int i = 0; i < 4; ++i) cudaEventDestroy(ev[i]);
    return r;
  };
  return (rk_status)finish_status(run());
}

rk_status rk_predict_traffic(const rk_setup* s, int32_t p, double* b) {
  // pass 1: weights (n M), sorted base/perm (8 n), c gathers (8 n), cell_start (4 (G + 1)),
  //         T write (16 H1 M2); pass 2: T read, quarter spectrum (8 H1 Q2), U write (16 H1 m2);
  // pass 3: U read, covariates (8 N p), field write (8 N)
  const double n = (double)s->n, M = (double)s->M, G = (double)s->M1 * s->M2;
  const double N = (double)s->m1 * s->m2, H = (double)s->H1;
  b[0] = n * M * 8.0 + 16.0 * n + 4.0 * (G + 1.0) + 16.0 * H * s->M2;
  b[1] = 16.0 * H * s->M2 + 8.0 * H * s->Q2 + 16.0 * H * s->m2;
  b[2] = 16.0 * H * s->m2 + 8.0 * N * (double)p + 8.0 * N;
  return RK_OK;
}

rk_status rk_predict_host(const rk_setup* s, const double* c, const double* beta, int32_t p,
                          const double* xg, double* out, void* stream) {
  auto run = [&]() -> Status {
    cudaStream_t st = (cudaStream_t)stream;
    if (beta && !xg && p != 1)
      return Status::err(RK_DOMAIN, "grid covariates are required when beta_hat has more than one entry");
    const int64_t N = (int64_t)s->m1 * s->m2;
    const size_t bc = sizeof(double) * s->n, bb = beta ? sizeof(double) * p : 0,
                 bx = xg ? sizeof(double) * N * p : 0, bo = sizeof(double) * N;
    char* ws = nullptr;
    RK_TRY(scratch_alloc((void**)&ws, bc + bb + bx + bo + 64, st));
    double* dc = (double*)ws;
    double* db = beta ? (double*)(ws + bc) : nullptr;
    double* dx = xg ? (double*)(ws + bc + bb) : nullptr;
    double* dout = (double*)(ws + bc + bb + bx);
    RK_CUDA_TRY(cudaMemcpyAsync(dc, c, bc, cudaMemcpyHostToDevice, st));
    if (beta) RK_CUDA_TRY(cudaMemcpyAsync(db, beta, bb, cudaMemcpyHostToDevice, st));
    if (xg) RK_CUDA_TRY(cudaMemcpyAsync(dx, xg, bx, cudaMemcpyHostToDevice, st));
    PredictBatch pb;
    pb.batch = 1;
    pb.c = dc;
    pb.c_stride = s->n;
    pb.beta = db;
    pb.p = p;
    pb.xg = dx;
    pb.out = dout;
    RK_TRY(predict_batch(s, pb, st));
    RK_CUDA_TRY(cudaMemcpyAsync(out, dout, bo, cudaMemcpyDeviceToHost, st));
    scratch_free(ws, st);
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    return Status::ok();
  };
  return (rk_status)finish_status(run());
}

}  // extern "C"
