// rapidkrig B200: rapid predict = deterministic scatter + circulant FFT convolution.
//
// Reference mapping (/root/reference/pkg/src/rapidkrig/rapid.py):
//   coefficients_to_grid 164-174 (np.add.at)  -> per-node GATHER from a sparse plan built at
//       setup (fixed order, no atomics): fused into pass 1 for predict, cstar_rows_kernel
//       for the standalone coefficients_to_grid
//   convolve_filter 89-100 (fft2 * spectrum, ifft2, crop) -> 3 passes:
//       pass 1 row_fwd_kernel : two real padded rows (gathered in smem, or TMA bulk-staged) per complex FFT of
//                               length p1, split into two half spectra, written transposed
//                               T[kx][y] (only the M2 nonzero rows exist)
//       pass 2 col_kernel     : column kx (TMA bulk load) -> FFT(p2) -> x real-even spectrum
//                               (quarter column prefetched by TMA during the FFT, 1/(p1 p2)
//                               folded in) -> IFFT -> TMA bulk store of the m2 interior rows
//       pass 3 row_inv_kernel : Hermitian-combined pair of interior rows, IFFT(p1), keep the
//                               m1 interior columns, fused fixed-part / draw epilogue
//   _fixed_part 233-249 / predict_rapid 252-261 -> epilogue of pass 3
//   build_filter_spectrum 72-86 -> spectrum_quarter(): lag table on the quarter torus,
//       pass 1 (lag mode) + pass 2 (spectrum mode, real part of ky <= p2/2)
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include <cooperative_groups.h>

#include "rk_internal.cuh"

namespace cg = cooperative_groups;

namespace rk {
// Per-CTA phase timestamps (%globaltimer, ns) for the three predict kernels, compiled in with
// RK_PHASE_TIMING=1 at build time and read back with rk_phase_timestamps (tools/phase_probe.py).
#ifdef RK_PHASE_TIMING
__device__ unsigned long long g_phase_ts[3 * 4096 * 8];
#define RK_PHASE(k, ph)                                                                       \
  do {                                                                                        \
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x < 4096) {                           \
      unsigned long long t_;                                                                  \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
      g_phase_ts[((k) * 4096 + blockIdx.x) * 8 + (ph)] = t_;                                  \
    }                                                                                         \
  } while (0)
#else
#define RK_PHASE(k, ph) \
  do {                  \
  } while (0)
#endif

// ----------------------------------------------------------------- gather
// Sparse gather plan (built at setup): per padded row, its active nodes in ascending
// order, each with its contributions (index into wsort, original observation index) in the
// fixed order dy asc, sorted j asc -> bitwise reproducible, identical for every batch / stream.
struct SparseSrc {
  const int32_t* node_q;
  const int32_t* node_off;
  const int32_t* row_node;
  const int32_t* ent_w;
  const int32_t* ent_c;
  const double* wsort;
  const double* ent_wv;      // weight per contribution (pass 1: no wsort indirection)
  const int4* pair_info;     // per row pair {node0, node of the odd row, contribution0, contributions
                             // of its first ceil(nodes / 2) nodes}
  const double* c;
  int64_t c_stride;
  int M1;
};

// c*[y, x] for the active nodes of padded row y, written through put(x, value)
template <class Put>
__device__ __forceinline__ void gather_row(const SparseSrc& g, const double* __restrict__ c, int y, int t,
                                           int nt, Put put) {
  const int a0 = __ldg(&g.row_node[y]), a1 = __ldg(&g.row_node[y + 1]);
  const int rowq = y * g.M1;
  for (int a = a0 + t; a < a1; a += nt) {
    const int e0 = __ldg(&g.node_off[a]), e1 = __ldg(&g.node_off[a + 1]);
    double acc = 0.0;
    for (int e = e0; e < e1; ++e) {
      const double w = __ldg(&g.wsort[__ldg(&g.ent_w[e])]);
      const double cj = __ldg(&c[__ldg(&g.ent_c[e])]);
      acc = __dadd_rn(acc, __dmul_rn(w, cj));   // (w * c) then add, as np.add.at
    }
    put(__ldg(&g.node_q[a]) - rowq, acc);
  }
}

// ----------------------------------------------------------------- pass 1
// SRC_SPARSE: the scatter c* = A'c is formed in shared memory from the sparse plan (no c*
// round trip through HBM); SRC_ROWS: dense input rows; SRC_LAG: the quarter lag table.
enum RowSrc { SRC_ROWS = 1, SRC_LAG = 2, SRC_SPARSE = 3 };

struct RowFwdArgs {
  FftPlan pl;
  int lpc;
  int nrows;                 // input rows
  int ncols;                 // nonzero input columns
  double2* T;                // (H, ldT) per batch
  int64_t ldT, T_bstride;
  const double* rows;        // SRC_ROWS: (nrows, ld_in) per batch
  int64_t ld_in, in_bstride;
  int tma;                   // SRC_ROWS: rows are 16-byte aligned -> TMA bulk staging
  const double* lagq;        // SRC_LAG: quarter lag table (p2/2+1, p1/2+1)
  int lag_ld, p2;
  SparseSrc sp;              // SRC_SPARSE: gather plan + coefficients
  int prod_off, prod_cap;    // SRC_SPARSE: smem offset (double2 units) / per-line size (doubles)
                             // of the staged products w * c of the line's row pair
  int c_off, c_n;            // SRC_SPARSE, c_n > 0: the whole coefficient vector (c_n entries)
                             // is bulk-copied to smem at offset c_off (double2 units) up front
  const unsigned char* pblk;  // SRC_SPARSE (one-wave launches): the setup's per-pair plan blocks,
  int64_t pblk_stride;       // fetched per line into smem at pl_off (double2 units)
  int pblk_cap, pl_off;
  int tw_off;                // smem offset (double2 units) of the staged twiddle table
  SplitTw sw;                // split-length kernels: w_P^n tables (staged at sw.off)
};

// FFT kernels: WIDE instantiations run 64-register threads (fft_kmax_wide butterflies each)
#define RK_FFT_BOUNDS(FM) __launch_bounds__((FM) == 1 ? kFftWideThreads : (FM) == 2 ? kFftSplitThreads : 512, 1)

template <int SRC, bool TWS, int FM>   // FM: FFT mode of fft_line (0 normal / spread, 1 WIDE, 2 split)
__global__ void RK_FFT_BOUNDS(FM) row_fwd_kernel(const RowFwdArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  double2* buf = smem + (size_t)line * n;
  const int ya = 2 * (blockIdx.x * a.lpc + line);
  const int yb = ya + 1;
  const bool va = ya < a.nrows, vb = yb < a.nrows;
  RK_PHASE(0, 0);
  const TwPrefetch twp = TWS ? twiddles_prefetch(a.pl) : TwPrefetch{};
  pdl_wait();   // everything below reads the predecessor's output
  if (SRC == SRC_ROWS) {
    const double* rin = a.rows + (int64_t)b * a.in_bstride;
    // staging of the two real rows: tma == 2 puts them in the zero-pad tail of the line
    // buffer itself (no extra smem; needs n - ld_in >= ncols), tma == 1 in a separate area
    const bool inl = a.tma == 2;
    double* extra = (double*)(smem + (size_t)a.lpc * n);
    auto stage_of = [&](int l) -> double* {
      return inl ? (double*)(smem + (size_t)(l + 1) * n) - 2 * a.ld_in : extra + (size_t)l * 2 * a.ld_in;
    };
    uint64_t* bar = inl ? (uint64_t*)extra : (uint64_t*)(extra + (size_t)a.lpc * 2 * a.ld_in);
    const double* sa = stage_of(line);
    const double* sb = sa + a.ld_in;
    if (a.tma) {
      if (threadIdx.x == 0) mbar_init(bar, 1);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t cnt = 0;
        for (int l = 0; l < a.lpc; ++l) {
          const int r0 = 2 * (blockIdx.x * a.lpc + l);
          cnt += (r0 < a.nrows ? 1u : 0u) + (r0 + 1 < a.nrows ? 1u : 0u);
        }
        mbar_expect_tx(bar, cnt * (uint32_t)(a.ld_in * 8));
        for (int l = 0; l < a.lpc; ++l) {
          const int r0 = 2 * (blockIdx.x * a.lpc + l);
          double* d = stage_of(l);
          if (r0 < a.nrows) bulk_g2s(d, rin + (int64_t)r0 * a.ld_in, (uint32_t)(a.ld_in * 8), bar);
          if (r0 + 1 < a.nrows)
            bulk_g2s(d + a.ld_in, rin + (int64_t)(r0 + 1) * a.ld_in, (uint32_t)(a.ld_in * 8), bar);
        }
      }
      // zero padding beyond the nonzero columns while the copies fly (separate staging)
      if (!inl)
        for (int x = a.ncols + tl; x < n; x += nthr) buf[x] = make_double2(0.0, 0.0);
      mbar_wait(bar, 0);
      for (int x = tl; x < a.ncols; x += nthr)
        buf[x] = make_double2(va ? sa[x] : 0.0, vb ? sb[x] : 0.0);
      if (inl) {   // the staging tail is consumed: now zero it
        __syncthreads();
        for (int x = a.ncols + tl; x < n; x += nthr) buf[x] = make_double2(0.0, 0.0);
      }
    } else {
      for (int x = tl; x < n; x += nthr) {
        double u = 0.0, v = 0.0;
        if (x < a.ncols) {
          if (va) u = rin[(int64_t)ya * a.ld_in + x];
          if (vb) v = rin[(int64_t)yb * a.ld_in + x];
        }
        buf[x] = make_double2(u, v);
      }
    }
  } else if (SRC == SRC_SPARSE) {
    // the row pair's contributions are contiguous in the plan.  Three dependent global
    // round trips: the pair record; the node records and contribution (weight, observation)
    // pairs, all in flight together; the coefficients.  Products w * c and node records
    // are staged in shared memory, then each active node adds its own products in the
    // fixed plan order.
    const SparseSrc& g = a.sp;
    const double* __restrict__ cb = g.c + (int64_t)b * g.c_stride;
    double* __restrict__ prod = (double*)(smem + a.prod_off) + (size_t)line * 2 * a.prod_cap;
    int2* __restrict__ nrec = (int2*)(prod + a.prod_cap);
    const int pidx = blockIdx.x * a.lpc + line;
    // the coefficients travel by one TMA bulk copy issued before the plan is read, so the
    // per-contribution lookups c[j] hit shared memory: two dependent global round trips
    // (pair record, plan entries) instead of three
    const double* __restrict__ cl = cb;
    uint64_t* cbar = nullptr;
    if (a.c_n > 0) {
      double* cs = (double*)(smem + a.c_off);
      cbar = (uint64_t*)(cs + ((a.c_n + 1) & ~1));
      if (threadIdx.x == 0) {
        const uint32_t b16 = (uint32_t)(a.c_n * 8) & ~15u;
        mbar_init(cbar, 1);
        mbar_expect_tx(cbar, b16);
        if (b16) bulk_g2s(cs, cb, b16, cbar);
        if (a.c_n & 1) cs[a.c_n - 1] = __ldg(&cb[a.c_n - 1]);
      }
      cl = cs;
      __syncthreads();   // barrier initialised before anyone waits on it
    }
    for (int x = tl; x < n; x += nthr) buf[x] = make_double2(0.0, 0.0);
    bool cwait = cbar != nullptr;
    int nn = 0;
    const int2* nrp = nrec;   // the node records the sums below read
    if (FM != 1 && a.pblk) {
      // one-wave launches: the pair's whole plan (counts, node records, weights, observation
      // indices) is one fixed-stride block fetched by ONE bulk copy -- a single global round
      // trip for any pair size, where the most loaded pair of a clustered design otherwise
      // takes a dependent round trip per 4 * nthr contributions and sets the pass's end
      unsigned char* blk = reinterpret_cast<unsigned char*>(smem + a.pl_off) + (size_t)line * (a.pblk_stride + 16);
      uint64_t* pbar = reinterpret_cast<uint64_t*>(blk + a.pblk_stride);
      if (tl == 0) mbar_init(pbar, 1);
      __syncthreads();
      if (tl == 0) {
        mbar_expect_tx(pbar, va ? (uint32_t)a.pblk_stride : 0u);
        if (va) bulk_g2s(blk, a.pblk + (int64_t)pidx * a.pblk_stride, (uint32_t)a.pblk_stride, pbar);
      }
      mbar_wait(pbar, 0);
      const int cnt = va ? reinterpret_cast<const int*>(blk)[0] : 0;
      nn = va ? reinterpret_cast<const int*>(blk)[1] : 0;
      nrp = reinterpret_cast<const int2*>(blk + 16);
      const double* wv = reinterpret_cast<const double*>(blk + 16 + (size_t)a.pblk_cap * 8);
      const int* ci = reinterpret_cast<const int*>(blk + 16 + (size_t)a.pblk_cap * 16);
      if (cwait) {
        mbar_wait(cbar, 0);
        cwait = false;
      }
      for (int i = tl; i < cnt; i += nthr) prod[i] = __dmul_rn(wv[i], cl[ci[i]]);
    } else {
      int4 P0 = make_int4(0, 0, 0, 0), P1 = P0;
      if (va) {
        P0 = __ldg(&g.pair_info[pidx]);
        P1 = __ldg(&g.pair_info[pidx + 1]);
      }
      const int n0 = P0.x, n1 = P0.y, e0 = P0.z;
      nn = P1.x - n0;
      const int cnt = P1.z - e0;
      const int rowq = ya * g.M1;
      // one pass issues the contribution loads and the node-record loads together; only the
      // coefficient loads depend on them
      constexpr int U = 4;
      const int m = max(cnt, nn);
      for (int i0 = tl; i0 < m; i0 += U * nthr) {
        double w[U];
        int ci[U], nq[U], ne[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * nthr;
          w[u] = i < cnt ? __ldg(&g.ent_wv[e0 + i]) : 0.0;
          ci[u] = i < cnt ? __ldg(&g.ent_c[e0 + i]) : 0;
          nq[u] = i < nn ? __ldg(&g.node_q[n0 + i]) : 0;
          ne[u] = i < nn ? __ldg(&g.node_off[n0 + i + 1]) : 0;
        }
        if (cwait) {   // first use: the bulk copy (init ordered by the barrier above) has landed
          mbar_wait(cbar, 0);
          cwait = false;
        }
        double cv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) cv[u] = i0 + u * nthr < cnt ? cl[ci[u]] : 0.0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = i0 + u * nthr;
          if (i < cnt) prod[i] = __dmul_rn(w[u], cv[u]);
          if (i < nn) {   // node i: end of its products, its x | odd-row bit
            const int odd = n0 + i >= n1;
            nrec[i] = make_int2(ne[u] - e0, 2 * (nq[u] - rowq - odd * g.M1) + odd);
          }
        }
      }
    }
    if (cwait) mbar_wait(cbar, 0);   // no contributions here: still retire the copy before exit
    __syncthreads();
    RK_PHASE(0, 1);
    double* bd = (double*)buf;
    for (int k = tl; k < nn; k += nthr) {
      const int s0 = k ? nrp[k - 1].x : 0;
      const int2 r = nrp[k];
      double acc = 0.0;
      for (int i = s0; i < r.x; ++i) acc = __dadd_rn(acc, prod[i]);   // (w * c) then add, as np.add.at
      bd[r.y] = acc;
    }
  } else {
    for (int x = tl; x < n; x += nthr) {
      const int bx = min(x, n - x);
      const double u = va ? __ldg(&a.lagq[(int64_t)min(ya, a.p2 - ya) * a.lag_ld + bx]) : 0.0;
      const double v = vb ? __ldg(&a.lagq[(int64_t)min(yb, a.p2 - yb) * a.lag_ld + bx]) : 0.0;
      buf[x] = make_double2(u, v);
    }
  }
  const FftPlan pls = TWS ? twiddles_commit(a.pl, twp, smem + a.tw_off) : a.pl;
  __syncthreads();
  RK_PHASE(0, 2);
  fft_line<false, TWS, FM, true, FM == 1 ? 3 : 0>(buf, pls, tl, a.lpc > 1 ? 1 + line : 0);
  if (a.lpc > 1) __syncthreads();   // the split below reads every line
  RK_PHASE(0, 3);
  pdl_trigger();   // the column pass may start staging while the split rows are stored
  // split Z = FFT(u + i v) into U = (Z + conj Z[-k]) / 2, V = (Z - conj Z[-k]) / 2i
  const int nr = 2 * a.lpc;
  const int H = n / 2 + 1;
  double2* T = a.T + (int64_t)b * a.T_bstride;
  if (aligned32(T, a.ldT)) {   // both rows of a pair in one 32-byte store (one thread per (kx, pair))
    for (int idx = threadIdx.x; idx < H * a.lpc; idx += blockDim.x) {
      const int l = idx % a.lpc, kx = idx / a.lpc;
      const int row = 2 * (blockIdx.x * a.lpc + l);
      if (row >= a.nrows) continue;
      const double2* bl = smem + (size_t)l * n;
      const double2 z = bl[kx];
      const double2 zc = bl[kx == 0 ? 0 : n - kx];
      const double2 o0 = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
      const double2 o1 = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
      double2* dst = T + (int64_t)kx * a.ldT + row;
      if (row + 1 < a.nrows) stg256(dst, o0, o1);
      else dst[0] = o0;
    }
  } else {
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
  RK_PHASE(0, 4);
}

// ----------------------------------------------------------------- pass 2
struct ColArgs {
  FftPlan pl;
  int lpc;
  int ncols;                 // number of columns (kx)
  int nin;                   // nonzero input rows
  const double2* T;
  int64_t ldT, T_bstride;
  const double* spec_q;      // filter mode: (ncols, ldq)
  int ldq;                   // even, >= p2/2 + 1
  int row0, nout;            // filter mode: keep rows [row0, row0 + nout)
  double2* U;
  int64_t ldU, U_bstride;
  double* out_q;             // spectrum mode: out_q[kx * ldq + ky] = Re * scale, ky <= p2/2
  double scale;
  int tw_off;                // smem offset (double2 units) of the staged twiddle table
  SplitTw sw;                // split-length kernel: w_P^n tables
  const double* spec_s;      // split-length kernel: parity-split spectrum (ncols, 2, ldh)
  int ldh;
  int upair;                 // split-length kernel: write U pair-blocked (see UPair)
  int64_t ldp;
  int hh;
  int x_off;                 // col_pair_kernel: smem offset (double2 units) of its 2 mbarriers
  int batch;                 // col_pair_kernel: fields per launch (persistent over columns x batch)
  int fold;                  // col_split_kernel: input rows beyond the half (nin - H > 0: execution
                             // torus), folded into the half transforms' inputs
  int fuse_pp;               // col_split_kernel: twist / spectrum product fused into the first /
                             // last forward stage (fft_line_pp; RK_FUSE_PP=0 keeps the passes)
  CtPlan ct;                 // col_split_ct_kernel: in-place Cooley-Tukey plan of the half length
  int ct_off;                // smem offset (double2 units) where its twiddles are staged
};

// FAM 1 (WIDE filter mode only): lines 6 9^a with the other stage bodies compiled out (fft_line FAM)
template <int MODE, bool TWS, int FM, int FAM = 0>  // MODE 0 = filter (fwd, x spectrum, inv, crop), 1 = spectrum (fwd, real part)
__global__ void RK_FFT_BOUNDS(FM) col_kernel(const ColArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  const int kx = blockIdx.x * a.lpc + line;
  const bool valid = kx < a.ncols;
  double2* buf = smem + (size_t)line * n;
  double* specs = (double*)(smem + (size_t)a.lpc * n);          // lpc x ldq (filter mode)
  uint64_t* bar = (uint64_t*)(specs + (MODE == 0 ? (size_t)a.lpc * a.ldq : 0));
  const double2* Tb = a.T + (int64_t)b * a.T_bstride;
  RK_PHASE(1, 0);
  if (threadIdx.x == 0) mbar_init(bar, 1);
  __syncthreads();
  const uint32_t colb = (uint32_t)a.nin * 16u;
  if (threadIdx.x == 0) {
    int nv = 0;
    for (int l = 0; l < a.lpc; ++l) nv += (blockIdx.x * a.lpc + l) < a.ncols;
    const uint32_t specb = MODE == 0 ? (uint32_t)a.ldq * 8u : 0u;
    mbar_expect_tx(bar, (uint32_t)nv * (colb + specb));
    if (MODE == 0)
      for (int l = 0; l < a.lpc; ++l) {
        const int k = blockIdx.x * a.lpc + l;
        if (k < a.ncols) bulk_g2s(specs + (size_t)l * a.ldq, a.spec_q + (int64_t)k * a.ldq, specb, bar);
      }
  }
  pdl_wait();   // T is the predecessor's output
  if (threadIdx.x == 0)
    for (int l = 0; l < a.lpc; ++l) {
      const int k = blockIdx.x * a.lpc + l;
      if (k < a.ncols) bulk_g2s(smem + (size_t)l * n, Tb + (int64_t)k * a.ldT, colb, bar);
    }
  const FftPlan pls = TWS ? fft_twiddles_to_smem(a.pl, smem + a.tw_off) : a.pl;
  for (int y = a.nin + tl; y < n; y += nthr) buf[y] = make_double2(0.0, 0.0);
  if (!valid)
    for (int y = tl; y < a.nin; y += nthr) buf[y] = make_double2(0.0, 0.0);
  mbar_wait(bar, 0);
  __syncthreads();
  RK_PHASE(1, 1);
  fft_line<false, TWS, FM, true, FM == 1 ? 3 : 0, FAM>(buf, pls, tl, a.lpc > 1 ? 1 + line : 0);
  RK_PHASE(1, 2);
  if (MODE == 0) {
    const double* S = specs + (size_t)line * a.ldq;
    for (int ky = tl; ky < n; ky += nthr) buf[ky] = cscale(buf[ky], valid ? S[min(ky, n - ky)] : 0.0);
    group_sync(a.lpc > 1 ? 1 + line : 0, nthr);
    fft_line<true, TWS, FM, true, FM == 1 ? 3 : 0, FAM>(buf, pls, tl, a.lpc > 1 ? 1 + line : 0);
    RK_PHASE(1, 3);
    pdl_trigger();
    // TMA bulk store of the kept rows
    fence_async_smem();
    __syncthreads();
    if (threadIdx.x == 0) {
      for (int l = 0; l < a.lpc; ++l) {
        const int k = blockIdx.x * a.lpc + l;
        if (k >= a.ncols) continue;
        bulk_s2g(a.U + (int64_t)b * a.U_bstride + (int64_t)k * a.ldU, smem + (size_t)l * n + a.row0,
                 (uint32_t)a.nout * 16u);
      }
      bulk_commit();
      bulk_wait_read0();
    }
    __syncthreads();
    RK_PHASE(1, 4);
  } else {
    if (valid)
      for (int ky = tl; ky <= n / 2; ky += nthr) a.out_q[(int64_t)kx * a.ldq + ky] = buf[ky].x * a.scale;
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
  int tw_off;                // smem offset (double2 units) of the staged twiddle table
  int ep_off;                // smem offset (double2 units) of the prefetched epilogue operands
  int ep_smem;               // 1: epilogue operands prefetched to smem, 0: read from global
  int xg_bulk;               // X_g is 16-byte aligned: one TMA bulk copy per CTA
  SplitTw sw;                // split-length kernel: w_P^n tables
  int upair;                 // split-length kernel: U is pair-blocked (see UPair)
  int64_t ldp;
  int hh;
  // aliased-lag corrections of the execution torus (AliasCorr): corr[b][pair][x], added to the
  // convolution of interior row ac_row0 + y for the pairs whose output row it is
  const double* ac_corr;
  int64_t ac_cbs;
  int ac_row0;
  AliasCorr ac;
};

__device__ __forceinline__ double ac_row_corr(const RowInvArgs& a, int b, int y, int x) {
  double v = 0.0;
  const int yi = a.ac_row0 + y;
  if (yi < a.ac.row_lo || yi >= a.ac.row_hi)
    for (int k = 0; k < a.ac.nrp; ++k)
      if (a.ac.rp_out[k] == yi) v += a.ac_corr[(int64_t)b * a.ac_cbs + (int64_t)k * a.ncols + x];
  return v;
}

template <bool TWS, int FM>
__global__ void RK_FFT_BOUNDS(FM) row_inv_kernel(const RowInvArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int n = a.pl.n;
  const int nthr = a.pl.nthr;
  const int line = threadIdx.x / nthr;
  const int tl = threadIdx.x - line * nthr;
  const int b = blockIdx.y;
  const int H = n / 2 + 1;
  const double2* U = a.U + (int64_t)b * a.U_bstride;
  RK_PHASE(2, 0);
  const TwPrefetch twp = TWS ? twiddles_prefetch(a.pl) : TwPrefetch{};
  // prefetch the epilogue operands of the CTA's rows (covariates X_g: one contiguous block,
  // a TMA bulk copy; CS field g: strided rows, 8-byte async copies); they land while the U
  // rows are gathered and transformed
  const int pc = a.epi == EPI_COV ? a.p : 0;
  const int hasg = a.g ? 1 : 0;
  const int y0 = 2 * blockIdx.x * a.lpc;
  const int nr = min(2 * a.lpc, a.nrows - y0);
  double* epx = (double*)(smem + a.ep_off);                    // (2 lpc, ncols, pc)
  double* epg = epx + (size_t)2 * a.lpc * a.ncols * pc;        // (2 lpc, ncols)
  uint64_t* bar = (uint64_t*)(epg + (size_t)2 * a.lpc * a.ncols * hasg);
  const double* gb = a.g ? a.g + (int64_t)b * a.g_bstride : nullptr;
  bool xwait = false;
  if (a.ep_smem && pc) {
    const double* src = a.xg + (int64_t)y0 * a.ncols * pc;
    const int cnt = nr * a.ncols * pc;
    if (a.xg_bulk) {
      const uint32_t b16 = (uint32_t)(cnt * 8) & ~15u;
      xwait = b16 > 0;
      if (threadIdx.x == 0) {
        if (xwait) {
          mbar_init(bar, 1);
          mbar_expect_tx(bar, b16);
          bulk_g2s(epx, src, b16, bar);
        }
        if (b16 != (uint32_t)cnt * 8) epx[cnt - 1] = __ldg(&src[cnt - 1]);   // odd tail
      }
    } else {
      for (int e = threadIdx.x; e < cnt; e += blockDim.x) cp_async8(epx + e, src + e);
    }
  }
  if (a.ep_smem && hasg) {
    for (int e = threadIdx.x; e < nr * a.ncols; e += blockDim.x) {
      const int r = e / a.ncols, x = e - r * a.ncols;
      cp_async8(epg + e, gb + (int64_t)(a.g_row0 + y0 + r) * a.g_ld + a.g_col0 + x);
    }
  }
  pdl_wait();   // U is the predecessor's output
  // strided gather of both rows of every line (Z[k] = A[k] + i B[k], Hermitian upper half),
  // batched 5 deep per thread for memory-level parallelism (5 x 512 threads cover a 4374-point
  // line's 2188 entries in one round trip; 8 deep spilled the 64-register kernels)
  const int tot = a.lpc * H;
  constexpr int D = 5;
  const bool al32 = aligned32(U, a.ldU);   // row pairs start at even rows
  for (int base = threadIdx.x; base < tot; base += D * blockDim.x) {
    double2 A[D], B[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int idx = base + d * blockDim.x;
      A[d] = B[d] = make_double2(0.0, 0.0);
      if (idx < tot) {
        const int l = idx % a.lpc, k = idx / a.lpc;
        const int ya = 2 * (blockIdx.x * a.lpc + l);
        const double2* u = U + (int64_t)k * a.ldU + ya;
        if (ya + 1 < a.nrows && al32) {
          ldg256(u, A[d], B[d]);   // both rows' entries in one 32-byte request
        } else {
          if (ya < a.nrows) A[d] = u[0];
          if (ya + 1 < a.nrows) B[d] = u[1];
        }
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int idx = base + d * blockDim.x;
      if (idx < tot) {
        const int l = idx % a.lpc, k = idx / a.lpc;
        double2* bl = smem + (size_t)l * n;
        bl[k] = make_double2(A[d].x - B[d].y, A[d].y + B[d].x);
        if (k >= 1 && k <= n - H) bl[n - k] = make_double2(A[d].x + B[d].y, B[d].x - A[d].y);
      }
    }
  }
  RK_PHASE(2, 1);
  const FftPlan pls = TWS ? twiddles_commit(a.pl, twp, smem + a.tw_off) : a.pl;
  cp_async_wait_all();
  __syncthreads();
  RK_PHASE(2, 2);
  double2* buf = smem + (size_t)line * n;
  fft_line<true, TWS, FM, true, FM == 1 ? 1 : 0>(buf, pls, tl, a.lpc > 1 ? 1 + line : 0);
  if (xwait) mbar_wait(bar, 0);   // init is ordered by the barrier above
  RK_PHASE(2, 3);
  const int ya = 2 * (blockIdx.x * a.lpc + line);
  const double* beta = a.beta ? a.beta + (int64_t)b * a.p : nullptr;
  double* out = a.out + (int64_t)b * a.out_bstride;
  for (int e = tl; e < 2 * a.ncols; e += nthr) {
    const int which = e >= a.ncols;
    const int x = e - which * a.ncols;
    const int y = ya + which;
    if (y >= a.nrows) continue;
    const double2 z = buf[a.col0 + x];
    double v = which ? z.y : z.x;
    if (a.ac_corr) v += ac_row_corr(a, b, y, x);
    const int lr = 2 * line + which;
    if (a.epi == EPI_SCALAR) {
      v = v + beta[0];
    } else if (a.epi == EPI_COV) {
      const double* xr = a.ep_smem ? epx + ((size_t)lr * a.ncols + x) * pc : a.xg + ((int64_t)y * a.ncols + x) * pc;
      double fx = 0.0;
      for (int q = 0; q < pc; ++q) fx = fma(xr[q], beta[q], fx);
      v = v + fx;
    }
    if (gb) v = (a.ep_smem ? epg[lr * a.ncols + x] : gb[(int64_t)(a.g_row0 + y) * a.g_ld + a.g_col0 + x]) - v;
    out[(int64_t)y * a.ldo + x] = v;
  }
  RK_PHASE(2, 4);
}

// ----------------------------------------------------------------- split-length passes
// For a transform length P = 2H whose input is zero beyond H (the M nonzero rows / columns of
// the padded grid: P >= 2M - 1 and P even give M <= H) and whose kept outputs lie below H (the
// interior), one length-P transform is two independent length-H transforms:
//   X[2m] = F_H(x)[m],  X[2m+1] = F_H(x w_P^n)[m]                     (forward, x[n >= H] = 0)
//   y[n]  = F_H^-1(Y_e)[n] + w_P^-n F_H^-1(Y_o)[n],  n < H            (inverse, Y_e[m] = Y[2m])
// (w_P = exp(-2 pi i / P), transforms unnormalised).  For the large tori (8748 = 2 x 4374) the
// half length has a WIDE plan (64-register kernels, 1024 FFT threads per SM) and a twiddle
// table that fits in shared memory next to the lines; the full length has neither.  The
// w_P^n factors come from two staged tables, w_P^n = hi[n / 128] lo[n % 128] (one complex
// product), built on the host in long double.

// One CTA per half line (two CTAs per SM: ~86-111 KB of shared memory each, so one CTA's
// global phases overlap the other's transform).  Pass 1 needs no exchange (each half yields the
// outputs kx of its parity); passes 2 and 3 pair the two halves of a line in a 2-CTA cluster and
// combine them through distributed shared memory.
constexpr int kSplitThreads = 512;   // the WIDE plan's threads per half line (n <= 4608)

// pass 1, sparse gather: row pair -> this CTA's half line -> T rows kx with kx % 2 == half.
// The pair's two CTAs (a 2-CTA cluster) split the gather by nodes: each forms the sums of half
// the pair's active nodes and writes them into both half lines (its own and, over DSMEM, its
// partner's); the odd half then twists its copy by w_P^x.
template <bool LEAN>   // LEAN: a line 6 9^a with the other stage bodies compiled out (fft_line FAM)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kSplitThreads, 2) row_fwd_split_kernel(const RowFwdArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int half = (int)cl.block_rank();
  const int H = a.pl.n;
  const int nthr = a.pl.nthr;
  const int tl = threadIdx.x;
  const int pidx = blockIdx.x >> 1;
  const int b = blockIdx.y;
  double2* buf = smem;
  double* bo_remote = (double*)cl.map_shared_rank(buf, half ^ 1);
  const int ya = 2 * pidx;
  const bool va = ya < a.nrows;
  const FftPlan pls = fft_twiddles_to_smem(a.pl, smem + a.tw_off);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  pdl_wait();
  const SparseSrc& g = a.sp;
  const double* __restrict__ cb = g.c + (int64_t)b * g.c_stride;
  double* __restrict__ prod = (double*)(smem + a.prod_off);
  int2* __restrict__ nrec = (int2*)(prod + a.prod_cap);
  for (int x = tl; x < H; x += nthr) buf[x] = make_double2(0.0, 0.0);
  int4 P0 = make_int4(0, 0, 0, 0), P1 = P0;
  if (va) {
    P0 = __ldg(&g.pair_info[pidx]);
    P1 = __ldg(&g.pair_info[pidx + 1]);
  }
  const int n0 = P0.x, n1 = P0.y, e0 = P0.z;
  const int nn = P1.x - n0;
  // this CTA's nodes [kA, kB) and their contributions [eA, eB) (relative to e0); the split
  // point's contribution offset comes with the pair record (no dependent node_off round trip)
  const int kA = half ? (nn + 1) / 2 : 0, kB = half ? nn : (nn + 1) / 2;
  const int eA = half ? P0.w : 0;
  const int eB = half ? P1.z - e0 : P0.w;
  const int cnt = max(eB - eA, 0), nk = kB - kA;
  const int rowq = ya * g.M1;
  constexpr int U = 4;
  const int m = max(cnt, nk);
  for (int i0 = tl; i0 < m; i0 += U * nthr) {
    double w[U];
    int ci[U], nq[U], ne[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nthr;
      w[u] = i < cnt ? __ldg(&g.ent_wv[e0 + eA + i]) : 0.0;
      ci[u] = i < cnt ? __ldg(&g.ent_c[e0 + eA + i]) : 0;
      nq[u] = i < nk ? __ldg(&g.node_q[n0 + kA + i]) : 0;
      ne[u] = i < nk ? __ldg(&g.node_off[n0 + kA + i + 1]) : 0;
    }
    double cv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cv[u] = i0 + u * nthr < cnt ? __ldg(&cb[ci[u]]) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * nthr;
      if (i < cnt) prod[i] = __dmul_rn(w[u], cv[u]);
      if (i < nk) {
        const int odd = n0 + kA + i >= n1;
        nrec[i] = make_int2(ne[u] - e0 - eA, 2 * (nq[u] - rowq - odd * g.M1) + odd);
      }
    }
  }
  cl.sync();   // products staged here; both half lines zeroed (remote writes may follow)
  double* bd = (double*)buf;
  for (int k = tl; k < nk; k += nthr) {
    const int s0 = k ? nrec[k - 1].x : 0;
    const int2 r = nrec[k];
    double acc = 0.0;
    for (int i = s0; i < r.x; ++i) acc = __dadd_rn(acc, prod[i]);   // (w * c) then add, as np.add.at
    bd[r.y] = acc;
    bo_remote[r.y] = acc;
  }
  cl.sync();   // both CTAs' sums are in both lines
  if (half) {
    for (int x = tl; x < a.ncols; x += nthr) buf[x] = cmul(buf[x], split_w(wt, x));
    __syncthreads();
  }
  fft_line<false, true, 1, true, 3, LEAN ? 1 : 0>(buf, pls, tl);
  pdl_trigger();
  // Z[kx], kx = 2 mm + half, is buf[mm]; conj Z[P - kx] comes from the same half
  const int Hf = H + 1;
  const int nkx = (Hf - half + 1) / 2;   // this half's kx count
  double2* T = a.T + (int64_t)b * a.T_bstride;
  for (int idx = tl; idx < 2 * nkx; idx += nthr) {
    const int r = idx & 1, mm = idx >> 1;
    const int kx = 2 * mm + half;
    const int row = ya + r;
    if (row >= a.nrows) continue;
    const double2 z = buf[mm];
    const double2 zc = buf[half ? H - 1 - mm : (mm ? H - mm : 0)];
    double2 o;
    if (r == 0) o = make_double2(0.5 * (z.x + zc.x), 0.5 * (z.y - zc.y));
    else o = make_double2(0.5 * (z.y + zc.y), -0.5 * (z.x - zc.x));
    T[(int64_t)kx * a.ldT + row] = o;
  }
}

// U layouts between the column and inverse-row passes: standard U[kx][y] (column pass output
// contiguous), or pair-blocked when both passes are split-length: element (U row y, column kx) at
// U[(y / 2) ldp + (kx % 2) 2 hh + 2 (kx / 2) + y % 2], hh = ceil(H1 / 2), ldp = 4 hh -- the
// inverse-row pass then reads each row pair's parity half as one contiguous run.

// pass 2: column kx, this CTA's half (cluster rank) -> x real-even spectrum -> inverse half;
// the cluster's two halves are combined over DSMEM, each CTA finishing half the kept rows
// LEAN: the default configuration on a line 6 9^a (fused hooks, standard U, no fold) with everything
// else compiled out
template <bool LEAN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kSplitThreads, 2) col_split_kernel(const ColArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int half = (int)cl.block_rank();
  const int H = a.pl.n;
  const int nthr = a.pl.nthr;
  const int tl = threadIdx.x;
  const int b = blockIdx.y;
  const int kx = blockIdx.x >> 1;
  double2* buf = smem;                             // H (+ fold) entries
  double* S = (double*)(smem + H + a.fold);        // this half's spectrum (ldh)
  uint64_t* bar = (uint64_t*)(S + a.ldh);
  uint64_t* xb = bar + 1;                          // exit protection (cluster_arrive_partner)
  const double2* Tb = a.T + (int64_t)b * a.T_bstride;
  if (tl == 0) {
    mbar_init(bar, 1);
    mbar_init(xb, 1);
  }
  __syncthreads();
  const uint32_t colb = (uint32_t)a.nin * 16u, sb = (uint32_t)a.ldh * 8u;
  if (tl == 0) {
    mbar_expect_tx(bar, colb + sb);
    bulk_g2s(S, a.spec_s + ((int64_t)kx * 2 + half) * a.ldh, sb, bar);
  }
  pdl_wait();
  if (tl == 0) bulk_g2s(buf, Tb + (int64_t)kx * a.ldT, colb, bar);
  const FftPlan pls = fft_twiddles_to_smem(a.pl, smem + a.tw_off);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  for (int y = a.nin + tl; y < H; y += nthr) buf[y] = make_double2(0.0, 0.0);
  mbar_wait(bar, 0);
  __syncthreads();
  if (!LEAN && a.fold) {   // rows y >= H: X[2m] = F_H(x[n] + x[n + H]), X[2m + 1] = F_H((x[n] - x[n + H]) w^n)
    for (int n = tl; n < a.fold; n += nthr) buf[n] = half ? csub(buf[n], buf[H + n]) : cadd(buf[n], buf[H + n]);
    __syncthreads();
  }
  const int nin_h = min(a.nin, H);
  // S[k] for k = 2 mm + half: S_half[min(mm, H - half - mm)]
  if (LEAN || a.fuse_pp) {   // the odd half's twist on the first stage's loads, the product on the last stage's stores
    auto pre_tw = [&](int y, double2 v) { return half ? cmul(v, split_w(wt, y)) : v; };
    auto post_sp = [&](int mm, double2 v) { return cscale(v, S[min(mm, H - half - mm)]); };
    fft_line_pp<false, true, 1, decltype(pre_tw), decltype(post_sp), true, LEAN ? 1 : 0>(buf, pls, tl, 0, pre_tw,
                                                                                        post_sp);
  } else {
    if (half) {
      for (int y = tl; y < nin_h; y += nthr) buf[y] = cmul(buf[y], split_w(wt, y));
      __syncthreads();
    }
    fft_line<false, true, 1, true, 3>(buf, pls, tl);
    for (int mm = tl; mm < H; mm += nthr) buf[mm] = cscale(buf[mm], S[min(mm, H - half - mm)]);
    __syncthreads();
  }
  fft_line<true, true, 1, true, 3, LEAN ? 1 : 0>(buf, pls, tl);
  pdl_trigger();
  cl.sync();   // both halves transformed
  const double2* other = cl.map_shared_rank(buf, half ^ 1);
  if (!LEAN && a.upair) {   // pair-blocked U: each thread finishes one U row pair (32 contiguous bytes)
    const int nq = (a.nout + 1) >> 1, qm = (nq + 1) >> 1;
    const int q0 = half ? qm : 0, q1 = half ? nq : qm;
    double2* Ub = a.U + (int64_t)b * a.U_bstride + (int64_t)(kx & 1) * 2 * a.hh + 2 * (kx >> 1);
    for (int q = q0 + tl; q < q1; q += nthr) {
      double2 v[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int yo = 2 * q + r;
        v[r] = make_double2(0.0, 0.0);
        if (yo < a.nout) {
          const int y = a.row0 + yo;
          const double2 e = half ? other[y] : buf[y];
          const double2 o = half ? buf[y] : other[y];
          v[r] = cadd(e, cmulc(o, split_w(wt, y)));   // + w^-y (inverse half)
        }
      }
      double2* dst = Ub + (int64_t)q * a.ldp;
      dst[0] = v[0];
      dst[1] = v[1];
    }
    __syncthreads();
    if (tl == 0) cluster_arrive_partner(xb, (uint32_t)(half ^ 1));
    cluster_wait_partner(xb);   // the partner has finished reading this CTA's shared memory
    return;
  }
  const int mid = a.row0 + ((a.nout + 1) >> 1);
  const int y0 = half ? mid : a.row0, y1 = half ? a.row0 + a.nout : mid;
  // y < H: e[y] + w^-y o[y]; y >= H (execution torus): e[y - H] - w^-(y - H) o[y - H] -- those
  // sources lie below row0 (nout <= H), which no CTA overwrites
  for (int y = y0 + tl; y < y1; y += nthr) {
    const int yy = y < H ? y : y - H;
    const double2 e = half ? other[yy] : buf[yy];
    const double2 o = half ? buf[yy] : other[yy];
    const double2 t = cmulc(o, split_w(wt, yy));
    buf[y] = y < H ? cadd(e, t) : csub(e, t);
  }
  fence_async_smem();
  __syncthreads();   // this CTA's remote reads and its rows' combination are done
  if (tl == 0) {
    cluster_arrive_partner(xb, (uint32_t)(half ^ 1));
    if (y1 > y0) {   // the store (own rows only) overlaps the wait for the partner
      bulk_s2g(a.U + (int64_t)b * a.U_bstride + (int64_t)kx * a.ldU + (y0 - a.row0), buf + y0,
               (uint32_t)(y1 - y0) * 16u);
      bulk_commit();
    }
  }
  cluster_wait_partner(xb);   // the partner has finished reading this CTA's shared memory
  if (tl == 0) bulk_wait_read0();
  __syncthreads();
}

// pass 2, one CTA per SM holding a whole column: two 512-thread groups, group 0 the odd half
// (buffer A, input twisted by w_P^y), group 1 the even half (buffer B), each transforming with its
// own named barrier, so the halves are combined from the same shared memory (no cluster barrier,
// no DSMEM, no partner skew as in col_split_kernel).  The staging buffer X is time-shared by TMA:
// the column's input, then its spectrum, which lands during the forward transforms.
//   A, B: H double2 each; X: max(nin double2, 2 ldh doubles); twiddle tables; 2 mbarriers.
// (One column per CTA: a persistent loop over columns, which would let the next column's input
// land during the inverse transforms, makes ptxas spill the butterflies at the 64-register bound.)
__global__ void __launch_bounds__(2 * kSplitThreads, 1) col_pair_kernel(const ColArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  const int H = a.pl.n, G = a.pl.nthr;
  const int grp = (int)threadIdx.x >= G;   // 0: odd half (A), 1: even half (B)
  const int tl = threadIdx.x - grp * G;
  double2* A = smem;
  double2* B = smem + H;
  const double2* X = smem + 2 * H;
  double2* mine = smem + grp * H;
  uint64_t* bar = (uint64_t*)(smem + a.x_off);   // [0] input, [1] spectrum
  const int kx = blockIdx.x;
  const int64_t b = blockIdx.y;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    mbar_expect_tx(bar, (uint32_t)a.nin * 16u);
    bulk_g2s(smem + 2 * H, a.T + b * a.T_bstride + (int64_t)kx * a.ldT, (uint32_t)a.nin * 16u, bar);
  }
  const FftPlan pls = fft_twiddles_to_smem(a.pl, smem + a.tw_off);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  for (int y = a.nin + tl; y < H; y += G) mine[y] = make_double2(0.0, 0.0);
  __syncthreads();
  mbar_wait(bar, 0);
  if (grp == 0) {
    for (int y = tl; y < a.nin; y += G) A[y] = cmul(X[y], split_w(wt, y));
  } else {
    for (int y = tl; y < a.nin; y += G) B[y] = X[y];
  }
  fence_async_smem();
  __syncthreads();   // X consumed
  if (threadIdx.x == 0) {
    mbar_expect_tx(bar + 1, (uint32_t)a.ldh * 16u);
    bulk_g2s(smem + 2 * H, a.spec_s + (int64_t)kx * 2 * a.ldh, (uint32_t)a.ldh * 16u, bar + 1);
  }
  fft_line<false, true, 1, true, 3>(mine, pls, tl, 1 + grp);
  mbar_wait(bar + 1, 0);
  {
    const int half = grp ^ 1;
    const double* S = (const double*)X + half * a.ldh;
    for (int mm = tl; mm < H; mm += G) mine[mm] = cscale(mine[mm], S[min(mm, H - half - mm)]);
  }
  group_sync(1 + grp, G);
  fft_line<true, true, 1, true, 3>(mine, pls, tl, 1 + grp);
  __syncthreads();   // both halves transformed
  for (int y = a.row0 + (int)threadIdx.x; y < a.row0 + a.nout; y += 2 * G)
    B[y] = cadd(B[y], cmulc(A[y], split_w(wt, y)));   // even + w^-y odd
  fence_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    bulk_s2g(a.U + b * a.U_bstride + (int64_t)kx * a.ldU, B + a.row0, (uint32_t)a.nout * 16u);
    bulk_commit();
    bulk_wait_read0();
  }
}

// pass 2 as col_split_kernel, with the in-place Cooley-Tukey engine (rk_fft_ct.cuh): forward DIF,
// the spectrum product fused into the last forward / first inverse stage (frequency of each
// digit-reversed position computed on the fly), inverse DIT; one barrier per stage, group-local
// barriers after the first stage.  kCtThreads bounds the threads per half line (9 groups of 64
// for the 4374-point halves of cfg5's 8748 torus).
// MAXT: 576 (9 groups of 64, 56 registers) or 288 (9 single-warp groups, barriers after the
// first stage are __syncwarp, up to 113 registers).
constexpr int kCtThreads = 576;
template <int MAXT>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(MAXT, 2) col_split_ct_kernel(const __grid_constant__ ColArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int half = (int)cl.block_rank();
  const int H = a.ct.n;
  const int nthr = a.ct.nthr;
  const int tl = threadIdx.x;
  const int b = blockIdx.y;
  const int kx = blockIdx.x >> 1;
  double2* buf = smem;
  double* S = (double*)(smem + H);                 // this half's spectrum (ldh)
  uint64_t* bar = (uint64_t*)(S + a.ldh);
  const double2* Tb = a.T + (int64_t)b * a.T_bstride;
  if (tl == 0) {
    mbar_init(bar, 1);
    const uint32_t colb = (uint32_t)a.nin * 16u, sb = (uint32_t)a.ldh * 8u;
    mbar_expect_tx(bar, colb + sb);
    bulk_g2s(S, a.spec_s + ((int64_t)kx * 2 + half) * a.ldh, sb, bar);
    bulk_g2s(buf, Tb + (int64_t)kx * a.ldT, colb, bar);
  }
  const CtPlan& cp = a.ct;   // parameter space (grid constant): indexed per stage without a local copy
  double2* tws = smem + a.ct_off;
  for (int i = tl; i < cp.ntw; i += nthr) tws[i] = __ldg(&cp.tw[i]);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  for (int y = a.nin + tl; y < H; y += nthr) buf[y] = make_double2(0.0, 0.0);
  __syncthreads();   // barrier initialised, tables staged
  mbar_wait(bar, 0);
  if (half) {
    for (int y = tl; y < a.nin; y += nthr) buf[y] = cmul(buf[y], split_w(wt, y));
    __syncthreads();
  }
  // S[k] for k = 2 f + half: S_half[min(f, H - half - f)]
  ct_filter_line(buf, cp, tws, tl, 0, [&](int f) { return S[min(f, H - half - f)]; });
  cl.sync();   // both halves transformed
  const double2* other = cl.map_shared_rank(buf, half ^ 1);
  const int mid = a.row0 + ((a.nout + 1) >> 1);
  const int y0 = half ? mid : a.row0, y1 = half ? a.row0 + a.nout : mid;
  for (int y = y0 + tl; y < y1; y += nthr) {
    const double2 e = half ? other[y] : buf[y];
    const double2 o = half ? buf[y] : other[y];
    buf[y] = cadd(e, cmulc(o, split_w(wt, y)));   // + w^-y (inverse half)
  }
  fence_async_smem();
  cl.sync();   // the partner's remote reads of this CTA's rows are done
  if (tl == 0 && y1 > y0) {
    bulk_s2g(a.U + (int64_t)b * a.U_bstride + (int64_t)kx * a.ldU + (y0 - a.row0), buf + y0,
             (uint32_t)(y1 - y0) * 16u);
    bulk_commit();
    bulk_wait_read0();
  }
  __syncthreads();
}

// pass 3: Hermitian pair of interior rows -> this CTA's half spectrum (Z[k], k % 2 == half) ->
// inverse half; the cluster combines the halves over DSMEM, each CTA finishing half the
// kept columns (fixed-part / draw epilogue)
template <bool LEAN>   // LEAN: a line 6 9^a, standard U, the other code compiled out
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kSplitThreads, 2) row_inv_split_kernel(const RowInvArgs a) {
  extern __shared__ __align__(16) double2 smem[];
  cg::cluster_group cl = cg::this_cluster();
  const int half = (int)cl.block_rank();
  const int H = a.pl.n;
  const int nthr = a.pl.nthr;
  const int tl = threadIdx.x;
  const int b = blockIdx.y;
  const int Hf = H + 1;
  const int ya = 2 * (blockIdx.x >> 1);
  const double2* U = a.U + (int64_t)b * a.U_bstride;
  double2* buf = smem;
  uint64_t* xb = (uint64_t*)(smem + a.ep_off);   // exit protection (cluster_arrive_partner)
  if (tl == 0) mbar_init(xb, 1);                 // published by the first cl.sync below
  const FftPlan pls = fft_twiddles_to_smem(a.pl, smem + a.tw_off);
  const double2* wt = stage_split_tw(a.sw, smem + a.sw.off);
  pdl_wait();
  // gather: k = 2 mm + half < Hf -> Z[k] at buf[mm]; its mirror Z[P - k] (1 <= k <= H - 1) at
  // buf[H - mm] (even) / buf[H - 1 - mm] (odd)
  const int nk = (Hf - half + 1) / 2;
  const bool vA = ya < a.nrows, vB = ya + 1 < a.nrows;
  constexpr int D = 5;   // 5 x 512 threads cover a half line's <= 2305 entries in one round trip
  // (one 256-bit load per row pair, as row_inv_kernel does, measured slower here: the aligned
  // 8-register groups make the 64-register kernel spill; cfg5 pass 3 0.250 -> 0.258 ms)
  for (int base = tl; base < nk; base += D * nthr) {
    double2 A[D], B[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int mm = base + d * nthr;
      A[d] = B[d] = make_double2(0.0, 0.0);
      if (mm < nk) {
        if (!LEAN && a.upair) {   // the pair's parity run: contiguous 32-byte records
          const double2* u = U + (int64_t)(ya >> 1) * a.ldp + (int64_t)half * 2 * a.hh + 2 * mm;
          A[d] = u[0];
          B[d] = u[1];
        } else {
          const double2* u = U + (int64_t)(2 * mm + half) * a.ldU + ya;
          if (vA) A[d] = u[0];
          if (vB) B[d] = u[1];
        }
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int mm = base + d * nthr;
      if (mm < nk) {
        const int k = 2 * mm + half;
        buf[mm] = make_double2(A[d].x - B[d].y, A[d].y + B[d].x);
        if (k >= 1 && k <= H - 1) buf[half ? H - 1 - mm : H - mm] = make_double2(A[d].x + B[d].y, B[d].x - A[d].y);
      }
    }
  }
  __syncthreads();
  fft_line<true, true, 1, true, 3, LEAN ? 1 : 0>(buf, pls, tl);
  cl.sync();   // both halves transformed
  const double2* other = cl.map_shared_rank(buf, half ^ 1);
  const double* beta = a.beta ? a.beta + (int64_t)b * a.p : nullptr;
  const double* gb = a.g ? a.g + (int64_t)b * a.g_bstride : nullptr;
  const int pc = a.epi == EPI_COV ? a.p : 0;
  double* out = a.out + (int64_t)b * a.out_bstride;
  const int xm = (a.ncols + 1) >> 1;
  const int x0 = half ? xm : 0, x1 = half ? a.ncols : xm;
  // each combined value z gives both rows (real part: row ya, imaginary part: row ya + 1), so the
  // partner's value is read over DSMEM once per column
  for (int x = x0 + tl; x < x1; x += nthr) {
    const int nn = a.col0 + x;
    const double2 ev = half ? other[nn] : buf[nn];
    const double2 ov = half ? buf[nn] : other[nn];
    const double2 z = cadd(ev, cmulc(ov, split_w(wt, nn)));
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const int y = ya + which;
      if (y >= a.nrows) break;
      double v = which ? z.y : z.x;
      if (a.ac_corr) v += ac_row_corr(a, b, y, x);
      if (a.epi == EPI_SCALAR) {
        v = v + beta[0];
      } else if (a.epi == EPI_COV) {
        const double* xr = a.xg + ((int64_t)y * a.ncols + x) * pc;
        double fx = 0.0;
        for (int q = 0; q < pc; ++q) fx = fma(xr[q], beta[q], fx);
        v = v + fx;
      }
      if (gb) v = gb[(int64_t)(a.g_row0 + y) * a.g_ld + a.g_col0 + x] - v;
      out[(int64_t)y * a.ldo + x] = v;
    }
  }
  __syncthreads();   // this CTA's remote reads are done
  if (tl == 0) cluster_arrive_partner(xb, (uint32_t)(half ^ 1));
  cluster_wait_partner(xb);   // ... and the partner's, before this CTA's shared memory goes away
}

// ----------------------------------------------------------------- aliased-lag corrections
// (AliasCorr, rk_internal.cuh; rk_core.cu choose_exec_y): for each pair (input row u, interior
// output row y) whose lag d = |y - u| exceeds half the execution torus P2, the convolution used
// K(P2 - d, .) where the reference uses K(d, .); the difference is the one-dimensional
// convolution corr[y][x] = sum_v c*[u][v] g_d(x - v), g_d(dx) = K(d, dx) - K(P2 - d, dx), added
// in pass 3's epilogue.  c* rows u ("strips") come from the sparse plan (or the dense input);
// the sums run in chunks of kAcChunk inputs (partial sums, then added in chunk order:
// deterministic).
constexpr int kAcChunk = 512, kAcTile = 128;

__global__ void __launch_bounds__(256) ac_strips_kernel(const SparseSrc g, const double* __restrict__ rows,
                                                        int64_t ld_rows, int64_t rows_bs, const AliasCorr ac,
                                                        int M1, double* __restrict__ strips, int64_t sbs) {
  const int k = blockIdx.x, b = blockIdx.y, u = ac.ru[k];
  double* st = strips + (int64_t)b * sbs + (int64_t)k * M1;
  for (int x = threadIdx.x; x < M1; x += blockDim.x)
    st[x] = rows ? rows[(int64_t)b * rows_bs + (int64_t)u * ld_rows + x] : 0.0;
  if (rows) return;
  __syncthreads();
  gather_row(g, g.c + (int64_t)b * g.c_stride, u, threadIdx.x, blockDim.x, [&](int x, double v) { st[x] = v; });
}

// grid (output tiles, row pairs, batch x chunks), kAcTile threads: partial sums of one chunk
__global__ void __launch_bounds__(kAcTile) ac_partial_kernel(const AliasCorr ac, const double* __restrict__ ker,
                                                             const double* __restrict__ strips, int64_t sbs,
                                                             int M1, int m1, int col0, int nchunk,
                                                             double* __restrict__ part, int64_t pbs) {
  __shared__ double sv[kAcChunk];
  __shared__ double sk[kAcChunk + kAcTile];
  const int k = blockIdx.y;
  const int b = blockIdx.z / nchunk, ch = blockIdx.z - b * nchunk;
  const int o0 = blockIdx.x * kAcTile;
  const int v0 = ch * kAcChunk, v1 = min(M1, v0 + kAcChunk);
  const double* st = strips + (int64_t)b * sbs + (int64_t)ac.rp_strip[k] * M1;
  const int L1 = 2 * M1 - 1;
  const double* kr = ker + (int64_t)ac.rp_ker[k] * L1;
  for (int i = threadIdx.x; i < v1 - v0; i += blockDim.x) sv[i] = st[v0 + i];
  // term (o, v): kr[col0 + o - v + M1 - 1]; the tile needs indices kbase .. kbase + klen - 1
  const int kbase = col0 + o0 - (v1 - 1) + M1 - 1, klen = (v1 - v0) + kAcTile - 1;
  for (int i = threadIdx.x; i < klen; i += blockDim.x) {
    const int idx = kbase + i;
    sk[i] = idx >= 0 && idx < L1 ? kr[idx] : 0.0;
  }
  __syncthreads();
  const int o = o0 + threadIdx.x;
  if (o >= m1) return;
  const int t = threadIdx.x + (v1 - 1);
  double acc = 0.0;
  for (int v = v0; v < v1; ++v) acc = fma(sv[v - v0], sk[t - v], acc);
  part[(int64_t)b * pbs + ((int64_t)k * nchunk + ch) * m1 + o] = acc;
}

__global__ void ac_reduce_kernel(int nrp, const double* __restrict__ part, int64_t pbs, int nchunk, int m1,
                                 double* __restrict__ corr, int64_t cbs, int batch) {
  const int64_t tot = (int64_t)batch * nrp * m1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(e % m1);
    const int64_t kb = e / m1;
    const int k = (int)(kb % nrp), b = (int)(kb / nrp);
    const double* p = part + (int64_t)b * pbs + (int64_t)k * nchunk * m1 + o;
    double acc = 0.0;
    for (int ch = 0; ch < nchunk; ++ch) acc += p[(int64_t)ch * m1];
    corr[(int64_t)b * cbs + (int64_t)k * m1 + o] = acc;
  }
}

// ----------------------------------------------------------------- launches
// dynamic smem = kernel-specific region (bytes, 16-aligned) + the staged twiddle table
static inline int tw_slot(size_t bytes_before) { return (int)((bytes_before + 15) / 16); }
static inline size_t with_tw(size_t bytes_before, const FftPlan& pl) {
  return (size_t)tw_slot(bytes_before) * 16 + (size_t)pl.ntw * 16;
}
// the table is staged in smem when it fits next to the lines (else read through L1/L2)
static constexpr size_t kSmemMax = 227 * 1024;
static constexpr size_t kCSmemMax = 16 * 1024;   // largest c (bytes) pass 1 stages in smem
static inline bool tw_fits(size_t bytes_before, const FftPlan& pl) { return with_tw(bytes_before, pl) <= kSmemMax; }
// WIDE kernels are only instantiated with the table in smem (wide plans exist for n <= 4608)
static inline Status wide_needs_tws(const FftPlan& pl, bool tws) {
  if (pl.wide >= 2 && !tws) return Status::err(RK_INTERNAL, "wide FFT plan without room for its twiddle table");
  return Status::ok();
}

// LEAN instantiations of the split-length kernels and the WIDE column pass: lines 6 9^a (4374: the halves of the 8748 torus),
// every other stage body and option compiled out (RK_LEAN=0: the general kernels)
static bool lean_family(const FftPlan& pl) {
  static const bool lean_env = !(getenv("RK_LEAN") && atoi(getenv("RK_LEAN")) == 0);
  return lean_env && fft_family69(pl);
}

static Status launch_row_fwd(int src, const RowFwdArgs& a0, int batch, cudaStream_t st) {
  RowFwdArgs a = a0;
  const int pairs = (a.nrows + 1) / 2;
  const dim3 grid((unsigned)ceil_div(pairs, a.lpc), (unsigned)batch);
  size_t smem = sizeof(double2) * a.pl.n * a.lpc;
  const int threads = a.lpc * a.pl.nthr;
  if (src == SRC_ROWS) smem += (a.tma == 2 ? 0 : (size_t)a.lpc * 2 * a.ld_in * sizeof(double)) + 16;
  if (src == SRC_SPARSE) {
    a.prod_off = tw_slot(smem);
    smem = (size_t)a.prod_off * 16 + sizeof(double) * (size_t)a.lpc * 2 * a.prod_cap;
    if (a.pblk) {   // per line: one plan block + its barrier
      a.pl_off = tw_slot(smem);
      smem = (size_t)a.pl_off * 16 + (size_t)a.lpc * (size_t)(a.pblk_stride + 16);
    }
    if (a.c_n > 0) {   // whole c in smem only while it stays a small share of the CTA's budget
      const bool aligned = (reinterpret_cast<uintptr_t>(a.sp.c) & 15) == 0 && (a.sp.c_stride * 8) % 16 == 0;
      if (aligned && (size_t)a.c_n * 8 <= kCSmemMax) {
        a.c_off = tw_slot(smem);
        smem = (size_t)a.c_off * 16 + sizeof(double) * (size_t)((a.c_n + 1) & ~1) + 16;
      } else {
        a.c_n = 0;
      }
    }
  }
  a.tw_off = tw_slot(smem);
  const bool tws = tw_fits(smem, a.pl);
  if (tws) smem = with_tw(smem, a.pl);
  RK_TRY(wide_needs_tws(a.pl, tws));
  auto kern = a.pl.wide == 2 ? (src == SRC_ROWS ? row_fwd_kernel<SRC_ROWS, true, 1>
                                : src == SRC_LAG ? row_fwd_kernel<SRC_LAG, true, 1>
                                                 : row_fwd_kernel<SRC_SPARSE, true, 1>)
              : a.pl.wide == 3 ? (src == SRC_ROWS ? row_fwd_kernel<SRC_ROWS, true, 2>
                                  : src == SRC_LAG ? row_fwd_kernel<SRC_LAG, true, 2>
                                                   : row_fwd_kernel<SRC_SPARSE, true, 2>)
              : src == SRC_ROWS ? (tws ? row_fwd_kernel<SRC_ROWS, true, 0> : row_fwd_kernel<SRC_ROWS, false, 0>)
              : src == SRC_LAG  ? (tws ? row_fwd_kernel<SRC_LAG, true, 0> : row_fwd_kernel<SRC_LAG, false, 0>)
                                : (tws ? row_fwd_kernel<SRC_SPARSE, true, 0> : row_fwd_kernel<SRC_SPARSE, false, 0>);
  RK_TRY(set_smem_attr((const void*)kern, smem));
  RK_CUDA_TRY(launch_pdl(kern, grid, dim3(threads), smem, st, a));
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

static Status launch_col(int mode, const ColArgs& a0, int batch, cudaStream_t st) {
  ColArgs a = a0;
  const dim3 grid((unsigned)ceil_div(a.ncols, a.lpc), (unsigned)batch);
  size_t smem = sizeof(double2) * a.pl.n * a.lpc + 16;
  const int threads = a.lpc * a.pl.nthr;
  if (mode == 0) smem += sizeof(double) * (size_t)a.lpc * a.ldq;
  a.tw_off = tw_slot(smem);
  const bool tws = tw_fits(smem, a.pl);
  if (tws) smem = with_tw(smem, a.pl);
  RK_TRY(wide_needs_tws(a.pl, tws));
  auto kern = a.pl.wide == 2 ? (mode == 0 ? (lean_family(a.pl) ? col_kernel<0, true, 1, 1> : col_kernel<0, true, 1>)
                                          : col_kernel<1, true, 1>)
              : a.pl.wide == 3 ? (mode == 0 ? col_kernel<0, true, 2> : col_kernel<1, true, 2>)
              : mode == 0 ? (tws ? col_kernel<0, true, 0> : col_kernel<0, false, 0>)
                          : (tws ? col_kernel<1, true, 0> : col_kernel<1, false, 0>);
  RK_TRY(set_smem_attr((const void*)kern, smem));
  RK_CUDA_TRY(launch_pdl(kern, grid, dim3(threads), smem, st, a));
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

static Status launch_row_inv(const RowInvArgs& a0, int batch, cudaStream_t st) {
  RowInvArgs a = a0;
  const int pairs = (a.nrows + 1) / 2;
  const dim3 grid((unsigned)ceil_div(pairs, a.lpc), (unsigned)batch);
  size_t smem = sizeof(double2) * a.pl.n * a.lpc;
  a.ep_off = tw_slot(smem);
  const int pc = a.epi == EPI_COV ? a.p : 0;
  const size_t ep_bytes = sizeof(double) * (size_t)a.lpc * 2 * a.ncols * (pc + (a.g ? 1 : 0)) + 16;
  a.xg_bulk = a.xg && (reinterpret_cast<uintptr_t>(a.xg) & 15) == 0;
  // prefetching the epilogue operands must not cost the twiddle table or occupancy: only
  // when both fit (large rows read them from global in the epilogue instead)
  a.ep_smem = (size_t)a.ep_off * 16 + ep_bytes + (size_t)a.pl.ntw * 16 + 16 <= kSmemMax;
  if (a.ep_smem) smem = (size_t)a.ep_off * 16 + ep_bytes;
  a.tw_off = tw_slot(smem);
  const bool tws = tw_fits(smem, a.pl);
  if (tws) smem = with_tw(smem, a.pl);
  RK_TRY(wide_needs_tws(a.pl, tws));
  auto kern = a.pl.wide == 2 ? row_inv_kernel<true, 1>
              : a.pl.wide == 3 ? row_inv_kernel<true, 2>
              : tws ? row_inv_kernel<true, 0> : row_inv_kernel<false, 0>;
  RK_TRY(set_smem_attr((const void*)kern, smem));
  RK_CUDA_TRY(launch_pdl(kern, grid, dim3(a.lpc * a.pl.nthr), smem, st, a));
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

// split-length launches (see row_fwd_split_kernel); *done = false when the layout does not fit
static inline size_t split_tail(size_t bytes, const FftPlan& pl, SplitTw* sw, int* tw_off) {
  *tw_off = tw_slot(bytes);
  bytes = (size_t)*tw_off * 16 + (size_t)pl.ntw * 16;
  sw->off = tw_slot(bytes);
  return (size_t)sw->off * 16 + (size_t)(128 + sw->nhi) * 16;
}

static Status launch_row_fwd_split(const RowFwdArgs& a0, int batch, cudaStream_t st, bool* done) {
  RowFwdArgs a = a0;
  *done = false;
  a.lpc = 1;
  if (a.pl.nthr > kSplitThreads) return Status::ok();
  size_t smem = sizeof(double2) * (size_t)a.pl.n;
  a.prod_off = tw_slot(smem);
  smem = (size_t)a.prod_off * 16 + sizeof(double) * 2 * (size_t)a.prod_cap;
  smem = split_tail(smem, a.pl, &a.sw, &a.tw_off);
  if (smem > kSmemMax) return Status::ok();
  const dim3 grid((unsigned)(2 * ((a.nrows + 1) / 2)), (unsigned)batch);
  if (lean_family(a.pl)) {
    RK_TRY(set_smem_attr((const void*)row_fwd_split_kernel<true>, smem));
    row_fwd_split_kernel<true><<<grid, a.pl.nthr, smem, st>>>(a);
  } else {
    RK_TRY(set_smem_attr((const void*)row_fwd_split_kernel<false>, smem));
    row_fwd_split_kernel<false><<<grid, a.pl.nthr, smem, st>>>(a);
  }
  count_launch();
  RK_LAUNCH_CHECK();
  *done = true;
  return Status::ok();
}

static Status launch_col_split(const ColArgs& a0, int batch, cudaStream_t st, bool* done) {
  ColArgs a = a0;
  *done = false;
  a.lpc = 1;
  if (a.pl.nthr > kSplitThreads) return Status::ok();
  if (!a.spec_s) return Status::ok();
  a.fold = std::max(0, a.nin - a.pl.n);
  if (a.fold > kSplitFold || (a.fold && a.upair)) return Status::ok();
  size_t smem = sizeof(double2) * (size_t)(a.pl.n + a.fold) + sizeof(double) * (size_t)a.ldh + 16;
  smem = split_tail(smem, a.pl, &a.sw, &a.tw_off);
  if (smem > kSmemMax) return Status::ok();
  static const bool fuse = !(getenv("RK_FUSE_PP") && atoi(getenv("RK_FUSE_PP")) == 0);
  a.fuse_pp = fuse && fft_line_pp_ok(a.pl);
  const dim3 grid((unsigned)(2 * a.ncols), (unsigned)batch);
  if (lean_family(a.pl) && a.fuse_pp && !a.upair && a.fold == 0) {
    RK_TRY(set_smem_attr((const void*)col_split_kernel<true>, smem));
    col_split_kernel<true><<<grid, a.pl.nthr, smem, st>>>(a);
  } else {
    RK_TRY(set_smem_attr((const void*)col_split_kernel<false>, smem));
    col_split_kernel<false><<<grid, a.pl.nthr, smem, st>>>(a);
  }
  count_launch();
  RK_LAUNCH_CHECK();
  *done = true;
  return Status::ok();
}

// one CTA per SM, both halves of a column per CTA (col_pair_kernel); *done = false when it does not
// apply (pair-blocked U, plan wider than a group, shared memory)
static Status launch_col_pair(const ColArgs& a0, int batch, cudaStream_t st, bool* done) {
  ColArgs a = a0;
  *done = false;
  // measured on cfg5 (B200): 0.765 ms vs the cluster kernel's 0.698 -- one CTA per SM exposes
  // each column's input load, which two co-resident cluster CTAs hide; off unless RK_COL_PAIR=1
  static const bool on = getenv("RK_COL_PAIR") && atoi(getenv("RK_COL_PAIR")) == 1;
  if (!on || a.upair || !a.spec_s || a.pl.nthr > kSplitThreads) return Status::ok();
  if (a.nin > a.pl.n || a.row0 + a.nout > a.pl.n) return Status::ok();   // no fold / tail rows here
  a.lpc = 1;
  a.batch = batch;
  const size_t xb = std::max((size_t)a.nin * 16, (size_t)a.ldh * 16);
  size_t smem = sizeof(double2) * 2 * (size_t)a.pl.n + xb;
  smem = split_tail(smem, a.pl, &a.sw, &a.tw_off);
  a.x_off = tw_slot(smem);
  smem = (size_t)a.x_off * 16 + 16;
  if (smem > kSmemMax) return Status::ok();
  RK_TRY(set_smem_attr((const void*)col_pair_kernel, smem));
  col_pair_kernel<<<dim3((unsigned)a.ncols, (unsigned)batch), 2 * a.pl.nthr, smem, st>>>(a);
  count_launch();
  RK_LAUNCH_CHECK();
  *done = true;
  return Status::ok();
}

// split-length column pass on the Cooley-Tukey engine (col_split_ct_kernel); *done = false when it
// does not apply (RK_COL_CT=0, pair-blocked U, no plan within kCtThreads, shared memory)
static Status launch_col_split_ct(const ColArgs& a0, int batch, cudaStream_t st, bool* done) {
  ColArgs a = a0;
  *done = false;
  // measured on cfg5 (B200): G = 64 0.804 ms, G = 32 0.701 ms vs the Stockham cluster kernel's
  // 0.696 (ncu: 40 % more instructions -- per-butterfly index arithmetic, the radix dispatch,
  // digit reversal -- and 3x the bank conflicts of the strided in-place stages eat the saved
  // barriers); off unless RK_COL_CT=1
  static const bool on = getenv("RK_COL_CT") && atoi(getenv("RK_COL_CT")) == 1;
  static const int g_env = getenv("RK_CT_G") ? atoi(getenv("RK_CT_G")) : 0;
  if (!on || a.upair || !a.spec_s) return Status::ok();
  if (a.nin > a.pl.n || a.row0 + a.nout > a.pl.n) return Status::ok();   // no fold / tail rows here
  CtPlan cp{};
  if (!ct_plan_for(a.pl.n, g_env, &cp).good() || cp.nthr > kCtThreads) return Status::ok();
  a.ct = cp;
  a.lpc = 1;
  size_t smem = sizeof(double2) * (size_t)cp.n + sizeof(double) * (size_t)a.ldh + 16;
  a.ct_off = tw_slot(smem);
  smem = (size_t)a.ct_off * 16 + (size_t)cp.ntw * 16;
  a.sw.off = tw_slot(smem);
  smem = (size_t)a.sw.off * 16 + (size_t)(128 + a.sw.nhi) * 16;
  if (smem > kSmemMax) return Status::ok();
  auto kern = cp.nthr <= 288 ? col_split_ct_kernel<288> : col_split_ct_kernel<kCtThreads>;
  RK_TRY(set_smem_attr((const void*)kern, smem));
  const dim3 grid((unsigned)(2 * a.ncols), (unsigned)batch);
  kern<<<grid, cp.nthr, smem, st>>>(a);
  count_launch();
  RK_LAUNCH_CHECK();
  *done = true;
  return Status::ok();
}

static Status launch_row_inv_split(const RowInvArgs& a0, int batch, cudaStream_t st, bool* done) {
  RowInvArgs a = a0;
  *done = false;
  a.lpc = 1;
  if (a.pl.nthr > kSplitThreads) return Status::ok();
  size_t smem = sizeof(double2) * (size_t)a.pl.n;
  smem = split_tail(smem, a.pl, &a.sw, &a.tw_off);
  a.ep_off = tw_slot(smem);   // the exit-protection mbarrier
  smem = (size_t)a.ep_off * 16 + 16;
  if (smem > kSmemMax) return Status::ok();
  const dim3 grid((unsigned)(2 * ((a.nrows + 1) / 2)), (unsigned)batch);
  if (lean_family(a.pl) && !a.upair) {
    RK_TRY(set_smem_attr((const void*)row_inv_split_kernel<true>, smem));
    row_inv_split_kernel<true><<<grid, a.pl.nthr, smem, st>>>(a);
  } else {
    RK_TRY(set_smem_attr((const void*)row_inv_split_kernel<false>, smem));
    row_inv_split_kernel<false><<<grid, a.pl.nthr, smem, st>>>(a);
  }
  count_launch();
  RK_LAUNCH_CHECK();
  *done = true;
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

int quarter_ld(int p2) { return ((p2 / 2 + 1) + 1) & ~1; }

// Re(fft2(lag filter))[ky, kx] * scale for kx <= p1/2, ky <= p2/2, stored out_q[kx * ldq + ky]
Status spectrum_quarter(const MaternDev& P, double hx, double hy, int p1, int p2, double scale,
                        double* out_q, int ldq, cudaStream_t st) {
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
  RK_CUDA_TRY(cudaMemsetAsync(out_q, 0, sizeof(double) * (size_t)H1 * ldq, st));
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
  ca.ldq = ldq;
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

// Standalone scatter (coefficients_to_grid): one CTA per padded row, zero-filled in smem,
// gathered from the sparse plan, written out coalesced.  Work ~ n M + G.

__global__ void __launch_bounds__(256) cstar_rows_kernel(SparseSrc g, double* __restrict__ out,
                                                         int64_t ldo, int64_t out_bstride) {
  extern __shared__ __align__(16) double rowbuf[];
  const int y = blockIdx.x, b = blockIdx.y;
  const double* c = g.c + (int64_t)b * g.c_stride;
  for (int x = threadIdx.x; x < g.M1; x += blockDim.x) rowbuf[x] = 0.0;
  __syncthreads();
  gather_row(g, c, y, threadIdx.x, blockDim.x, [&](int x, double v) { rowbuf[x] = v; });
  pdl_trigger();   // the row-FFT pass may stage its twiddles while the rows are stored
  __syncthreads();
  double* o = out + (int64_t)b * out_bstride + (int64_t)y * ldo;
  for (int x = threadIdx.x; x < g.M1; x += blockDim.x) o[x] = rowbuf[x];
}

static SparseSrc sparse_src(const rk_setup* s, const double* c, int64_t c_stride) {
  SparseSrc g;
  g.node_q = s->node_q;
  g.node_off = s->node_off;
  g.row_node = s->row_node;
  g.ent_w = s->ent_w;
  g.ent_c = s->ent_c;
  g.wsort = s->wsort;
  g.ent_wv = s->ent_wv;
  g.pair_info = s->pair_info;
  g.c = c;
  g.c_stride = c_stride;
  g.M1 = s->M1;
  return g;
}

// pass 1 stages one row pair's products per line: fused while that stays small
// (RK_FUSED_GATHER=0 forces the standalone scatter; tests compare both)
static bool fused_gather(const rk_setup* s) {
  static const bool allow = !(getenv("RK_FUSED_GATHER") && atoi(getenv("RK_FUSED_GATHER")) == 0);
  return allow && s->max_pair_ent * 16 <= 64 * 1024;
}

static Status launch_cstar(const rk_setup* s, const double* c, int64_t c_stride, double* out,
                           int64_t ldo, int batch, cudaStream_t st) {
  const SparseSrc g = sparse_src(s, c, c_stride);
  const size_t smem = sizeof(double) * (size_t)s->M1;
  RK_TRY(set_smem_attr((const void*)cstar_rows_kernel, smem));
  cstar_rows_kernel<<<dim3((unsigned)s->M2, (unsigned)batch), 256, smem, st>>>(g, out, ldo, ldo * s->M2);
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

static inline int64_t round_even(int64_t v) { return (v + 1) & ~int64_t(1); }

// aliased-lag corrections of one conv_pipeline call (interior outputs): strips, partial sums,
// corrections corr[b][pair][x] (*corr null when the setup has none); *owned: scratch to free
static Status alias_corrections(const rk_setup* s, const SparseSrc* sp, const double* rows, int64_t ld_in,
                                int64_t in_bstride, int batch, Workspace* ws, cudaStream_t st, double** corr,
                                int64_t* cbs, double** owned) {
  *corr = nullptr;
  *owned = nullptr;
  const AliasCorr& ac = s->ac;
  if (ac.nrp == 0) return Status::ok();
  const int M1 = s->M1, m1 = s->m1, nchunk = (int)ceil_div(M1, kAcChunk);
  const int64_t sbs = (int64_t)ac.nru * M1, pbs = (int64_t)ac.nrp * nchunk * m1, cb = (int64_t)ac.nrp * m1;
  const size_t per = (size_t)(sbs + pbs + cb);
  double* buf = nullptr;
  if (ws && batch == 1) {
    if (ws->ac_cap < per) {
      cudaFree(ws->ac_buf);
      ws->ac_buf = nullptr;
      ws->ac_cap = 0;
      RK_CUDA_TRY(cudaMalloc(&ws->ac_buf, sizeof(double) * per));
      ws->ac_cap = per;
    }
    buf = ws->ac_buf;
  } else {
    RK_TRY(scratch_alloc((void**)&buf, sizeof(double) * per * batch, st));
    *owned = buf;
  }
  double* strips = buf;
  double* part = strips + sbs * batch;
  double* cr = part + pbs * batch;
  SparseSrc g = sp ? *sp : SparseSrc{};
  ac_strips_kernel<<<dim3((unsigned)ac.nru, (unsigned)batch), 256, 0, st>>>(g, sp ? nullptr : rows, ld_in, in_bstride,
                                                                            ac, M1, strips, sbs);
  ac_partial_kernel<<<dim3((unsigned)ceil_div(m1, kAcTile), (unsigned)ac.nrp, (unsigned)(batch * nchunk)), kAcTile,
                      0, st>>>(ac, s->ac_ker, strips, sbs, M1, m1, s->grid.pad[0], nchunk, part, pbs);
  ac_reduce_kernel<<<(int)std::min<int64_t>(ceil_div((int64_t)batch * cb, 256), 148 * 8), 256, 0, st>>>(
      ac.nrp, part, pbs, nchunk, m1, cr, cb, batch);
  count_launch(3);
  RK_LAUNCH_CHECK();
  *corr = cr;
  *cbs = cb;
  return Status::ok();
}

// Shared 3-pass convolution. `rows` (nrows = M2, ld_in) holds the padded real input
// (c* or a caller field); output rows [row0, row0 + nout) x cols [col0, col0 + ncols).
static Status conv_pipeline(const rk_setup* s, const double* rows, int64_t ld_in, int64_t in_bstride,
                            int batch, int row0, int nout, int col0, int ncols, RowInvArgs epi,
                            cudaStream_t st, cudaEvent_t* ev = nullptr, Workspace* ws = nullptr,
                            const HostIo* hio = nullptr, const SparseSrc* sp = nullptr) {
  const int64_t ldT = round_even(s->M2);
  const int64_t ldU = round_even(nout);
  // pair-blocked U when both the column and the inverse-row passes are split-length
  const bool split2 = s->h2v.v[2].n && s->spec_s && nout <= s->p2 / 2 && row0 + nout <= s->p2 / 2 + kSplitFold;
  const bool split3 = s->h1v.v[2].n && col0 + ncols <= s->p1 / 2;
  // measured on cfg5 (B200): pair-blocked U takes pass 3 from 0.336 to 0.291 ms but pass 2's
  // scattered 32-byte stores cost more (0.697 -> 0.813 ms); off unless RK_UPAIR=1
  static const bool upair_env = getenv("RK_UPAIR") && atoi(getenv("RK_UPAIR")) == 1;
  const bool upair = upair_env && split2 && split3 && s->M2 <= s->p2 / 2 && row0 + nout <= s->p2 / 2;
  const int hh = (s->H1 + 1) / 2;
  const int64_t U_bstride = (int64_t)(s->H1 + 1) * ldU;   // holds either layout
  double2 *T = nullptr, *U = nullptr;
  const bool own = !(ws && batch == 1);
  if (own) {
    RK_TRY(scratch_alloc((void**)&T, sizeof(double2) * (size_t)s->H1 * ldT * batch, st));
    RK_TRY(scratch_alloc((void**)&U, sizeof(double2) * (size_t)U_bstride * batch, st));
  } else {
    T = ws->T;
    U = ws->U;
  }
  // execution torus: the aliased-lag corrections only read the input, so with a workspace they run
  // on its second side stream beside passes 1 and 2 and are joined before pass 3
  double* ac_owned = nullptr;
  double* corr = nullptr;
  int64_t cbs = 0;
  bool ac_forked = false;
  if (s->ac.nrp) {
    if (row0 != s->grid.pad[2] || nout != s->m2 || col0 != s->grid.pad[0] || ncols != s->m1)
      return Status::err(RK_INTERNAL, "execution-torus convolution for non-interior outputs");
    static const bool ac_async = !(getenv("RK_AC_ASYNC") && atoi(getenv("RK_AC_ASYNC")) == 0);
    if (ac_async && ws && batch == 1 && !ev) {
      RK_CUDA_TRY(cudaEventRecord(ws->ac_fork, st));
      RK_CUDA_TRY(cudaStreamWaitEvent(ws->aux2, ws->ac_fork, 0));
      RK_TRY(alias_corrections(s, sp, rows, ld_in, in_bstride, batch, ws, ws->aux2, &corr, &cbs, &ac_owned));
      RK_CUDA_TRY(cudaEventRecord(ws->ac_join, ws->aux2));
      ac_forked = true;
    }
  }
  RowFwdArgs ra{};
  ra.pl = plan_pick(s->pl1v, (int64_t)((s->M2 + 1) / 2) * batch);
  ra.lpc = pick_lpc(ra.pl, 4, (int64_t)((s->M2 + 1) / 2) * batch);
  ra.nrows = s->M2;
  ra.ncols = s->M1;
  ra.T = T;
  ra.ldT = ldT;
  ra.T_bstride = (int64_t)s->H1 * ldT;
  ra.rows = rows;
  ra.ld_in = ld_in;
  ra.in_bstride = in_bstride;
  ra.tma = ((ld_in * 8) % 16 == 0) && ((reinterpret_cast<uintptr_t>(rows) & 15) == 0) &&
           ((in_bstride * 8) % 16 == 0);
  if (ra.tma && s->pl1.n - ld_in >= s->M1) ra.tma = 2;   // stage inside the line's zero tail
  if (sp) {
    ra.sp = *sp;
    ra.tma = 0;
    ra.prod_cap = (int)((s->max_pair_ent + 1) & ~int64_t(1));
    static const bool c_smem = !(getenv("RK_C_SMEM") && atoi(getenv("RK_C_SMEM")) == 0);
    ra.c_n = c_smem ? (int)s->n : 0;
    // plan ranges by TMA only for one-wave launches (spread / split plans): elsewhere the extra
    // shared memory would cost occupancy
    static const bool plan_tma = !(getenv("RK_PLAN_TMA") && atoi(getenv("RK_PLAN_TMA")) == 0);
    if (plan_tma && s->pblk && (ra.pl.wide == 1 || ra.pl.wide == 3) &&
        (size_t)ra.lpc * (size_t)(s->pblk_stride + 16) <= 64 * 1024) {
      ra.pblk = s->pblk;
      ra.pblk_stride = s->pblk_stride;
      ra.pblk_cap = s->pblk_cap;
    }
  }
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[1], st));
  bool done = false;
  if (sp && s->h1v.v[2].n) {   // split-length row pass (p1 = 2 H, the M1 nonzero columns < H)
    RowFwdArgs rs = ra;
    rs.pl = s->h1v.v[2];
    rs.sw = s->sw1;
    rs.prod_cap = (int)((s->max_half_ent + 1) & ~int64_t(1));   // each CTA stages half the nodes
    RK_TRY(launch_row_fwd_split(rs, batch, st, &done));
  }
  if (!done) RK_TRY(launch_row_fwd(sp ? SRC_SPARSE : SRC_ROWS, ra, batch, st));
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[2], st));
  ColArgs ca{};
  ca.pl = plan_pick(s->pl2v, (int64_t)s->H1 * batch);
  ca.lpc = pick_lpc(ca.pl, 4, (int64_t)s->H1 * batch);
  ca.ncols = s->H1;
  ca.nin = s->M2;
  ca.T = T;
  ca.ldT = ldT;
  ca.T_bstride = ra.T_bstride;
  ca.spec_q = s->spec_q;
  ca.ldq = s->Q2;
  ca.row0 = row0;
  ca.nout = nout;
  ca.U = U;
  ca.ldU = ldU;
  ca.U_bstride = U_bstride;
  done = false;
  if (split2) {   // split-length column pass
    ColArgs cs = ca;
    cs.pl = s->h2v.v[2];
    cs.sw = s->sw2;
    cs.spec_s = s->spec_s;
    cs.ldh = s->ldh;
    cs.upair = upair;
    cs.hh = hh;
    cs.ldp = 4LL * hh;
    RK_TRY(launch_col_pair(cs, batch, st, &done));
    if (!done) RK_TRY(launch_col_split_ct(cs, batch, st, &done));
    if (!done) RK_TRY(launch_col_split(cs, batch, st, &done));
  }
  if (!done) RK_TRY(launch_col(0, ca, batch, st));
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[3], st));
  if (s->ac.nrp) {   // execution torus: exact only with the corrections, for the interior
    if (ac_forked) RK_CUDA_TRY(cudaStreamWaitEvent(st, ws->ac_join, 0));
    else RK_TRY(alias_corrections(s, sp, rows, ld_in, in_bstride, batch, ws, st, &corr, &cbs, &ac_owned));
    epi.ac_corr = corr;
    epi.ac_cbs = cbs;
    epi.ac_row0 = 0;
    epi.ac = s->ac;
  }
  RowInvArgs ia = epi;
  ia.pl = plan_pick(s->pl1v, (int64_t)((nout + 1) / 2) * batch);
  ia.lpc = pick_lpc(ia.pl, 4, (int64_t)((nout + 1) / 2) * batch);
  ia.nrows = nout;
  ia.U = U;
  ia.ldU = ldU;
  ia.U_bstride = ca.U_bstride;
  ia.col0 = col0;
  ia.ncols = ncols;
  if (!hio) {
    done = false;
    if (split3) {   // split-length inverse row pass
      RowInvArgs is = ia;
      is.pl = s->h1v.v[2];
      is.sw = s->sw1;
      is.upair = upair;
      is.hh = hh;
      is.ldp = 4LL * hh;
      RK_TRY(launch_row_inv_split(is, batch, st, &done));
    }
    if (!done) RK_TRY(launch_row_inv(ia, batch, st));
  } else {   // batch == 1: row blocks, each followed by its device -> host copy
    const int per = chunk_rows(nout, hio->chunks);
    for (int k = 0, r0 = 0; r0 < nout; ++k, r0 += per) {
      const int r1 = std::min(nout, r0 + per);
      RowInvArgs ck = ia;
      ck.nrows = r1 - r0;
      ck.ac_row0 = r0;
      ck.U = upair && split3 ? U + (int64_t)(r0 / 2) * 4LL * hh : U + r0;   // r0 is even
      ck.out = ia.out + (int64_t)r0 * ia.ldo;
      if (ck.xg) ck.xg = ia.xg + (int64_t)r0 * ncols * ia.p;
      ck.g_row0 = ia.g_row0 + r0;
      ck.lpc = pick_lpc(ck.pl, 4, (int64_t)((ck.nrows + 1) / 2));
      if (hio->xev) RK_CUDA_TRY(cudaStreamWaitEvent(st, hio->xev[k], 0));
      done = false;
      if (split3) {
        RowInvArgs is = ck;
        is.pl = s->h1v.v[2];
        is.sw = s->sw1;
        is.upair = upair;
        is.hh = hh;
        is.ldp = 4LL * hh;
        RK_TRY(launch_row_inv_split(is, 1, st, &done));
      }
      if (!done) RK_TRY(launch_row_inv(ck, 1, st));
      if (hio->out_host) {
        cudaStream_t cq = st;
        if (hio->copy) {   // overlap this block's copy with the next block's pass 3
          RK_CUDA_TRY(cudaEventRecord(hio->oev[k], st));
          RK_CUDA_TRY(cudaStreamWaitEvent(hio->copy, hio->oev[k], 0));
          cq = hio->copy;
        }
        RK_CUDA_TRY(cudaMemcpyAsync(hio->out_host + (int64_t)r0 * ia.ldo, ck.out,
                                    sizeof(double) * (size_t)(r1 - r0) * ia.ldo, cudaMemcpyDeviceToHost, cq));
      }
    }
    if (hio->out_host && hio->copy) {
      RK_CUDA_TRY(cudaEventRecord(hio->join, hio->copy));
      RK_CUDA_TRY(cudaStreamWaitEvent(st, hio->join, 0));
    }
  }
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[4], st));
  if (own) {
    scratch_free(T, st);
    scratch_free(U, st);
  }
  if (ac_owned) scratch_free(ac_owned, st);
  return Status::ok();
}

int chunk_rows(int nrows, int chunks) {
  const int per = (int)ceil_div(nrows, std::max(chunks, 1));
  return std::max(2, per + (per & 1));
}

Status predict_batch(const rk_setup* s, const PredictBatch& pb, cudaStream_t st, cudaEvent_t* ev,
                     Workspace* ws, const HostIo* hio) {
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
  if (ev) RK_CUDA_TRY(cudaEventRecord(ev[0], st));
  if (fused_gather(s)) {   // c* is formed in shared memory per row pair inside pass 1
    const SparseSrc sp = sparse_src(s, pb.c, pb.c_stride);
    return conv_pipeline(s, nullptr, s->M1, 0, pb.batch, s->grid.pad[2], s->m2, s->grid.pad[0], s->m1, e, st,
                         ev, ws, hio, &sp);
  }
  // very dense row pairs: standalone scatter kernel, c* through HBM
  const int64_t ldc = round_even(s->M1);
  double* cstar = nullptr;
  RK_TRY(scratch_alloc((void**)&cstar, sizeof(double) * (size_t)ldc * s->M2 * pb.batch, st));
  RK_TRY(launch_cstar(s, pb.c, pb.c_stride, cstar, ldc, pb.batch, st));
  Status r = conv_pipeline(s, cstar, ldc, ldc * s->M2, pb.batch, s->grid.pad[2], s->m2, s->grid.pad[0], s->m1,
                           e, st, ev, ws, hio);
  scratch_free(cstar, st);
  return r;
}

// ------------------------------------------------- persistent workspace + graph replay
static void free_ws(Workspace* w) {
  if (!w) return;
  for (auto& g : w->graphs) cudaGraphExecDestroy(g.second);
  for (auto& g : w->hgraphs) cudaGraphExecDestroy(g.second);
  if (w->aux) cudaStreamDestroy(w->aux);
  if (w->aux2) cudaStreamDestroy(w->aux2);
  if (w->ac_fork) cudaEventDestroy(w->ac_fork);
  if (w->ac_join) cudaEventDestroy(w->ac_join);
  if (w->fork) cudaEventDestroy(w->fork);
  if (w->join) cudaEventDestroy(w->join);
  cudaFree(w->ac_buf);
  for (auto& e : w->oev)
    if (e) cudaEventDestroy(e);
  for (auto& e : w->xev)
    if (e) cudaEventDestroy(e);
  cudaFreeHost(w->cb_h);
  cudaFree(w->T);
  cudaFree(w->U);
  cudaFree(w->c_in);   // beta_in lives in the same allocation
  cudaFree(w->xg_in);
  cudaFree(w->out);
  if (w->cap) cudaStreamDestroy(w->cap);
  delete w;
}

// at most this many per-stream workspaces per setup: a caller cycling through streams evicts
// the least recently created one (after a device synchronisation, since its stream may be
// gone) instead of growing without bound
static constexpr size_t kMaxWorkspaces = 8;

static Status get_ws(rk_setup* s, cudaStream_t st, Workspace** out) {
  std::lock_guard<std::mutex> lk(s->ws_mu);
  auto it = s->ws.find(st);
  if (it != s->ws.end()) {
    *out = it->second;
    return Status::ok();
  }
  if (s->ws.size() >= kMaxWorkspaces) {
    auto victim = s->ws.begin();
    for (auto jt = s->ws.begin(); jt != s->ws.end(); ++jt)
      if (jt->second->serial < victim->second->serial) victim = jt;
    RK_CUDA_TRY(cudaDeviceSynchronize());
    free_ws(victim->second);
    s->ws.erase(victim);
  }
  std::unique_ptr<Workspace, void (*)(Workspace*)> w(new Workspace(), free_ws);   // freed on any failure below
  static uint64_t serial = 0;
  w->serial = ++serial;
  const int64_t ldT = round_even(s->M2), ldU = round_even(s->m2);
  RK_CUDA_TRY(cudaMalloc(&w->T, sizeof(double2) * (size_t)s->H1 * ldT));
  RK_CUDA_TRY(cudaMalloc(&w->U, sizeof(double2) * (size_t)(s->H1 + 1) * ldU));   // either U layout
  // c and beta staged back to back (one upload per host-path call): beta at an even offset
  const int64_t boff = (std::max<int64_t>(s->n, 2) + 1) & ~int64_t(1);
  RK_CUDA_TRY(cudaMalloc(&w->c_in, sizeof(double) * (boff + 16)));
  w->beta_in = w->c_in + boff;
  RK_CUDA_TRY(cudaMalloc(&w->out, sizeof(double) * (size_t)s->m1 * s->m2));
  RK_CUDA_TRY(cudaStreamCreateWithFlags(&w->cap, cudaStreamNonBlocking));
  RK_CUDA_TRY(cudaStreamCreateWithFlags(&w->aux, cudaStreamNonBlocking));
  RK_CUDA_TRY(cudaStreamCreateWithFlags(&w->aux2, cudaStreamNonBlocking));
  RK_CUDA_TRY(cudaEventCreateWithFlags(&w->ac_fork, cudaEventDisableTiming));
  RK_CUDA_TRY(cudaEventCreateWithFlags(&w->ac_join, cudaEventDisableTiming));
  RK_CUDA_TRY(cudaEventCreateWithFlags(&w->fork, cudaEventDisableTiming));
  for (auto& e : w->xev) RK_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  for (auto& e : w->oev) RK_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  RK_CUDA_TRY(cudaEventCreateWithFlags(&w->join, cudaEventDisableTiming));
  RK_CUDA_TRY(cudaMallocHost(&w->cb_h, sizeof(double) * (boff + 16)));
  *out = w.get();
  s->ws[st] = w.release();
  return Status::ok();
}

void free_workspaces(rk_setup* s) {
  if (s->host_st) {
    cudaStreamDestroy(s->host_st);
    s->host_st = nullptr;
  }
  for (auto& kv : s->ws) free_ws(kv.second);
  s->ws.clear();
}

// graph bookkeeping per workspace stays bounded: pointer sets seen once are forgotten in bulk
static constexpr size_t kMaxSeen = 256;

// Predict of one field through the workspace: direct launches the first time a pointer
// set is seen, a CUDA graph (captured on the workspace's private stream, replayed on
// `st`) from the second time on.
// kernels in one graphed predict: gather + row FFT, column filter, row IFFT + epilogue
static constexpr int kPredictKernels = 3;

static Status predict_graphed(rk_setup* s, Workspace* w, const PredictBatch& pb, cudaStream_t st) {
  const GraphKey key{(uintptr_t)pb.c, (uintptr_t)pb.beta, (uintptr_t)pb.xg, (uintptr_t)pb.out, pb.p};
  cudaGraphExec_t exec = nullptr;
  bool capture = false;
  {
    std::lock_guard<std::mutex> lk(s->ws_mu);
    auto it = w->graphs.find(key);
    if (it != w->graphs.end()) exec = it->second;
    else {
      if (w->seen.size() >= kMaxSeen) w->seen.clear();
      capture = (++w->seen[key] >= 2) && w->graphs.size() < 64;
    }
  }
  static const bool use_graph = !(getenv("RK_DEV_GRAPH") && atoi(getenv("RK_DEV_GRAPH")) == 0);
  if (!use_graph) return predict_batch(s, pb, st, nullptr, w);
  if (exec) {
    RK_CUDA_TRY(cudaGraphLaunch(exec, st));
    count_launch(kPredictKernels);
    return Status::ok();
  }
  if (!capture) return predict_batch(s, pb, st, nullptr, w);
  cudaGraph_t g = nullptr;
  RK_CUDA_TRY(cudaStreamBeginCapture(w->cap, cudaStreamCaptureModeThreadLocal));
  Status r = predict_batch(s, pb, w->cap, nullptr, w);
  const cudaError_t ec = cudaStreamEndCapture(w->cap, &g);
  count_launch(-kPredictKernels);   // captured, not executed
  if (!r.good()) {
    if (g) cudaGraphDestroy(g);
    return r;
  }
  RK_CUDA_TRY(ec);
  RK_CUDA_TRY(cudaGraphInstantiate(&exec, g, 0));
  cudaGraphDestroy(g);
  {
    std::lock_guard<std::mutex> lk(s->ws_mu);
    w->graphs[key] = exec;
  }
  RK_CUDA_TRY(cudaGraphLaunch(exec, st));
  count_launch(kPredictKernels);
  return Status::ok();
}

}  // namespace rk

using namespace rk;

static bool is_pinned(const void* p) {
  cudaPointerAttributes at{};
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeHost;
}

static int finish_status(const Status& s) {
  if (!s.good()) rk::set_error(s.code, s.msg);
  return s.code;
}

extern "C" {

// diagnostics: copies the 3 x 4096 x 8 phase timestamps (RK_PHASE_TIMING builds only)
rk_status rk_phase_timestamps(unsigned long long* out) {
#ifdef RK_PHASE_TIMING
  if (cudaMemcpyFromSymbol(out, g_phase_ts, sizeof(g_phase_ts)) != cudaSuccess) return RK_CUDA;
  static const unsigned long long zero[3 * 4096 * 8] = {};   // next read shows only new launches
  return cudaMemcpyToSymbol(g_phase_ts, zero, sizeof(zero)) == cudaSuccess ? RK_OK : RK_CUDA;
#else
  (void)out;
  rk::set_error(RK_INTERNAL, "library built without RK_PHASE_TIMING");
  return RK_INTERNAL;
#endif
}

rk_status rk_coefficients_to_grid(const rk_setup* s, const double* c_dev, double* cstar_dev,
                                  void* stream) {
  return (rk_status)finish_status(launch_cstar(s, c_dev, 0, cstar_dev, s->M1, 1, (cudaStream_t)stream));
}

rk_status rk_convolve_filter(const rk_setup* s, const double* values_dev, double* out_dev,
                             void* stream) {
  auto run = [&]() -> Status {
    RowInvArgs e{};
    e.out = out_dev;
    e.ldo = s->M1;
    e.epi = EPI_PLAIN;
    const cudaStream_t st = (cudaStream_t)stream;
    if (s->p1 == s->rp1 && s->p2 == s->rp2)
      return conv_pipeline(s, values_dev, s->M1, 0, 1, 0, s->M2, 0, s->M1, e, st);
    // the setup executes on a smaller torus (interior outputs only): convolve_filter's whole
    // padded output runs on the reference's torus, its spectrum built here (rapid.py:89-100)
    rk_setup t;
    t.M1 = s->M1;
    t.M2 = s->M2;
    t.p1 = t.rp1 = s->rp1;
    t.p2 = t.rp2 = s->rp2;
    t.H1 = t.p1 / 2 + 1;
    t.Q2 = quarter_ld(t.p2);
    RK_TRY(scratch_alloc((void**)&t.spec_q, sizeof(double) * (size_t)t.H1 * t.Q2, st));
    Status r = spectrum_quarter(s->mat, s->grid.hx, s->grid.hy, t.p1, t.p2, 1.0 / ((double)t.p1 * (double)t.p2),
                                t.spec_q, t.Q2, st);
    if (r.good()) r = setup_plans(&t);
    if (r.good()) r = conv_pipeline(&t, values_dev, s->M1, 0, 1, 0, s->M2, 0, s->M1, e, st);
    scratch_free(t.spec_q, st);
    t.spec_q = nullptr;
    return r;
  };
  return (rk_status)finish_status(run());
}

rk_status rk_convolve_spectrum(const double* spec_q_dev, int32_t p1, int32_t p2,
                               const double* values_dev, int32_t M1, int32_t M2, double* out_dev,
                               void* stream) {
  auto run = [&]() -> Status {
    if (p1 < 2 * M1 - 2 || p2 < 2 * M2 - 2)
      return Status::err(RK_DOMAIN, "embedding dims too small for the padded grid");
    if (reinterpret_cast<uintptr_t>(spec_q_dev) & 15)
      return Status::err(RK_DOMAIN, "quarter spectrum must be 16-byte aligned");
    rk_setup t;   // descriptor only: the pipeline reads plans, dims and the spectrum
    t.M1 = M1;
    t.M2 = M2;
    t.p1 = p1;
    t.p2 = p2;
    t.H1 = p1 / 2 + 1;
    t.Q2 = quarter_ld(p2);
    t.spec_q = const_cast<double*>(spec_q_dev);
    RK_TRY(setup_plans(&t));
    RowInvArgs e{};
    e.out = out_dev;
    e.ldo = M1;
    e.epi = EPI_PLAIN;
    Status st = conv_pipeline(&t, values_dev, M1, 0, 1, 0, M2, 0, M1, e, (cudaStream_t)stream);
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
    rk_setup* ms = const_cast<rk_setup*>(s);
    Workspace* w = nullptr;
    RK_TRY(get_ws(ms, (cudaStream_t)stream, &w));
    return predict_graphed(ms, w, pb, (cudaStream_t)stream);
  };
  return (rk_status)finish_status(run());
}

rk_status rk_predict_profile(const rk_setup* s, const double* c_dev, const double* beta_dev,
                             int32_t p, const double* xg_dev, double* out_dev, void* stream,
                             float* ms_out) {
  auto run = [&]() -> Status {
    cudaStream_t st = (cudaStream_t)stream;
    cudaEvent_t ev[5];
    for (int i = 0; i < 5; ++i) RK_CUDA_TRY(cudaEventCreate(&ev[i]));
    PredictBatch pb;
    pb.batch = 1;
    pb.c = c_dev;
    pb.c_stride = s->n;
    pb.beta = beta_dev;
    pb.p = p;
    pb.xg = xg_dev;
    pb.out = out_dev;
    Workspace* w = nullptr;
    RK_TRY(get_ws(const_cast<rk_setup*>(s), st, &w));
    Status r = predict_batch(s, pb, st, ev, w);
    if (r.good()) {
      RK_CUDA_TRY(cudaEventSynchronize(ev[4]));
      for (int i = 0; i < 4; ++i) RK_CUDA_TRY(cudaEventElapsedTime(&ms_out[i], ev[i], ev[i + 1]));
    }
    for (int i = 0; i < 5; ++i) cudaEventDestroy(ev[i]);
    return r;
  };
  return (rk_status)finish_status(run());
}

rk_status rk_predict_traffic(const rk_setup* s, int32_t p, double* b) {
  // the scatter is fused into pass 1, so entry 0 is empty.  pass 1: weights (8 n M), plan
  // indices (8 n M: wsort index + observation index), c (8 n), node lists (8 nnodes + 4 M2),
  // T write (16 H1 M2); pass 2: T read, quarter spectrum (8 H1 (p2/2+1)), U write (16 H1 m2);
  // pass 3: U read, covariates (8 N p), field write (8 N)
  const double n = (double)s->n, M = (double)s->M;
  const double N = (double)s->m1 * s->m2, H = (double)s->H1;
  b[0] = 0.0;
  b[1] = n * M * 16.0 + 8.0 * n + 8.0 * (double)s->nnodes + 4.0 * s->M2 + 16.0 * H * s->M2;
  b[2] = 16.0 * H * s->M2 + 8.0 * H * (s->p2 / 2 + 1) + 16.0 * H * s->m2;
  b[3] = 16.0 * H * s->m2 + 8.0 * N * (double)p + 8.0 * N;
  return RK_OK;
}

rk_status rk_predict_host(const rk_setup* s, const double* c, const double* beta, int32_t p,
                          const double* xg, double* out, void* stream) {
  rk_setup* hs = const_cast<rk_setup*>(s);
  std::unique_lock<std::mutex> host_lock(hs->host_mu, std::defer_lock);
  auto run = [&]() -> Status {
    cudaStream_t st = (cudaStream_t)stream;
    if (!st) {   // no caller stream: the setup's own non-blocking stream, one call at a time
      host_lock.lock();
      if (!hs->host_st) RK_CUDA_TRY(cudaStreamCreateWithFlags(&hs->host_st, cudaStreamNonBlocking));
      st = hs->host_st;
    }
    if (beta && !xg && p != 1)
      return Status::err(RK_DOMAIN, "grid covariates are required when beta_hat has more than one entry");
    if (p > 16) return Status::err(RK_DOMAIN, "at most 16 covariates");
    rk_setup* ms = const_cast<rk_setup*>(s);
    Workspace* w = nullptr;
    RK_TRY(get_ws(ms, st, &w));
    const int64_t N = (int64_t)s->m1 * s->m2;
    if (xg && w->xg_cap < (size_t)(N * p)) {
      std::lock_guard<std::mutex> lk(ms->ws_mu);
      RK_CUDA_TRY(cudaStreamSynchronize(st));
      cudaFree(w->xg_in);
      for (auto& g : w->graphs) cudaGraphExecDestroy(g.second);   // keys held the old pointer
      for (auto& g : w->hgraphs) cudaGraphExecDestroy(g.second);
      w->graphs.clear();
      w->seen.clear();
      w->hgraphs.clear();
      w->hseen.clear();
      w->xg_in = nullptr;
      RK_CUDA_TRY(cudaMalloc(&w->xg_in, sizeof(double) * N * p));
      w->xg_cap = (size_t)(N * p);
    }
    PredictBatch pb;
    pb.batch = 1;
    pb.c = w->c_in;
    pb.c_stride = s->n;
    pb.beta = beta ? w->beta_in : nullptr;
    pb.p = p;
    pb.xg = xg ? w->xg_in : nullptr;
    pb.out = w->out;
    if (!(is_pinned(c) && is_pinned(out) && (!xg || is_pinned(xg)))) {
      // pageable buffers: plain staged copies around the graphed device predict
      RK_CUDA_TRY(cudaMemcpyAsync(w->c_in, c, sizeof(double) * s->n, cudaMemcpyHostToDevice, st));
      if (beta) RK_CUDA_TRY(cudaMemcpyAsync(w->beta_in, beta, sizeof(double) * p, cudaMemcpyHostToDevice, st));
      if (xg) RK_CUDA_TRY(cudaMemcpyAsync(w->xg_in, xg, sizeof(double) * N * p, cudaMemcpyHostToDevice, st));
      RK_TRY(predict_graphed(ms, w, pb, st));
      RK_CUDA_TRY(cudaMemcpyAsync(out, w->out, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
      RK_CUDA_TRY(cudaStreamSynchronize(st));
      return Status::ok();
    }
    // pinned buffers: uploads, kernels and downloads in one graph; X_g rows go up on the
    // side stream in row blocks that pass 3 consumes as they land
    // c and beta into one pinned staging block (the previous call has completed)
    const int64_t boff = w->beta_in - w->c_in;
    memcpy(w->cb_h, c, sizeof(double) * s->n);
    if (beta) memcpy(w->cb_h + boff, beta, sizeof(double) * p);
    const size_t cb_bytes = sizeof(double) * (size_t)(beta ? boff + p : s->n);
    // one block by default: on B200 (cfg2, 2.9 MB of X_g) the single side-stream upload
    // hidden behind the gather / FFT passes measured 114 us per call; 2 / 4 / 8 row blocks
    // 294 / 169 / 279 us (the interleaved small copies serialise on the copy engines)
    // Large fields (>= 16 MB) instead go through device memory, pass 3 in 4 row blocks, each
    // block's device -> host copy on the side stream overlapping the next block (measured on
    // cfg5's 134 MB field: 3.51 ms per call vs 3.61-4.04 ms zero-copy, whose kernel-issued PCIe
    // writes vary from box to box; the DMA copies run at ~56 GB/s).
    const bool big = (double)N * 8.0 >= 16.0e6;
    static const int k_env = getenv("RK_HOST_CHUNKS") ? atoi(getenv("RK_HOST_CHUNKS")) : -1;
    static const int graph_env = getenv("RK_HOST_GRAPH") ? atoi(getenv("RK_HOST_GRAPH")) : 1;
    const int K = std::max(1, std::min(k_env >= 0 ? k_env : (big ? 4 : 1), Workspace::kMaxChunks));
    // small fields: pass 3 writes the field straight into the pinned output through its device
    // mapping, the device -> host traffic overlapping the last pass instead of following it
    static const int zc_env = getenv("RK_HOST_ZEROCOPY") ? atoi(getenv("RK_HOST_ZEROCOPY")) : -1;
    const bool zc = zc_env >= 0 ? zc_env != 0 : !big;
    double* out_map = nullptr;
    if (zc && cudaHostGetDevicePointer((void**)&out_map, out, 0) != cudaSuccess) {
      cudaGetLastError();
      out_map = nullptr;
    }
    if (out_map) pb.out = out_map;
    auto enqueue = [&](cudaStream_t q) -> Status {
      HostIo hio;
      hio.chunks = K;
      hio.out_host = out_map ? nullptr : out;
      if (!out_map && K > 1) {   // field copies on the side stream, overlapped with pass 3
        hio.copy = w->aux;
        hio.oev = w->oev;
        hio.join = w->join;
      }
      if (xg) {   // fork first: the X_g upload starts before anything else
        RK_CUDA_TRY(cudaEventRecord(w->fork, q));
        RK_CUDA_TRY(cudaStreamWaitEvent(w->aux, w->fork, 0));
        const int per = chunk_rows(s->m2, K);
        for (int k = 0, r0 = 0; r0 < s->m2; ++k, r0 += per) {
          const int r1 = std::min(s->m2, r0 + per);
          const size_t off = (size_t)r0 * s->m1 * p;
          RK_CUDA_TRY(cudaMemcpyAsync(w->xg_in + off, xg + off, sizeof(double) * (size_t)(r1 - r0) * s->m1 * p,
                                      cudaMemcpyHostToDevice, w->aux));
          RK_CUDA_TRY(cudaEventRecord(w->xev[k], w->aux));
        }
        hio.xev = w->xev;
      }
      RK_CUDA_TRY(cudaMemcpyAsync(w->c_in, w->cb_h, cb_bytes, cudaMemcpyHostToDevice, q));
      return predict_batch(s, pb, q, nullptr, w, &hio);
    };
    const GraphKey key{(uintptr_t)c, (uintptr_t)(beta ? 1 : 0), (uintptr_t)xg, (uintptr_t)out, p};
    cudaGraphExec_t exec = nullptr;
    bool capture = false;
    {
      std::lock_guard<std::mutex> lk(ms->ws_mu);
      auto it = w->hgraphs.find(key);
      if (it != w->hgraphs.end()) exec = it->second;
      else {
        if (w->hseen.size() >= kMaxSeen) w->hseen.clear();
        capture = graph_env && (++w->hseen[key] >= 2) && w->hgraphs.size() < 64;
      }
    }
    const int nk = kPredictKernels + (K - 1);
    if (!exec && !capture) {
      RK_TRY(enqueue(st));
    } else {
      if (!exec) {
        cudaGraph_t g = nullptr;
        RK_CUDA_TRY(cudaStreamBeginCapture(w->cap, cudaStreamCaptureModeThreadLocal));
        const int64_t l0 = rk_launch_count();
        Status r = enqueue(w->cap);
        const cudaError_t ec = cudaStreamEndCapture(w->cap, &g);
        count_launch((int)(l0 - rk_launch_count()));   // captured, not executed
        if (!r.good()) {
          if (g) cudaGraphDestroy(g);
          return r;
        }
        RK_CUDA_TRY(ec);
        RK_CUDA_TRY(cudaGraphInstantiate(&exec, g, 0));
        cudaGraphDestroy(g);
        std::lock_guard<std::mutex> lk(ms->ws_mu);
        w->hgraphs[key] = exec;
      }
      RK_CUDA_TRY(cudaGraphLaunch(exec, st));
      count_launch(nk);
    }
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    return Status::ok();
  };
  return (rk_status)finish_status(run());
}

}  // extern "C"
