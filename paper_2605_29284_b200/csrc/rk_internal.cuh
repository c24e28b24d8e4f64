// Internal structures shared by the rapidkrig B200 translation units.
#pragma once

#include <map>
#include <mutex>
#include <vector>

#include "rk_common.cuh"
#include "rk_fft.cuh"
#include "rk_fft_ct.cuh"
#include "rk_matern.cuh"

namespace rk {

// --------------------------------------------------------------- bookkeeping
void count_launch(int k = 1);
Status plan_for(int n, FftPlan* out, int wide = 0);   // cached per (device, n, wide)
// the plan variants of one length: v[0] normal, v[1] spread, v[2] wide, v[3] split radix-9
// (n == 0 if absent)
struct PlanSet {
  FftPlan v[4] = {};
};
// w_P^n = hi[n >> 7] * lo[n & 127] for 0 <= n < P / 2 (split-length passes, rk_predict.cu)
struct SplitTw {
  const double2* lo = nullptr;   // 128 entries
  const double2* hi = nullptr;   // nhi entries
  int nhi = 0;
  int off = 0;                   // smem offset (double2 units) where a kernel stages them
};
Status split_table(int P, SplitTw* out);   // cached per (device, P)
Status ct_plan_for(int n, int G, CtPlan* out);   // cached per (device, n, G); rk_fft_ct.cuh
__device__ __forceinline__ const double2* stage_split_tw(const SplitTw& t, double2* dst) {
  for (int i = threadIdx.x; i < 128 + t.nhi; i += blockDim.x) dst[i] = i < 128 ? __ldg(&t.lo[i]) : __ldg(&t.hi[i - 128]);
  return dst;
}
__device__ __forceinline__ double2 split_w(const double2* tw, int n) {   // w_P^n (staged tables)
  return cmul(tw[128 + (n >> 7)], tw[n & 127]);
}
Status plan_set(int n, PlanSet* out);
// spread while the launch's CTAs are all resident at once (latency-bound small grids), else
// wide (64-register kernels, twice the resident warps), else normal
const FftPlan& plan_pick(const PlanSet& ps, int64_t lines);
// lines per CTA for a kernel: pack up to max_lines, but only while the launch still has
// >= 2 CTAs per SM for `total_lines` lines (small grids are latency bound, not occupancy)
int pick_lpc(const FftPlan& pl, int max_lines, int64_t total_lines = (int64_t)1 << 40);
Status set_smem_attr(const void* fn, size_t bytes);

// RAII-free stream-ordered scratch (cudaMallocAsync pool)
Status scratch_alloc(void** p, size_t bytes, cudaStream_t st);
void scratch_free(void* p, cudaStream_t st);

// ------------------------------------------------------------------- setup
// Execution torus smaller than the reference's (rk_core.cu choose_exec_torus): the convolution runs
// on a torus whose half length covers every interior-output lag but a band of a few lags; the
// pairs (input row u, output row y) and (input column v, output column x) whose lag falls in that
// band are corrected exactly by one-dimensional convolutions of the outer input rows / columns
// of c* ("strips") with kernel differences (rk_predict.cu, alias_corrections).
constexpr int kAcMax = 16;
constexpr int kSplitFold = 16;   // input rows beyond the half the split column pass folds in
struct AliasCorr {
  int nrp = 0, ncp = 0;                    // row pairs, column pairs
  int rp_strip[kAcMax] = {}, rp_out[kAcMax] = {}, rp_ker[kAcMax] = {};   // strip, interior output row, kernel
  int cp_strip[kAcMax] = {}, cp_out[kAcMax] = {}, cp_ker[kAcMax] = {};   // strip, interior output column, kernel
  int nru = 0, ncv = 0;                    // strips: padded input rows ru[], padded input columns cv[]
  int ru[kAcMax] = {}, cv[kAcMax] = {};
  int nkr = 0, nkc = 0;                    // kernels: row pairs' (2 M1 - 1 each), then columns' (2 M2 - 1)
  int row_lo = 0, row_hi = 0;              // interior rows < row_lo or >= row_hi may carry row corrections
  int col_lo = 0, col_hi = 0;              // same for columns
};

struct Embedding {
  bool ready = false;
  int ps1 = 0, ps2 = 0, doubled = 0;
  int hs1 = 0, qs2 = 0;          // ps1/2+1, ps2/2+1
  FftPlan pl1{}, pl2{};
  PlanSet ps1v, ps2v;            // all plan variants of ps1 / ps2
  PlanSet hs1v, hs2v;            // half-length plans of split-length passes (n = 0 if unused)
  SplitTw sws1, sws2;            // w_P^n tables for P = ps1, ps2
  double* root_q = nullptr;      // (qs2, hs1) row-major: sqrt(clip(lambda,0)) * sqrt(P)/P
};

// Per-(setup, stream) persistent predict workspace: intermediate buffers for one
// field, staging buffers for the host-buffer path, and a cache of instantiated CUDA
// graphs of the 4-kernel predict keyed by the caller's pointers.
struct GraphKey {
  uintptr_t c, beta, xg, out;
  int p;
  bool operator<(const GraphKey& o) const {
    if (c != o.c) return c < o.c;
    if (beta != o.beta) return beta < o.beta;
    if (xg != o.xg) return xg < o.xg;
    if (out != o.out) return out < o.out;
    return p < o.p;
  }
};

struct Workspace {
  uint64_t serial = 0;          // creation order (eviction of the oldest, rk_predict.cu get_ws)
  double2* T = nullptr;         // (H1, ldT)
  double2* U = nullptr;         // (H1, ldU)
  double* c_in = nullptr;       // host-path staging: c, then beta at an even offset
  double* beta_in = nullptr;    // (inside the c_in allocation)
  double* xg_in = nullptr;
  size_t xg_cap = 0;
  double* out = nullptr;
  cudaStream_t cap = nullptr;   // private stream used only for graph capture
  std::map<GraphKey, cudaGraphExec_t> graphs;
  std::map<GraphKey, int> seen;
  // host-buffer path: X_g upload on a side stream, chunk by chunk, overlapped with the
  // gather / FFT passes; graphs keyed by the (pinned) host pointers
  static constexpr int kMaxChunks = 8;
  cudaStream_t aux = nullptr;
  cudaEvent_t fork = nullptr;
  cudaEvent_t xev[kMaxChunks] = {};
  cudaEvent_t oev[kMaxChunks] = {};   // field row block k computed (its copy may start)
  double* ac_buf = nullptr;           // aliased-lag corrections: strips, partial sums, corrections (batch 1)
  size_t ac_cap = 0;
  cudaStream_t aux2 = nullptr;        // the corrections run here, beside passes 1 and 2 (they only read c)
  cudaEvent_t ac_fork = nullptr, ac_join = nullptr;
  cudaEvent_t join = nullptr;         // the side stream's last field copy issued
  double* cb_h = nullptr;       // pinned staging of c and beta (beta at beta_in - c_in)
  std::map<GraphKey, cudaGraphExec_t> hgraphs;
  std::map<GraphKey, int> hseen;
};

// Host-buffer predict: pass 3 runs in `chunks` row blocks; block k waits for xev[k] (its
// covariate rows uploaded on the side stream) and its field rows are copied to out_host
// right after it, so PCIe traffic in both directions overlaps the kernels.
struct HostIo {
  int chunks = 1;
  const cudaEvent_t* xev = nullptr;
  double* out_host = nullptr;
  // with a copy stream: block k's device -> host copy runs there (after oev[k]) while block k + 1
  // is computed; the launching stream waits on `join` after the last block
  cudaStream_t copy = nullptr;
  const cudaEvent_t* oev = nullptr;
  cudaEvent_t join = nullptr;
};
int chunk_rows(int nrows, int chunks);   // rows per block (even)

}  // namespace rk

struct rk_setup {
  int device = 0;
  rk_model model{};
  rk::MaternDev mat{};
  rk_grid grid{};
  int L = 0, bs = 0, M = 0;      // bs = 2L, M = bs^2
  int64_t n = 0;
  int M1 = 0, M2 = 0, m1 = 0, m2 = 0;
  double px0 = 0, py0 = 0;
  int p1 = 0, p2 = 0, H1 = 0, Q2 = 0;   // the EXECUTION torus (and its half / quarter sizes)
  int rp1 = 0, rp2 = 0;                 // the reference's torus (rapid.py:72-86): embed_dims, filter_spectrum
  rk::AliasCorr ac;                     // corrections when (p1, p2) != (rp1, rp2)
  double* ac_ker = nullptr;             // device: the correction kernels (AliasCorr)
  rk::FftPlan pl1{}, pl2{};
  rk::PlanSet pl1v, pl2v;       // all plan variants of p1 / p2, see plan_pick
  rk::PlanSet h1v, h2v;         // plan variants of p1 / 2, p2 / 2 (split-length passes; n = 0 if unused)
  rk::SplitTw sw1, sw2;         // w_P^n tables for P = p1, p2
  // device arrays
  double* obs = nullptr;        // (n, 2)
  int32_t* base = nullptr;      // (n) flat padded index of block entry 0
  double* weights = nullptr;    // (n, M) original order
  double* cond_var = nullptr;   // (n)
  int32_t* perm = nullptr;      // sorted -> original
  int32_t* bsort = nullptr;     // sorted base keys
  double* wsort = nullptr;      // (n, M) sorted order
  int32_t* cell_start = nullptr;  // (M1*M2 + 1) lower bounds of base keys
  // sparse gather plan (fixed per observation layout): active padded nodes, each with its
  // contributions (index into wsort, original obs index) in the order dy asc, sorted j asc
  int64_t nnodes = 0;
  int32_t* node_q = nullptr;      // (nnodes) flat padded node index, ascending
  int32_t* node_off = nullptr;    // (nnodes + 1) offsets into ent_w / ent_c
  int32_t* row_node = nullptr;    // (M2 + 1) first active node of each padded row
  int32_t* ent_w = nullptr;       // (n M) index into wsort
  int32_t* ent_c = nullptr;       // (n M) original observation index (into c)
  int64_t max_pair_ent = 0;       // most contributions of one row pair (2k, 2k+1)
  int64_t max_half_ent = 0;       // most contributions of half a row pair's nodes (split pass 1)
  double* ent_wv = nullptr;       // (n M) weight of each contribution (wsort[ent_w])
  int4* pair_info = nullptr;      // (ceil(M2/2) + 1) {node0, node of row 2p+1, contribution0, 0}
  // per-row-pair plan blocks at a fixed stride (small plans only): {count, nodes, 0, 0}, then
  // node records int2 {end of its products, 2 x + odd row} [cap], weights double [cap],
  // observation indices int [cap] -- pass 1 fetches a pair's whole plan in one bulk copy
  unsigned char* pblk = nullptr;
  int64_t pblk_stride = 0;        // bytes (multiple of 16)
  int pblk_cap = 0;
  double* spec_q = nullptr;     // (H1, Q2): Re fft2(filter)[ky, kx] / (p1 p2), ky <= p2/2
  double* spec_s = nullptr;     // split-length column pass: (H1, 2, ldh) spec_q[kx][2 j + h], j <= p2/4
  int ldh = 0;
  double* kn_chol_dev = nullptr;  // (M, M) row-major lower
  std::vector<double> kn_chol, kn_inv;
  double cond_var_min = 0;
  rk::Embedding emb;
  std::mutex ws_mu;
  std::map<cudaStream_t, rk::Workspace*> ws;
  std::mutex host_mu;               // serialises host-buffer predicts on the library's own stream
  cudaStream_t host_st = nullptr;   // that stream (created on first use)
};

struct rk_fit {
  int device = 0;
  rk_model model{};
  int64_t n = 0;
  int p = 0;
  double* U = nullptr;          // (n, n) column-major UPPER factor = row-major lower L
  double* X = nullptr;          // (n, p) column-major
  double* B = nullptr;          // L^-1 X (n, p) column-major
  double* Uinv = nullptr;       // U^-1 = L^-T (n, n) column-major upper, built on first batched refit
  double* beta = nullptr;       // (p)
  double* c = nullptr;          // (n)
  double* obs = nullptr;        // (n, 2) observation locations (exact prediction at targets)
  rk::MaternDev mat{};
  std::vector<double> gram_lu;  // (p, p) LU of B'B with partial pivoting (row-major)
  std::vector<int> gram_piv;
  void* cublas = nullptr;                    // handle of the creating thread / default stream
  std::mutex blas_mu;
  std::map<cudaStream_t, void*> blas_by_stream;   // one handle per stream (own workspace)
  std::mutex uinv_mu;                             // serialises the lazy U^-1 build
};

namespace rk {

// all FFT plans of a setup from its p1 / p2: full lengths, half lengths + w_P tables where a
// split-length pass applies (rk_core.cu)
Status setup_plans(rk_setup* s);
// the parity-split spectrum of the split-length column pass (after spec_q is built)
Status build_spec_split(rk_setup* s, cudaStream_t st);
// the embedding's plans from its ps1 / ps2 (same rules)
Status embedding_plans(rk_setup* s);

// destructors (device-aware: free on the object's own device)
void free_setup(rk_setup* s);
void free_fit(rk_fit* f);

// predict pipeline pieces (rk_predict.cu), used by the ensemble driver
enum EpiMode { EPI_PLAIN = 0, EPI_SCALAR = 1, EPI_COV = 2 };

struct PredictBatch {
  int batch = 1;
  const double* c = nullptr;      // (batch, n)
  int64_t c_stride = 0;
  const double* beta = nullptr;   // (batch, p) or null
  int p = 0;
  const double* xg = nullptr;     // (m1*m2, p) or null
  const double* g = nullptr;      // CS: (batch, M2, M1) unconditional fields, or null
  double* out = nullptr;          // (batch, m2, m1): field, or e = interior(g) - field in CS mode
};
Status predict_batch(const rk_setup* s, const PredictBatch& pb, cudaStream_t st,
                     cudaEvent_t* ev = nullptr, Workspace* ws = nullptr, const HostIo* hio = nullptr);
void free_workspaces(rk_setup* s);

// CS pieces (rk_sim.cu)
Status ensure_embedding(rk_setup* s, cudaStream_t st);

// exact-Kriging pieces (rk_exact.cu) used by the ensemble driver
// batched refit: Z (n x batch, column-major) -> beta (p x batch), C (n x batch)
Status gls_batch(const rk_fit* f, const double* Z, int64_t batch, double* beta, double* C, cudaStream_t st);
Status ensure_uinv(rk_fit* f, cudaStream_t st);   // U^-1 for the batched refits, built once
// refit products with the inverse factor (rk_refit.cu): out = L^-1 X (trans = false) or
// L^-T X (trans = true), X / out (n x S) column-major; rhs (S, p) = (B' A) per column
Status trmm_linv(const rk_fit* f, bool trans, const double* X, int64_t ldx, int64_t S, double* out, int64_t ldo,
                 cudaStream_t st);
Status bta(const rk_fit* f, const double* A, int64_t lda, int64_t S, double* rhs, cudaStream_t st);

}  // namespace rk
