// rapidkrig B200: library infrastructure, padded grid, rapid setup.
//
// Reference mapping (/root/reference/pkg/src/rapidkrig):
//   build_padded_grid   gridding.py:130-178   -> rk_build_padded_grid / pad_kernel
//   neighborhood        gridding.py:181-205   -> weights_kernel (stencil part)
//   neighbor_cov        rapid.py:103-117      -> host kn_matrix (M x M, tiny)
//   _factor_neighbor_cov rapid.py:120-135     -> host cholesky_lower with ridge retry
//   build_setup         rapid.py:177-230      -> rk_build_setup (weights_kernel + sort +
//                                                spectrum_quarter)
#include <algorithm>
#include <tuple>
#include <atomic>
#include <climits>
#include <set>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "rk_internal.cuh"

namespace rk {

// ------------------------------------------------------------------ errors
namespace {
thread_local std::string g_err;
thread_local int g_code = RK_OK;
std::atomic<int64_t> g_launches{0};   // process-wide: ensemble shards launch from worker threads
}  // namespace

void set_error(int code, const std::string& msg) {
  g_code = code;
  g_err = msg;
}
int last_code() { return g_code; }
void count_launch(int k) { g_launches += k; }

static int finish(const Status& s) {
  if (!s.good()) set_error(s.code, s.msg);
  return s.code;
}

// ------------------------------------------------------------------- plans
namespace {
std::mutex g_plan_mu;
std::map<std::pair<int, int>, FftPlan> g_plans;   // (device, 4 n + variant)
std::map<std::pair<int, const void*>, bool> g_smem_set;
}  // namespace

Status plan_for(int n, FftPlan* out, int wide) {
  int dev = 0;
  RK_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_plan_mu);
  auto key = std::make_pair(dev, n * 4 + wide);
  auto it = g_plans.find(key);
  if (it != g_plans.end()) {
    *out = it->second;
    return Status::ok();
  }
  FftPlan pl{};
  if (!fft_factor(n, &pl, wide))
    return Status::err(RK_INTERNAL, "FFT length " + std::to_string(n) + " is not 2^a 3^b");
  if (pl.nthr > fft_sm_threads(wide))
    return Status::err(RK_DOMAIN, "FFT length " + std::to_string(n) + " too large for one CTA");
  std::vector<double2> tw;
  fft_stage_twiddles(pl, tw, [](double c, double s) { return make_double2(c, s); });
  pl.ntw = (int)tw.size();
  tw.push_back(make_double2(1.0, 0.0));   // never empty
  double2* d = nullptr;
  RK_CUDA_TRY(cudaMalloc(&d, sizeof(double2) * tw.size()));
  RK_CUDA_TRY(cudaMemcpy(d, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice));
  pl.tw = d;
  g_plans[key] = pl;
  *out = pl;
  return Status::ok();
}

Status plan_set(int n, PlanSet* out) {
  RK_TRY(plan_for(n, &out->v[0]));
  // the variants keep the stage twiddle table in smem next to the line: n <= 4608
  for (int w = 1; w <= 3; ++w)
    if (n > 4608 || !plan_for(n, &out->v[w], w).good()) out->v[w] = FftPlan{};
  if (out->v[3].n && out->v[3].n9 == 0) out->v[3] = FftPlan{};   // split needs radix-9 stages
  return Status::ok();
}

Status split_table(int P, SplitTw* out) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, SplitTw> cache;
  int dev = 0;
  RK_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, P});
  if (it != cache.end()) {
    *out = it->second;
    return Status::ok();
  }
  const int H = P / 2, nhi = (H + 127) / 128;
  std::vector<double2> t(128 + nhi);
  const long double PI_L = 3.141592653589793238462643383279502884L;
  for (int i = 0; i < 128 + nhi; ++i) {
    const long long e = i < 128 ? i : 128LL * (i - 128);
    const long double ang = 2.0L * PI_L * (long double)e / (long double)P;
    t[i] = make_double2((double)cosl(ang), (double)(-sinl(ang)));
  }
  double2* d = nullptr;
  RK_CUDA_TRY(cudaMalloc(&d, sizeof(double2) * t.size()));
  RK_CUDA_TRY(cudaMemcpy(d, t.data(), sizeof(double2) * t.size(), cudaMemcpyHostToDevice));
  SplitTw w;
  w.lo = d;
  w.hi = d + 128;
  w.nhi = nhi;
  cache[{dev, P}] = w;
  *out = w;
  return Status::ok();
}

// in-place Cooley-Tukey plan (rk_fft_ct.cuh) with its twiddle table on the device, cached per
// (device, n, group threads); G = 0 picks the plan's default group size
Status ct_plan_for(int n, int G, CtPlan* out) {
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, CtPlan> cache;
  int dev = 0;
  RK_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find({dev, n, G});
  if (it != cache.end()) {
    *out = it->second;
    return Status::ok();
  }
  CtPlan p{};
  if (!ct_plan_make(n, &p, 1024, G)) return Status::err(RK_INTERNAL, "no Cooley-Tukey plan for this length");
  std::vector<double2> t;
  ct_twiddles(p, t, [](double x, double y) { return make_double2(x, y); });
  double2* d = nullptr;
  if (!t.empty()) {
    RK_CUDA_TRY(cudaMalloc(&d, sizeof(double2) * t.size()));
    RK_CUDA_TRY(cudaMemcpy(d, t.data(), sizeof(double2) * t.size(), cudaMemcpyHostToDevice));
  }
  p.tw = d;
  cache[{dev, n, G}] = p;
  *out = p;
  return Status::ok();
}

// a length-P pass splits into two length-P/2 transforms when P is even and larger than the
// lengths with WIDE plans (the half has one), see rk_predict.cu
static bool split_len(int P) {
  static const bool allow = !(getenv("RK_SPLIT") && atoi(getenv("RK_SPLIT")) == 0);
  return allow && P % 2 == 0 && P > 4608 && P / 2 <= 4608;
}

Status setup_plans(rk_setup* s) {
  RK_TRY(plan_for(s->p1, &s->pl1));
  RK_TRY(plan_for(s->p2, &s->pl2));
  RK_TRY(plan_set(s->p1, &s->pl1v));
  RK_TRY(plan_set(s->p2, &s->pl2v));
  s->h1v = PlanSet{};
  s->h2v = PlanSet{};
  if (split_len(s->p1) && s->M1 <= s->p1 / 2) {
    RK_TRY(plan_set(s->p1 / 2, &s->h1v));
    RK_TRY(split_table(s->p1, &s->sw1));
  }
  // the column pass folds up to kSplitFold input rows beyond the half (execution torus)
  if (split_len(s->p2) && s->M2 <= s->p2 / 2 + kSplitFold) {
    RK_TRY(plan_set(s->p2 / 2, &s->h2v));
    RK_TRY(split_table(s->p2, &s->sw2));
  }
  return Status::ok();
}

// ----------------------------------------------------------------- execution torus
// The reference embeds the padded grid in the smallest 2^a 3^b torus >= 2 M - 1 per axis
// (rapid.py:72-86): 8748 for configs[4]'s M = 4102, radix 6 9 9 9 per half.  Interior outputs,
// though, only meet lags <= maxlag = max(pad + m - 1, M - 1 - pad) (4098), so along y the
// convolution runs on the smallest 2^a 3^b length P >= 2 (maxlag - kAcBand) -- 8192, radix
// 8 8 8 8 per half, ~20 % fewer FP64 instructions per point and 6 % fewer points -- and the few
// (input row u, output row y) pairs with |y - u| > P / 2, whose wrapped lag P - |y - u| differs
// from the true one, are corrected exactly afterwards (AliasCorr, rk_predict.cu).  The x axis
// keeps the reference length (no corrections there).  embed_dims / filter_spectrum /
// convolve_filter stay on the reference torus.
// Measured on B200 and OFF by default (RK_EXEC_TORUS=1 enables it): cfg5 step 1.263 -> 1.456 ms,
// cfg3 0.337 -> 0.387 ms.  The power-of-two half lines make every Stockham stage's shared-memory
// stride a power of two (bank conflicts the 3-smooth lengths avoid: the column pass falls from
// 7.5 to 4.3 TF/s), and the corrections cost ~0.07 ms.  Exact either way (all parity tests pass
// with it on); worth it only with a conflict-free power-of-two layout in the engine.
static constexpr int kAcBand = 4;

__global__ void ac_kernel_build(MaternDev P, double hx, double hy, int M1, int p2, AliasCorr ac, const int* dks,
                                double* out, int* bad) {
  // row kernels g_d(dx) = K(d, dx) - K(p2 - d, dx), dx = -(M1 - 1) .. M1 - 1 (d: a y lag)
  const int L1 = 2 * M1 - 1;
  const int64_t tot = (int64_t)ac.nkr * L1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(e / L1), dx = abs((int)(e % L1) - (M1 - 1));
    const int d = dks[k];
    // K(a_y, b_x) = sigma2 phi(alpha hypot(b_x hx, a_y hy)), as the spectrum's lag table (lagq_kernel)
    out[e] = matern_cov(P, hypot((double)dx * hx, (double)d * hy), bad) -
             matern_cov(P, hypot((double)dx * hx, (double)(p2 - d) * hy), bad);
  }
}

// y-axis execution length and corrections for setup s (s->rp2 set); returns the length
static int choose_exec_y(rk_setup* s) {
  static const bool on = getenv("RK_EXEC_TORUS") && atoi(getenv("RK_EXEC_TORUS")) == 1;
  const int rp = s->rp2;
  s->ac = AliasCorr{};
  if (!on || rp < 4096) return rp;
  const int lo = s->grid.pad[2], m = s->m2, M = s->M2;
  const int maxlag = std::max(lo + m - 1, M - 1 - lo);
  int64_t best = rp;
  for (int64_t two = 1; two < 2 * (int64_t)rp; two *= 2)
    for (int64_t v = two; v < rp; v *= 3) {
      if (v < 2 * (int64_t)(maxlag - kAcBand) || v < M) continue;
      if (split_len((int)v) && (M > v / 2 + kSplitFold || m > v / 2)) continue;   // column pass fold / combine
      best = std::min(best, v);
    }
  if (best >= rp) return rp;
  const int P = (int)best;
  AliasCorr ac;
  for (int u = 0; u < M; ++u)
    for (int yo = 0; yo < m; ++yo) {
      const int d = std::abs(lo + yo - u);
      if (2 * d <= P) continue;
      if (ac.nrp == kAcMax) return rp;   // too many pairs: keep the reference torus
      int su = 0, sk = 0;
      while (su < ac.nru && ac.ru[su] != u) ++su;
      if (su == ac.nru) {
        if (ac.nru == kAcMax) return rp;
        ac.ru[ac.nru++] = u;
      }
      // kernel slot: distinct lags d, kept in cp_ker as scratch (column pairs are unused)
      while (sk < ac.nkr && ac.cp_ker[sk] != d) ++sk;
      if (sk == ac.nkr) ac.cp_ker[ac.nkr++] = d;
      ac.rp_strip[ac.nrp] = su;
      ac.rp_out[ac.nrp] = yo;
      ac.rp_ker[ac.nrp] = sk;
      ++ac.nrp;
    }
  if (ac.nrp == 0) return P;
  ac.row_lo = 0;
  ac.row_hi = m;
  for (int k = 0; k < ac.nrp; ++k) {   // pairs sit at the edges: rows < row_lo or >= row_hi
    if (ac.rp_out[k] < m / 2) ac.row_lo = std::max(ac.row_lo, ac.rp_out[k] + 1);
    else ac.row_hi = std::min(ac.row_hi, ac.rp_out[k]);
  }
  s->ac = ac;
  return P;
}

static Status build_alias_kernels(rk_setup* s) {
  cudaFree(s->ac_ker);
  s->ac_ker = nullptr;
  if (s->ac.nrp == 0) return Status::ok();
  const int L1 = 2 * s->M1 - 1;
  int* dks = nullptr;
  int* bad = nullptr;
  RK_CUDA_TRY(cudaMalloc(&s->ac_ker, sizeof(double) * (size_t)s->ac.nkr * L1));
  RK_CUDA_TRY(cudaMalloc(&dks, sizeof(int) * kAcMax));
  RK_CUDA_TRY(cudaMalloc(&bad, sizeof(int)));
  RK_CUDA_TRY(cudaMemcpy(dks, s->ac.cp_ker, sizeof(int) * kAcMax, cudaMemcpyHostToDevice));
  RK_CUDA_TRY(cudaMemset(bad, 0, sizeof(int)));
  ac_kernel_build<<<(int)std::min<int64_t>(ceil_div((int64_t)s->ac.nkr * L1, 256), 148 * 8), 256>>>(
      s->mat, s->grid.hx, s->grid.hy, s->M1, s->p2, s->ac, dks, s->ac_ker, bad);
  count_launch();
  RK_LAUNCH_CHECK();
  int hb = 0;
  RK_CUDA_TRY(cudaMemcpy(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(dks);
  cudaFree(bad);
  if (hb) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");
  for (int k = 0; k < kAcMax; ++k) s->ac.cp_ker[k] = 0;   // scratch of choose_exec_y
  return Status::ok();
}

__global__ void spec_split_kernel(const double* __restrict__ q, int Q2, int H1, int H, int ldh,
                                  double* __restrict__ out) {
  const int64_t tot = (int64_t)H1 * 2 * ldh;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = (int)(e % ldh), h = (int)((e / ldh) % 2);
    const int64_t kx = e / (2 * ldh);
    const int k = 2 * j + h;
    out[e] = k <= H ? q[kx * Q2 + k] : 0.0;
  }
}

Status build_spec_split(rk_setup* s, cudaStream_t st) {
  cudaFree(s->spec_s);
  s->spec_s = nullptr;
  s->ldh = 0;
  if (!s->h2v.v[2].n || !s->spec_q) return Status::ok();
  const int H = s->p2 / 2;
  s->ldh = ((H / 2 + 1) + 1) & ~1;   // even: 16-byte rows for the bulk copy
  RK_CUDA_TRY(cudaMalloc(&s->spec_s, sizeof(double) * (size_t)s->H1 * 2 * s->ldh));
  const int64_t tot = (int64_t)s->H1 * 2 * s->ldh;
  spec_split_kernel<<<(int)std::min<int64_t>(ceil_div(tot, 256), 148 * 32), 256, 0, st>>>(s->spec_q, s->Q2, s->H1, H,
                                                                                           s->ldh, s->spec_s);
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

Status embedding_plans(rk_setup* s) {
  Embedding& e = s->emb;
  RK_TRY(plan_for(e.ps1, &e.pl1));
  RK_TRY(plan_for(e.ps2, &e.pl2));
  RK_TRY(plan_set(e.ps1, &e.ps1v));
  RK_TRY(plan_set(e.ps2, &e.ps2v));
  e.hs1v = PlanSet{};
  e.hs2v = PlanSet{};
  if (split_len(e.ps1) && s->M1 <= e.ps1 / 2) {   // kept columns of the row pass < ps1 / 2
    RK_TRY(plan_set(e.ps1 / 2, &e.hs1v));
    RK_TRY(split_table(e.ps1, &e.sws1));
  }
  if (split_len(e.ps2) && s->M2 <= e.ps2 / 2) {   // kept rows of the column pass < ps2 / 2
    RK_TRY(plan_set(e.ps2 / 2, &e.hs2v));
    RK_TRY(split_table(e.ps2, &e.sws2));
  }
  return Status::ok();
}

const FftPlan& plan_pick(const PlanSet& ps, int64_t lines) {
  // RK_WIDE: 0 normal only, 1 auto, 2 spread, 3 wide, 4 split (where available)
  static const int mode = getenv("RK_WIDE") ? atoi(getenv("RK_WIDE")) : 1;
  const FftPlan& sp = ps.v[1];
  const FftPlan& wd = ps.v[2];
  const FftPlan& sl = ps.v[3];
  if (mode == 0) return ps.v[0];
  if (mode == 2) return sp.n ? sp : ps.v[0];
  if (mode == 3) return wd.n ? wd : ps.v[0];
  if (mode == 4) return sl.n ? sl : ps.v[0];
  auto one_wave = [&](const FftPlan& pl) {   // every CTA of the launch resident at once?
    if (!pl.n || pl.nthr <= ps.v[0].nthr) return false;
    const int lpc = pick_lpc(pl, 4, lines);
    const size_t line_bytes = (size_t)pl.n * sizeof(double2);
    const int by_regs = fft_sm_threads(pl.wide) / (lpc * pl.nthr);
    const int by_smem = (int)((227 * 1024) / (lpc * line_bytes + line_bytes / 8 + 64));
    return by_regs > 0 && ceil_div(lines, lpc) <= 148LL * std::min(by_regs, by_smem);
  };
  // split only while the launch has at most one line per SM: measured on cfg2 (178 row pairs)
  // the split rows were neutral back to back and ~2 us slower with a cold L2
  if (sl.n && lines <= 148 && one_wave(sl)) return sl;
  if (one_wave(sp)) return sp;
  return wd.n ? wd : ps.v[0];
}

// FFT kernels run at 128 registers/thread (__launch_bounds__(512, 1)), so an SM holds at
// most 512 of their threads (1024 for the 64-register WIDE kernels); pick the lines-per-CTA that maximises resident threads under
// that and the shared-memory limit (line buffers + ~1/8 for twiddles/staging), preferring
// more lines per CTA on ties (wider coalesced transposed I/O), and never packing so much
// that the launch has fewer than 2 CTAs per SM.
int pick_lpc(const FftPlan& pl, int max_lines, int64_t total_lines) {
  const size_t line_bytes = (size_t)pl.n * sizeof(double2);
  static const size_t cap = [] {
    const char* e = getenv("RK_LPC_SMEM_KB");
    return (size_t)(e ? atoi(e) : 112) * 1024;
  }();
  int best = 1;
  int64_t best_res = -1;
  const int tmax = fft_sm_threads(pl.wide);   // resident FFT threads per SM (registers)
  for (int lpc = 1; lpc <= std::max(1, max_lines); ++lpc) {
    const int threads = lpc * pl.nthr;
    const size_t smem = lpc * line_bytes + line_bytes / 8 + 64;
    if (threads > tmax || (lpc > 1 && (smem > cap || ceil_div(total_lines, lpc) < 2 * 148))) break;
    const int by_regs = tmax / threads;
    const int by_smem = (int)((227 * 1024) / smem);
    const int64_t res = (int64_t)std::min(by_regs, by_smem) * threads;
    if (res >= best_res) {
      best_res = res;
      best = lpc;
    }
  }
  return best;
}

Status set_smem_attr(const void* fn, size_t bytes) {
  if (bytes <= 48 * 1024) return Status::ok();
  int dev = 0;
  RK_CUDA_TRY(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    if (g_smem_set.count({dev, fn})) return Status::ok();
  }
  RK_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_smem_set[{dev, fn}] = true;
  return Status::ok();
}

Status scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  static std::mutex mu;
  static std::set<int> configured;   // per device: keep freed blocks cached in its pool
  int dev = 0;
  RK_CUDA_TRY(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    if (!configured.count(dev)) {
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t thr = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
      }
      configured.insert(dev);
    }
  }
  RK_CUDA_TRY(cudaMallocAsync(p, bytes ? bytes : 16, st));
  return Status::ok();
}

void scratch_free(void* p, cudaStream_t st) {
  if (p) cudaFreeAsync(p, st);
}

// ------------------------------------------------------------ Matern ABI
__global__ void matern_kernel(MaternDev P, const double* __restrict__ d, double* __restrict__ out,
                              int64_t n, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = matern_cov(P, d[i], bad);
}

// ------------------------------------------------------------- padded grid
// cells with the floor tie rule and 1e-9 snap (gridding.py:123-127)
__device__ __forceinline__ int snap_cell(double t) {
  const double r = rint(t);
  return fabs(__dsub_rn(t, r)) <= 1.0e-9 ? (int)r : (int)floor(t);
}

struct PadArgs {
  const double* obs;
  int64_t n;
  double x0, y0, hx, hy;
  double lox, hix, loy, hiy;   // inclusive domain bounds with 1e-9 h slack
  int L, m1, m2;
  int* out;                    // [0] first bad index, [1..4] max(L-1-cx), max(cx+L-(m1-1)), ...
};

__global__ void pad_kernel(PadArgs a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = a.obs[2 * i], y = a.obs[2 * i + 1];
    if (!(x >= a.lox && x <= a.hix && y >= a.loy && y <= a.hiy)) {
      atomicMin(&a.out[0], (int)i);
      continue;
    }
    const int cx = snap_cell(__ddiv_rn(__dsub_rn(x, a.x0), a.hx));
    const int cy = snap_cell(__ddiv_rn(__dsub_rn(y, a.y0), a.hy));
    atomicMax(&a.out[1], (a.L - 1) - cx);
    atomicMax(&a.out[2], cx + a.L - (a.m1 - 1));
    atomicMax(&a.out[3], (a.L - 1) - cy);
    atomicMax(&a.out[4], cy + a.L - (a.m2 - 1));
  }
}

// --------------------------------------------------------------- weights
// One warp per observation (rapid.py:202-225): stencil (gridding.py:181-205),
// k_i = sigma2 phi(alpha |node - obs|), w = K_N^-1 k_i by forward/back
// substitution against the shared lower factor (in shared memory), cond_var,
// on-node unit rows and the cond_var clamp.
struct WArgs {
  MaternDev P;
  const double* obs;
  int64_t n;
  double px0, py0, hx, hy;
  double hix, hiy;             // (M1 - 1) + 1e-9, (M2 - 1) + 1e-9
  int L, bs, M, M1, M2;
  const double* chol;          // (M, M) row-major lower (global)
  int32_t* base;
  double* weights;
  double* cond_var;
  int* err;                    // [0] domain idx, [1] internal idx, [2] bessel
};

template <int MPL>
__global__ void __launch_bounds__(256) weights_kernel(WArgs a) {
  extern __shared__ double wsm[];
  const int M = a.M;
  const bool smem_l = M <= 64;
  double* Lr = wsm;            // row-major
  double* Lc = wsm + M * M;    // column-major
  if (smem_l) {
    for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
      const int r = e / M, c = e % M;
      const double v = a.chol[e];
      Lr[e] = v;
      Lc[c * M + r] = v;
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  for (int64_t i = (int64_t)blockIdx.x * wpb + warp; i < a.n; i += (int64_t)gridDim.x * wpb) {
    const double x = a.obs[2 * i], y = a.obs[2 * i + 1];
    const double tx = __ddiv_rn(__dsub_rn(x, a.px0), a.hx);
    const double ty = __ddiv_rn(__dsub_rn(y, a.py0), a.hy);
    if (!(tx >= -1.0e-9 && tx <= a.hix && ty >= -1.0e-9 && ty <= a.hiy)) {
      if (lane == 0) atomicMin(&a.err[0], (int)i);
      continue;
    }
    const int cx = snap_cell(tx), cy = snap_cell(ty);
    const int xlo = cx - (a.L - 1), ylo = cy - (a.L - 1);
    if (xlo < 0 || ylo < 0 || cx + a.L > a.M1 - 1 || cy + a.L > a.M2 - 1) {
      if (lane == 0) atomicMin(&a.err[1], (int)i);
      continue;
    }
    const double ox = __dsub_rn(tx, (double)cx), oy = __dsub_rn(ty, (double)cy);
    const bool on_node = fabs(ox) <= 1.0e-9 && fabs(oy) <= 1.0e-9;
    double k[MPL], v[MPL];
    int bad = 0;
#pragma unroll
    for (int s = 0; s < MPL; ++s) {
      const int m = s * 32 + lane;
      k[s] = 0.0;
      if (m < M) {
        const int r = m / a.bs, q = m % a.bs;
        const double nx = __dadd_rn(a.px0, __dmul_rn((double)(xlo + q), a.hx));
        const double ny = __dadd_rn(a.py0, __dmul_rn((double)(ylo + r), a.hy));
        const double dist = hypot(__dsub_rn(nx, x), __dsub_rn(ny, y));
        k[s] = matern_cov(a.P, dist, &bad);
      }
      v[s] = k[s];
    }
    if (bad) atomicOr(&a.err[2], 1);
    // forward substitution L y = k (column oriented; y overwrites v)
#pragma unroll
    for (int s = 0; s < MPL; ++s) {
      for (int cc = 0; cc < 32; ++cc) {
        const int c = s * 32 + cc;
        if (c >= M) break;
        const double dcc = smem_l ? Lr[c * M + c] : a.chol[c * M + c];
        const double mine = v[s] / dcc;
        const double yc = __shfl_sync(0xffffffffu, mine, cc);
        if (lane == cc) v[s] = yc;
#pragma unroll
        for (int s2 = s; s2 < MPL; ++s2) {
          const int r = s2 * 32 + lane;
          if (r > c && r < M) {
            const double lrc = smem_l ? Lc[c * M + r] : a.chol[r * M + c];
            v[s2] = fma(-lrc, yc, v[s2]);
          }
        }
      }
    }
    // back substitution L^T w = y
#pragma unroll
    for (int s = MPL - 1; s >= 0; --s) {
      for (int cc = 31; cc >= 0; --cc) {
        const int c = s * 32 + cc;
        if (c >= M) continue;
        const double dcc = smem_l ? Lr[c * M + c] : a.chol[c * M + c];
        const double mine = v[s] / dcc;
        const double wc = __shfl_sync(0xffffffffu, mine, cc);
        if (lane == cc) v[s] = wc;
#pragma unroll
        for (int s2 = 0; s2 <= s; ++s2) {
          const int r = s2 * 32 + lane;
          if (r < c) {
            const double lcr = smem_l ? Lr[c * M + r] : a.chol[c * M + r];
            v[s2] = fma(-lcr, wc, v[s2]);
          }
        }
      }
    }
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < MPL; ++s) part = fma(v[s], k[s], part);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    double cv = a.P.sigma2 - part;
    const int corner = (a.L - 1) * a.bs + (a.L - 1);
#pragma unroll
    for (int s = 0; s < MPL; ++s) {
      const int m = s * 32 + lane;
      if (m < M) {
        double w = v[s];
        if (on_node) w = (m == corner) ? 1.0 : 0.0;
        a.weights[i * M + m] = w;
      }
    }
    if (on_node) cv = 0.0;
    if (cv < 0.0 && cv > -1.0e-10 * a.P.sigma2) cv = 0.0;
    if (lane == 0) {
      a.cond_var[i] = cv;
      a.base[i] = ylo * a.M1 + xlo;
    }
  }
}

// Same computation with the neighbour order a compile-time constant (L <= 4, M <= 64): the
// substitutions are fully unrolled, the factor's reciprocal diagonal replaces the division in
// each step, and for M <= 16 one warp serves 32 / M observations (shuffles of width M).  A
// step of the serial chain is then shuffle -> multiply -> FMA (~40 cycles), where the
// generic kernel pays a division, runtime index arithmetic and the loop bounds.
__device__ __forceinline__ int cb0(int c0) { return c0 >> 2; }   // 4-column block of column c0

// HELP (L = 3, M = 36, Bessel-path Matern): the four cross covariances of each observation
// beyond the warp's 32 lanes are evaluated by a ninth helper warp in parallel (one evaluation
// per thread instead of two serial rounds), handed over through shared memory.  Only for the
// latency-bound Bessel case: with the closed forms the extra barrier per trip costs more.
template <int L, bool HELP = false>
__global__ void __launch_bounds__(HELP ? 288 : 256, HELP ? 2 : 3) weights_kernel_l(WArgs a) {
  static_assert(!HELP || L == 3, "helper warp layout is for M = 36");
  constexpr int BS = 2 * L, M = BS * BS;
  constexpr int LPO = M <= 4 ? 4 : M <= 16 ? 16 : 32;   // lanes per observation
  constexpr int G = 32 / LPO;                            // observations per warp
  constexpr int MPL = (M + 31) / 32;
  extern __shared__ double wsm[];
  // the factor in two 4-column-blocked layouts, so a lane's four entries of a block are one
  // contiguous 32-byte read and a warp's reads are contiguous (no bank conflicts):
  double* LF = wsm;                // LF[((c / 4) * M + r) * 4 + c % 4] = L[r][c]   (forward)
  double* LB = wsm + M * M;        // LB[((c / 4) * M + r) * 4 + c % 4] = L[c][r]   (backward)
  double* rd = wsm + 2 * M * M;    // 1 / L[c][c]
  double* kx = rd + M;             // HELP: (8 observations, M - 32) helper-evaluated covariances
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
    const int r = e / M, c = e % M;
    const double v = a.chol[e];
    LF[((c >> 2) * M + r) * 4 + (c & 3)] = v;
    LB[((r >> 2) * M + c) * 4 + (r & 3)] = v;
  }
  for (int c = threadIdx.x; c < M; c += blockDim.x) rd[c] = 1.0 / a.chol[c * M + c];
  const int lane = threadIdx.x & 31;
  const int sub = lane / LPO, sl = lane - sub * LPO;
  const int warp = threadIdx.x >> 5;
  const int wpb = HELP ? 8 : blockDim.x >> 5;   // observation warps per CTA
  const bool helper = HELP && warp == 8;
  const int64_t nw = (a.n + G - 1) / G;
  // persistent CTAs (the factor is staged once per CTA); the trip count is the same for every
  // warp so the staging barrier can sit after the first cross covariances (their latency
  // overlaps the factor's loads)
  const int64_t stride = (int64_t)gridDim.x * wpb;
  const int64_t trips = (nw + stride - 1) / stride;
  for (int64_t it = 0; it < trips; ++it) {
    // the helper's lane l serves observation warp l / 4, covariance 32 + l % 4
    const int ow = helper ? lane >> 2 : warp;
    const int64_t wi = (int64_t)blockIdx.x * wpb + ow + it * stride;
    const int64_t i = wi * G + sub;
    bool live = i < a.n;
    const double x = live ? a.obs[2 * i] : a.px0, y = live ? a.obs[2 * i + 1] : a.py0;
    const double tx = __ddiv_rn(__dsub_rn(x, a.px0), a.hx);
    const double ty = __ddiv_rn(__dsub_rn(y, a.py0), a.hy);
    int cx = 0, cy = 0;
    if (live && !(tx >= -1.0e-9 && tx <= a.hix && ty >= -1.0e-9 && ty <= a.hiy)) {
      if (sl == 0 && !helper) atomicMin(&a.err[0], (int)i);
      live = false;
    }
    if (live) {
      cx = snap_cell(tx);
      cy = snap_cell(ty);
      if (cx - (L - 1) < 0 || cy - (L - 1) < 0 || cx + L > a.M1 - 1 || cy + L > a.M2 - 1) {
        if (sl == 0 && !helper) atomicMin(&a.err[1], (int)i);
        live = false;
      }
    }
    const int xlo = cx - (L - 1), ylo = cy - (L - 1);
    const double ox = __dsub_rn(tx, (double)cx), oy = __dsub_rn(ty, (double)cy);
    const bool on_node = fabs(ox) <= 1.0e-9 && fabs(oy) <= 1.0e-9;
    double k[MPL], v[MPL];
    int bad = 0;
#pragma unroll
    for (int s = 0; s < MPL; ++s) {
      // HELP: observation warps evaluate chunk 0 only; the helper lane evaluates entry 32 + l % 4
      const int m = helper ? 32 + (lane & 3) : s * 32 + sl;
      k[s] = 0.0;
      if (live && m < M && (!HELP || s == 0)) {
        const int r = m / BS, q = m % BS;
        const double nx = __dadd_rn(a.px0, __dmul_rn((double)(xlo + q), a.hx));
        const double ny = __dadd_rn(a.py0, __dmul_rn((double)(ylo + r), a.hy));
        const double dist = hypot(__dsub_rn(nx, x), __dsub_rn(ny, y));
        k[s] = matern_cov(a.P, dist, &bad);
      }
      v[s] = k[s];
    }
    if (bad) atomicOr(&a.err[2], 1);
    if (HELP) {
      double* kb = kx + (it & 1) * 32;   // double-buffered: trip t + 2 reuses it after trip t + 1's barrier
      if (helper) kb[lane] = k[0];
      __syncthreads();   // helper results (and, on the first trip, the factor) staged
      if (helper) continue;
      k[1] = sl < M - 32 ? kb[warp * (M - 32) + sl] : 0.0;
      v[1] = k[1];
    } else if (it == 0) {
      __syncthreads();   // factor staged
    }
    // forward substitution L y = k, column oriented (y overwrites v), four columns per step:
    // every lane gathers the block's four entries (independent shuffles) and solves the 4 x 4
    // diagonal block itself, then applies the four column updates to its rows with one 32-byte
    // row read -- the same operations in the same order as one column at a time (bitwise
    // identical), with a quarter of the dependent shuffle round trips
    constexpr int W = LPO;
    const int jm4 = sl & 3;
#pragma unroll
    for (int s = 0; s < MPL; ++s) {
      const int ncc = s == MPL - 1 ? M - s * 32 : 32;   // a multiple of 4 (M = 4 L^2)
#pragma unroll 2
      for (int cb = 0; cb < ncc; cb += 4) {
        const int c0 = s * 32 + cb;
        double x0 = __shfl_sync(0xffffffffu, v[s], cb, W), x1 = __shfl_sync(0xffffffffu, v[s], cb + 1, W);
        double x2 = __shfl_sync(0xffffffffu, v[s], cb + 2, W), x3 = __shfl_sync(0xffffffffu, v[s], cb + 3, W);
        const double* B = LF + ((cb0(c0) * M + c0) * 4);   // B[4 i + j] = L[c0 + i][c0 + j]
        const double y0 = x0 * rd[c0];
        x1 = fma(-B[4], y0, x1);
        const double y1 = x1 * rd[c0 + 1];
        x2 = fma(-B[8], y0, x2);
        x2 = fma(-B[9], y1, x2);
        const double y2 = x2 * rd[c0 + 2];
        x3 = fma(-B[12], y0, x3);
        x3 = fma(-B[13], y1, x3);
        x3 = fma(-B[14], y2, x3);
        const double y3 = x3 * rd[c0 + 3];
        {   // the lane's own entry: its position in the block is sl & 3 for every block
          const double ym = jm4 == 0 ? y0 : jm4 == 1 ? y1 : jm4 == 2 ? y2 : y3;
          if ((sl >> 2) == (cb >> 2)) v[s] = ym;
        }
#pragma unroll
        for (int s2 = s; s2 < MPL; ++s2) {
          const int r = s2 * 32 + sl;
          if (r > c0 + 3 && r < M) {
            const double2* q = reinterpret_cast<const double2*>(LF + (cb0(c0) * M + r) * 4);   // L[r][c0 .. c0 + 3]
            const double2 a01 = q[0], a23 = q[1];
            v[s2] = fma(-a01.x, y0, v[s2]);
            v[s2] = fma(-a01.y, y1, v[s2]);
            v[s2] = fma(-a23.x, y2, v[s2]);
            v[s2] = fma(-a23.y, y3, v[s2]);
          }
        }
      }
    }
    // back substitution L' w = y, four columns per step from the bottom
#pragma unroll
    for (int s = MPL - 1; s >= 0; --s) {
      const int ncc = s == MPL - 1 ? M - s * 32 : 32;
#pragma unroll 2
      for (int cb = ncc - 4; cb >= 0; cb -= 4) {
        const int c0 = s * 32 + cb;
        double x0 = __shfl_sync(0xffffffffu, v[s], cb, W), x1 = __shfl_sync(0xffffffffu, v[s], cb + 1, W);
        double x2 = __shfl_sync(0xffffffffu, v[s], cb + 2, W), x3 = __shfl_sync(0xffffffffu, v[s], cb + 3, W);
        const double* B = LF + ((cb0(c0) * M + c0) * 4);
        const double w3 = x3 * rd[c0 + 3];
        x2 = fma(-B[14], w3, x2);
        const double w2 = x2 * rd[c0 + 2];
        x1 = fma(-B[13], w3, x1);
        x1 = fma(-B[9], w2, x1);
        const double w1 = x1 * rd[c0 + 1];
        x0 = fma(-B[12], w3, x0);
        x0 = fma(-B[8], w2, x0);
        x0 = fma(-B[4], w1, x0);
        const double w0 = x0 * rd[c0];
        {
          const double wm = jm4 == 0 ? w0 : jm4 == 1 ? w1 : jm4 == 2 ? w2 : w3;
          if ((sl >> 2) == (cb >> 2)) v[s] = wm;
        }
#pragma unroll
        for (int s2 = 0; s2 <= s; ++s2) {
          const int r = s2 * 32 + sl;
          if (r < c0) {
            const double2* q = reinterpret_cast<const double2*>(LB + (cb0(c0) * M + r) * 4);   // L[c0 .. c0 + 3][r]
            const double2 a01 = q[0], a23 = q[1];
            v[s2] = fma(-a23.y, w3, v[s2]);
            v[s2] = fma(-a23.x, w2, v[s2]);
            v[s2] = fma(-a01.y, w1, v[s2]);
            v[s2] = fma(-a01.x, w0, v[s2]);
          }
        }
      }
    }
    double part = 0.0;
#pragma unroll
    for (int s = 0; s < MPL; ++s) part = fma(v[s], k[s], part);
#pragma unroll
    for (int o = LPO / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o, LPO);
    if (!live) continue;
    double cv = a.P.sigma2 - part;
    constexpr int corner = (L - 1) * BS + (L - 1);
#pragma unroll
    for (int s = 0; s < MPL; ++s) {
      const int m = s * 32 + sl;
      if (m < M) a.weights[i * M + m] = on_node ? (m == corner ? 1.0 : 0.0) : v[s];
    }
    if (on_node) cv = 0.0;
    if (cv < 0.0 && cv > -1.0e-10 * a.P.sigma2) cv = 0.0;
    if (sl == 0) {
      a.cond_var[i] = cv;
      a.base[i] = ylo * a.M1 + xlo;
    }
  }
}

// M = 36 / 64 (L = 3 / 4), one lane per stencil entry: OB observations per warp, their
// substitution chains interleaved step by step.  One observation's chain is a dependent
// shuffle -> multiply -> FMA sequence (latency bound: ~15 % issue with one chain per warp);
// OB independent chains per warp hide each other's latency, and each factor entry read from
// shared memory serves all OB observations.  Per observation the operations and their order
// are exactly those of weights_kernel_l (bitwise identical weights).
template <int L, int OB>
__global__ void __launch_bounds__(256, 2) weights_kernel_ob(WArgs a) {
  constexpr int BS = 2 * L, M = BS * BS;
  static_assert(M > 16, "sub-warp layouts use weights_kernel_l");
  constexpr int MPL = (M + 31) / 32;
  extern __shared__ double wsm[];
  double* LF = wsm;                // LF[((c / 4) * M + r) * 4 + c % 4] = L[r][c]   (forward)
  double* LB = wsm + M * M;        // LB[((c / 4) * M + r) * 4 + c % 4] = L[c][r]   (backward)
  double* rd = wsm + 2 * M * M;    // 1 / L[c][c]
  for (int e = threadIdx.x; e < M * M; e += blockDim.x) {
    const int r = e / M, c = e % M;
    const double v = a.chol[e];
    LF[((c >> 2) * M + r) * 4 + (c & 3)] = v;
    LB[((r >> 2) * M + c) * 4 + (r & 3)] = v;
  }
  for (int c = threadIdx.x; c < M; c += blockDim.x) rd[c] = 1.0 / a.chol[c * M + c];
  const int sl = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  const int64_t nw = (a.n + OB - 1) / OB;
  const int64_t stride = (int64_t)gridDim.x * wpb;
  const int64_t trips = (nw + stride - 1) / stride;
  const int jm4 = sl & 3;
  for (int64_t it = 0; it < trips; ++it) {
    const int64_t wi = (int64_t)blockIdx.x * wpb + warp + it * stride;
    bool live[OB], on_node[OB];
    int xlo[OB], ylo[OB];
    double xs[OB], ys[OB];
    double k[OB][MPL], v[OB][MPL];
    int bad = 0;
#pragma unroll
    for (int o = 0; o < OB; ++o) {
      const int64_t i = wi * OB + o;
      live[o] = i < a.n;
      const double x = live[o] ? a.obs[2 * i] : a.px0, y = live[o] ? a.obs[2 * i + 1] : a.py0;
      xs[o] = x;
      ys[o] = y;
      const double tx = __ddiv_rn(__dsub_rn(x, a.px0), a.hx);
      const double ty = __ddiv_rn(__dsub_rn(y, a.py0), a.hy);
      int cx = 0, cy = 0;
      if (live[o] && !(tx >= -1.0e-9 && tx <= a.hix && ty >= -1.0e-9 && ty <= a.hiy)) {
        if (sl == 0) atomicMin(&a.err[0], (int)i);
        live[o] = false;
      }
      if (live[o]) {
        cx = snap_cell(tx);
        cy = snap_cell(ty);
        if (cx - (L - 1) < 0 || cy - (L - 1) < 0 || cx + L > a.M1 - 1 || cy + L > a.M2 - 1) {
          if (sl == 0) atomicMin(&a.err[1], (int)i);
          live[o] = false;
        }
      }
      xlo[o] = cx - (L - 1);
      ylo[o] = cy - (L - 1);
      const double ox = __dsub_rn(tx, (double)cx), oy = __dsub_rn(ty, (double)cy);
      on_node[o] = fabs(ox) <= 1.0e-9 && fabs(oy) <= 1.0e-9;
    }
#pragma unroll
    for (int s = 0; s < MPL; ++s)
#pragma unroll
      for (int o = 0; o < OB; ++o) {
        const int m = s * 32 + sl;
        k[o][s] = 0.0;
        if (live[o] && m < M) {
          const int r = m / BS, q = m % BS;
          const double nx = __dadd_rn(a.px0, __dmul_rn((double)(xlo[o] + q), a.hx));
          const double ny = __dadd_rn(a.py0, __dmul_rn((double)(ylo[o] + r), a.hy));
          const double dist = hypot(__dsub_rn(nx, xs[o]), __dsub_rn(ny, ys[o]));
          k[o][s] = matern_cov(a.P, dist, &bad);
        }
        v[o][s] = k[o][s];
      }
    if (bad) atomicOr(&a.err[2], 1);
    if (it == 0) __syncthreads();   // factor staged
    // forward substitution L y = k, four columns per step (as weights_kernel_l)
#pragma unroll
    for (int s = 0; s < MPL; ++s) {
      const int ncc = s == MPL - 1 ? M - s * 32 : 32;
#pragma unroll 2
      for (int cb = 0; cb < ncc; cb += 4) {
        const int c0 = s * 32 + cb;
        const double* B = LF + ((cb0(c0) * M + c0) * 4);
        const double b4 = B[4], b8 = B[8], b9 = B[9], b12 = B[12], b13 = B[13], b14 = B[14];
        const double r0 = rd[c0], r1 = rd[c0 + 1], r2 = rd[c0 + 2], r3 = rd[c0 + 3];
        double y0[OB], y1[OB], y2[OB], y3[OB];
#pragma unroll
        for (int o = 0; o < OB; ++o) {
          double x0 = __shfl_sync(0xffffffffu, v[o][s], cb), x1 = __shfl_sync(0xffffffffu, v[o][s], cb + 1);
          double x2 = __shfl_sync(0xffffffffu, v[o][s], cb + 2), x3 = __shfl_sync(0xffffffffu, v[o][s], cb + 3);
          y0[o] = x0 * r0;
          x1 = fma(-b4, y0[o], x1);
          y1[o] = x1 * r1;
          x2 = fma(-b8, y0[o], x2);
          x2 = fma(-b9, y1[o], x2);
          y2[o] = x2 * r2;
          x3 = fma(-b12, y0[o], x3);
          x3 = fma(-b13, y1[o], x3);
          x3 = fma(-b14, y2[o], x3);
          y3[o] = x3 * r3;
          const double ym = jm4 == 0 ? y0[o] : jm4 == 1 ? y1[o] : jm4 == 2 ? y2[o] : y3[o];
          if ((sl >> 2) == (cb >> 2)) v[o][s] = ym;
        }
#pragma unroll
        for (int s2 = s; s2 < MPL; ++s2) {
          const int r = s2 * 32 + sl;
          if (r > c0 + 3 && r < M) {
            const double2* q = reinterpret_cast<const double2*>(LF + (cb0(c0) * M + r) * 4);
            const double2 a01 = q[0], a23 = q[1];
#pragma unroll
            for (int o = 0; o < OB; ++o) {
              v[o][s2] = fma(-a01.x, y0[o], v[o][s2]);
              v[o][s2] = fma(-a01.y, y1[o], v[o][s2]);
              v[o][s2] = fma(-a23.x, y2[o], v[o][s2]);
              v[o][s2] = fma(-a23.y, y3[o], v[o][s2]);
            }
          }
        }
      }
    }
    // back substitution L' w = y
#pragma unroll
    for (int s = MPL - 1; s >= 0; --s) {
      const int ncc = s == MPL - 1 ? M - s * 32 : 32;
#pragma unroll 2
      for (int cb = ncc - 4; cb >= 0; cb -= 4) {
        const int c0 = s * 32 + cb;
        const double* B = LF + ((cb0(c0) * M + c0) * 4);
        const double b4 = B[4], b8 = B[8], b9 = B[9], b12 = B[12], b13 = B[13], b14 = B[14];
        const double r0 = rd[c0], r1 = rd[c0 + 1], r2 = rd[c0 + 2], r3 = rd[c0 + 3];
        double w0[OB], w1[OB], w2[OB], w3[OB];
#pragma unroll
        for (int o = 0; o < OB; ++o) {
          double x0 = __shfl_sync(0xffffffffu, v[o][s], cb), x1 = __shfl_sync(0xffffffffu, v[o][s], cb + 1);
          double x2 = __shfl_sync(0xffffffffu, v[o][s], cb + 2), x3 = __shfl_sync(0xffffffffu, v[o][s], cb + 3);
          w3[o] = x3 * r3;
          x2 = fma(-b14, w3[o], x2);
          w2[o] = x2 * r2;
          x1 = fma(-b13, w3[o], x1);
          x1 = fma(-b9, w2[o], x1);
          w1[o] = x1 * r1;
          x0 = fma(-b12, w3[o], x0);
          x0 = fma(-b8, w2[o], x0);
          x0 = fma(-b4, w1[o], x0);
          w0[o] = x0 * r0;
          const double wm = jm4 == 0 ? w0[o] : jm4 == 1 ? w1[o] : jm4 == 2 ? w2[o] : w3[o];
          if ((sl >> 2) == (cb >> 2)) v[o][s] = wm;
        }
#pragma unroll
        for (int s2 = 0; s2 <= s; ++s2) {
          const int r = s2 * 32 + sl;
          if (r < c0) {
            const double2* q = reinterpret_cast<const double2*>(LB + (cb0(c0) * M + r) * 4);
            const double2 a01 = q[0], a23 = q[1];
#pragma unroll
            for (int o = 0; o < OB; ++o) {
              v[o][s2] = fma(-a23.y, w3[o], v[o][s2]);
              v[o][s2] = fma(-a23.x, w2[o], v[o][s2]);
              v[o][s2] = fma(-a01.y, w1[o], v[o][s2]);
              v[o][s2] = fma(-a01.x, w0[o], v[o][s2]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int o = 0; o < OB; ++o) {
      double part = 0.0;
#pragma unroll
      for (int s = 0; s < MPL; ++s) part = fma(v[o][s], k[o][s], part);
#pragma unroll
      for (int d = 16; d > 0; d >>= 1) part += __shfl_xor_sync(0xffffffffu, part, d);
      if (!live[o]) continue;
      const int64_t i = wi * OB + o;
      double cv = a.P.sigma2 - part;
      constexpr int corner = (L - 1) * BS + (L - 1);
#pragma unroll
      for (int s = 0; s < MPL; ++s) {
        const int m = s * 32 + sl;
        if (m < M) a.weights[i * M + m] = on_node[o] ? (m == corner ? 1.0 : 0.0) : v[o][s];
      }
      if (on_node[o]) cv = 0.0;
      if (cv < 0.0 && cv > -1.0e-10 * a.P.sigma2) cv = 0.0;
      if (sl == 0) {
        a.cond_var[i] = cv;
        a.base[i] = ylo[o] * a.M1 + xlo[o];
      }
    }
  }
}

// ----------------------------------------------------------------- K1 on FP64 tensor cores
// weights_kernel_mma<L>: a warp solves 8 observations at once as an (MP x 8) right-hand-side
// block Y (MP = M rounded up to a multiple of 8; padded rows have k = 0 and a unit diagonal, so
// they stay exactly 0), blocked by 8-row tiles:
//   forward  L y = k : for tile t: substitution inside the 8 x 8 diagonal block (column
//                      oriented, reciprocal diagonal), then Y_u -= L_ut Y_t for every u > t as
//                      two mma.m8n8k4 f64 (DMMA) per tile pair;
//   backward L'w = y : the same from the last tile up with L' (its blocks staged transposed).
// Y lives in the DMMA accumulator layout (lane = 4 g + q holds rows g, observations 2q, 2q+1 of
// every tile); a solved tile becomes the B operand of the updates by one shuffle per register.
// This is a blocked (backward-stable) TRSM, not the explicit inverse (hard part 1);
// each observation's solve depends only on its own column (DMMA columns are independent), so a
// weight row does not depend on which observations share the warp.  n (2 M^2) flops go from
// ~2440 issued instructions per observation (shuffle -> multiply -> FMA chains, weights_kernel_ob)
// to ~300, the off-diagonal work on the tensor pipe.
__device__ __forceinline__ void dmma884_w(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int L>
struct WMma {
  static constexpr int BS = 2 * L, M = BS * BS, T = (M + 7) / 8, MP = 8 * T;
  static constexpr int FRAG = T * T * 2 * 32;   // doubles per A-fragment table
  static constexpr int DLD = 72;                // padded 8 x 8 diagonal block: [g * 9 + r]
  static constexpr size_t smem_bytes() { return sizeof(double) * (2 * FRAG + 2 * T * DLD + MP + 8 * MP * 8); }
};

// HALF: half-integer nu (closed-form Matern only: a fraction of the code, which otherwise
// overflows the instruction cache -- ncu: 14 % no-instruction stalls with the Bessel paths inlined)
template <int L, bool HALF = false>
__global__ void __launch_bounds__(256, 2) weights_kernel_mma(WArgs a) {
  using W = WMma<L>;
  constexpr int BS = W::BS, M = W::M, T = W::T, MP = W::MP;
  extern __shared__ double wsm[];
  double* AF = wsm;                    // forward A fragments: -L[8u + g][8t + 4kb + q]
  double* AB = AF + W::FRAG;           // backward A fragments: -L[8t + 4kb + q][8u + g]
  double* DF = AB + W::FRAG;           // diagonal blocks: DF[t][g * 9 + r] = L[8t + g][8t + r]
  double* DB = DF + T * W::DLD;        // transposed:      DB[t][g * 9 + r] = L[8t + r][8t + g]
  double* rd = DB + T * W::DLD;        // 1 / L[m][m] (1 on padded rows)
  double* kw = rd + MP + (threadIdx.x >> 5) * MP * 8;   // this warp's cross covariances [m][obs]
  auto Lat = [&](int r, int c) -> double {
    if (r < M && c < M) return a.chol[r * M + c];
    return r == c ? 1.0 : 0.0;
  };
  for (int e = threadIdx.x; e < T * T * 2 * 32; e += blockDim.x) {
    const int ln = e & 31, kb = (e >> 5) & 1, tu = e >> 6, t = tu % T, u = tu / T;
    const int g = ln >> 2, q = ln & 3;
    AF[e] = -Lat(8 * u + g, 8 * t + 4 * kb + q);
    AB[e] = -Lat(8 * t + 4 * kb + q, 8 * u + g);
  }
  for (int e = threadIdx.x; e < T * 64; e += blockDim.x) {
    const int t = e >> 6, g = (e >> 3) & 7, r = e & 7;
    DF[t * W::DLD + g * 9 + r] = Lat(8 * t + g, 8 * t + r);
    DB[t * W::DLD + g * 9 + r] = Lat(8 * t + r, 8 * t + g);
  }
  for (int m = threadIdx.x; m < MP; m += blockDim.x) rd[m] = 1.0 / Lat(m, m);
  const int lane = threadIdx.x & 31, g = lane >> 2, q = lane & 3;
  const int warp = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int64_t ntask = (a.n + 7) / 8;
  const int64_t stride = (int64_t)gridDim.x * wpb;
  const int64_t trips = (ntask + stride - 1) / stride;
  for (int64_t it = 0; it < trips; ++it) {
    const int64_t i0 = ((int64_t)blockIdx.x * wpb + warp + it * stride) * 8;
    __syncwarp();   // the previous trip's reads of kw are done
    // this lane's two observations 2q, 2q + 1 of the task (accumulator columns) and, for the
    // cross covariances, observation lane & 7
    bool live[2], on_node[2];
    int xlo[2], ylo[2];
    double xs[2], ys[2];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int o = j < 2 ? 2 * q + j : (lane & 7);
      const int64_t i = i0 + o;
      bool lv = i < a.n;
      const double x = lv ? a.obs[2 * i] : a.px0, y = lv ? a.obs[2 * i + 1] : a.py0;
      const double tx = __ddiv_rn(__dsub_rn(x, a.px0), a.hx);
      const double ty = __ddiv_rn(__dsub_rn(y, a.py0), a.hy);
      int cx = 0, cy = 0;
      if (lv && !(tx >= -1.0e-9 && tx <= a.hix && ty >= -1.0e-9 && ty <= a.hiy)) {
        if (j == 2 && lane < 8) atomicMin(&a.err[0], (int)i);
        lv = false;
      }
      if (lv) {
        cx = snap_cell(tx);
        cy = snap_cell(ty);
        if (cx - (L - 1) < 0 || cy - (L - 1) < 0 || cx + L > a.M1 - 1 || cy + L > a.M2 - 1) {
          if (j == 2 && lane < 8) atomicMin(&a.err[1], (int)i);
          lv = false;
        }
      }
      if (j < 2) {
        live[j] = lv;
        xlo[j] = cx - (L - 1);
        ylo[j] = cy - (L - 1);
        const double ox = __dsub_rn(tx, (double)cx), oy = __dsub_rn(ty, (double)cy);
        on_node[j] = fabs(ox) <= 1.0e-9 && fabs(oy) <= 1.0e-9;
      } else {
        // cross covariances of observation lane & 7 to block rows m = lane / 8 + 4 k, staged in
        // the warp's (MP x 8) smem block (four independent evaluations per iteration; the Matern
        // code stays out of the register-resident solve)
        int bad = 0;
#pragma unroll 4
        for (int m = lane >> 3; m < MP; m += 4) {
          double kv = 0.0;
          if (lv && m < M) {
            const int r = m / BS, c = m % BS;
            const double nx = __dadd_rn(a.px0, __dmul_rn((double)(cx - (L - 1) + c), a.hx));
            const double ny = __dadd_rn(a.py0, __dmul_rn((double)(cy - (L - 1) + r), a.hy));
            const double dist = hypot(__dsub_rn(nx, x), __dsub_rn(ny, y));
            kv = HALF ? a.P.sigma2 * matern_phi_half(a.P, a.P.alpha * dist) : matern_cov(a.P, dist, &bad);
          }
          kw[m * 8 + (lane & 7)] = kv;
        }
        if (bad) atomicOr(&a.err[2], 1);
      }
    }
    __syncwarp();
    double Y[T][2];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int j = 0; j < 2; ++j) Y[t][j] = kw[(8 * t + g) * 8 + 2 * q + j];
    if (it == 0) __syncthreads();   // factor tables staged (their loads overlap the first k)
    // forward substitution L y = k
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const double* D = DF + t * W::DLD + g * 9;
#pragma unroll
      for (int r = 0; r < 8; ++r) {
        const double s = rd[8 * t + r];
        const double y0 = __shfl_sync(0xffffffffu, Y[t][0] * s, 4 * r + q);
        const double y1 = __shfl_sync(0xffffffffu, Y[t][1] * s, 4 * r + q);
        if (g == r) {
          Y[t][0] = y0;
          Y[t][1] = y1;
        } else if (g > r) {
          const double l = D[r];
          Y[t][0] = fma(-l, y0, Y[t][0]);
          Y[t][1] = fma(-l, y1, Y[t][1]);
        }
      }
      if (t + 1 < T) {
        double bf[2];
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          const int src = (4 * kb + q) * 4 + (g >> 1);
          const double v0 = __shfl_sync(0xffffffffu, Y[t][0], src);
          const double v1 = __shfl_sync(0xffffffffu, Y[t][1], src);
          bf[kb] = (g & 1) ? v1 : v0;
        }
#pragma unroll
        for (int u = t + 1; u < T; ++u)
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
            dmma884_w(Y[u][0], Y[u][1], AF[((u * T + t) * 2 + kb) * 32 + lane], bf[kb]);
      }
    }
    // back substitution L' w = y
#pragma unroll
    for (int t = T - 1; t >= 0; --t) {
      const double* D = DB + t * W::DLD + g * 9;
#pragma unroll
      for (int r = 7; r >= 0; --r) {
        const double s = rd[8 * t + r];
        const double w0 = __shfl_sync(0xffffffffu, Y[t][0] * s, 4 * r + q);
        const double w1 = __shfl_sync(0xffffffffu, Y[t][1] * s, 4 * r + q);
        if (g == r) {
          Y[t][0] = w0;
          Y[t][1] = w1;
        } else if (g < r) {
          const double l = D[r];
          Y[t][0] = fma(-l, w0, Y[t][0]);
          Y[t][1] = fma(-l, w1, Y[t][1]);
        }
      }
      if (t > 0) {
        double bf[2];
#pragma unroll
        for (int kb = 0; kb < 2; ++kb) {
          const int src = (4 * kb + q) * 4 + (g >> 1);
          const double v0 = __shfl_sync(0xffffffffu, Y[t][0], src);
          const double v1 = __shfl_sync(0xffffffffu, Y[t][1], src);
          bf[kb] = (g & 1) ? v1 : v0;
        }
#pragma unroll
        for (int u = 0; u < t; ++u)
#pragma unroll
          for (int kb = 0; kb < 2; ++kb)
            dmma884_w(Y[u][0], Y[u][1], AB[((u * T + t) * 2 + kb) * 32 + lane], bf[kb]);
      }
    }
    // cond_var = sigma2 - w . k (sum over this lane's rows, then over the 8 row groups)
    double part[2] = {0.0, 0.0};
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
      for (int j = 0; j < 2; ++j) part[j] = fma(Y[t][j], kw[(8 * t + g) * 8 + 2 * q + j], part[j]);
#pragma unroll
    for (int o = 4; o < 32; o <<= 1)
#pragma unroll
      for (int j = 0; j < 2; ++j) part[j] += __shfl_xor_sync(0xffffffffu, part[j], o);
    constexpr int corner = (L - 1) * BS + (L - 1);
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (!live[j]) continue;
      const int64_t i = i0 + 2 * q + j;
#pragma unroll
      for (int t = 0; t < T; ++t) {
        const int m = 8 * t + g;
        if (m < M) a.weights[i * M + m] = on_node[j] ? (m == corner ? 1.0 : 0.0) : Y[t][j];
      }
      if (g == 0) {
        double cv = a.P.sigma2 - part[j];
        if (on_node[j]) cv = 0.0;
        if (cv < 0.0 && cv > -1.0e-10 * a.P.sigma2) cv = 0.0;
        a.cond_var[i] = cv;
        a.base[i] = ylo[j] * a.M1 + xlo[j];
      }
    }
  }
}

// cell_start[b] = lower_bound(sorted keys, b) for b in [0, nb]
__global__ void cell_start_kernel(const int32_t* __restrict__ keys, int64_t n, int32_t* cs,
                                  int64_t nb) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= nb;
       b += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (keys[mid] < b) lo = mid + 1; else hi = mid;
    }
    cs[b] = (int32_t)lo;
  }
}

__global__ void iota_kernel(int32_t* v, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    v[i] = (int32_t)i;
}

__global__ void permute_rows_kernel(const double* __restrict__ w, const int32_t* __restrict__ perm,
                                    double* __restrict__ ws, int64_t n, int M) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * M;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / M;
    const int m = (int)(e % M);
    ws[e] = w[(int64_t)perm[j] * M + m];
  }
}

__global__ void expand_indices_kernel(const int32_t* __restrict__ base, int64_t n, int bs, int M1,
                                      int64_t* __restrict__ out) {
  const int M = bs * bs;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n * M;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = e / M;
    const int m = (int)(e % M);
    out[e] = (int64_t)base[i] + (int64_t)(m / bs) * M1 + (m % bs);
  }
}

// ----------------------------------------------------- host K_N (tiny, M x M)
// rapid.py:103-117: offsets (arange(2L) h) row-major over the block, cdist-free
// hypot distances, covariance, 0.5 (k + k') symmetrisation.
static Status kn_matrix_dev(const rk_setup* s, std::vector<double>* kn) {
  const int M = s->M, bs = s->bs;
  std::vector<double> dist((size_t)M * M);
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < M; ++j) {
      const double xi = (double)(i % bs) * s->grid.hx, yi = (double)(i / bs) * s->grid.hy;
      const double xj = (double)(j % bs) * s->grid.hx, yj = (double)(j / bs) * s->grid.hy;
      dist[(size_t)i * M + j] = std::hypot(xi - xj, yi - yj);
    }
  double *dd = nullptr, *dk = nullptr;
  int* bad = nullptr;
  const size_t bytes = sizeof(double) * M * M;
  RK_CUDA_TRY(cudaMalloc(&dd, bytes));
  RK_CUDA_TRY(cudaMalloc(&dk, bytes));
  RK_CUDA_TRY(cudaMalloc(&bad, sizeof(int)));
  RK_CUDA_TRY(cudaMemset(bad, 0, sizeof(int)));
  RK_CUDA_TRY(cudaMemcpy(dd, dist.data(), bytes, cudaMemcpyHostToDevice));
  matern_kernel<<<(M * M + 255) / 256, 256>>>(s->mat, dd, dk, (int64_t)M * M, bad);
  count_launch();
  RK_LAUNCH_CHECK();
  kn->resize((size_t)M * M);
  RK_CUDA_TRY(cudaMemcpy(kn->data(), dk, bytes, cudaMemcpyDeviceToHost));
  int hb = 0;
  RK_CUDA_TRY(cudaMemcpy(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost));
  cudaFree(dd);
  cudaFree(dk);
  cudaFree(bad);
  if (hb) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");
  for (int i = 0; i < M; ++i)
    for (int j = i + 1; j < M; ++j) {
      const double a = (*kn)[(size_t)i * M + j], b = (*kn)[(size_t)j * M + i];
      const double v = 0.5 * (a + b);
      (*kn)[(size_t)i * M + j] = v;
      (*kn)[(size_t)j * M + i] = v;
    }
  return Status::ok();
}

// lower Cholesky (right-looking, row-major); false if not positive definite
static bool cholesky_lower(std::vector<double>& a, int M) {
  for (int j = 0; j < M; ++j) {
    double d = a[(size_t)j * M + j];
    for (int k = 0; k < j; ++k) d -= a[(size_t)j * M + k] * a[(size_t)j * M + k];
    if (!(d > 0.0)) return false;
    d = std::sqrt(d);
    a[(size_t)j * M + j] = d;
    for (int i = j + 1; i < M; ++i) {
      double v = a[(size_t)i * M + j];
      for (int k = 0; k < j; ++k) v -= a[(size_t)i * M + k] * a[(size_t)j * M + k];
      a[(size_t)i * M + j] = v / d;
    }
    for (int k = j + 1; k < M; ++k) a[(size_t)j * M + k] = 0.0;
  }
  return true;
}

static void chol_inverse(const std::vector<double>& L, int M, std::vector<double>* inv) {
  // (L L')^-1 column by column: cho_solve(I) (rapid.py:193)
  inv->assign((size_t)M * M, 0.0);
  std::vector<double> y(M);
  for (int c = 0; c < M; ++c) {
    for (int i = 0; i < M; ++i) {
      double v = (i == c) ? 1.0 : 0.0;
      for (int k = 0; k < i; ++k) v -= L[(size_t)i * M + k] * y[k];
      y[i] = v / L[(size_t)i * M + i];
    }
    for (int i = M - 1; i >= 0; --i) {
      double v = y[i];
      for (int k = i + 1; k < M; ++k) v -= L[(size_t)k * M + i] * (*inv)[(size_t)k * M + c];
      (*inv)[(size_t)i * M + c] = v / L[(size_t)i * M + i];
    }
  }
}

Status spectrum_quarter(const MaternDev& P, double hx, double hy, int p1, int p2, double scale,
                        double* out_q, int ldq, cudaStream_t st);  // rk_predict.cu
int quarter_ld(int p2);                                             // rk_predict.cu

// ---------------------------------------------------- sparse gather plan (setup)
// Every (sorted obs j, block entry m) contributes w * c to node q = base_j + (m / BS) M1 +
// (m % BS).  A stable sort by (q, dy) keeps j ascending inside each (q, dy), which is the
// accumulation order of the dense gather; the per-predict gather then touches only the
// n M contributions instead of testing 2L cell ranges at every padded node.
__global__ void ent_gen_kernel(const int32_t* __restrict__ bsort, int64_t n, int M, int BS, int M1,
                               uint64_t* __restrict__ key, int32_t* __restrict__ val) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n * M;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / M;
    const int m = (int)(i % M);
    const int dy = m / BS, dx = m % BS;
    const int64_t q = (int64_t)bsort[j] + (int64_t)dy * M1 + dx;
    key[i] = (uint64_t)q * BS + dy;
    val[i] = (int32_t)i;
  }
}

__global__ void ent_fin_kernel(const uint64_t* __restrict__ key, const int32_t* __restrict__ val,
                               const int32_t* __restrict__ perm, int64_t tot, int M, int BS,
                               int32_t* ent_w, int32_t* ent_c, int32_t* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    ent_w[i] = val[i];
    ent_c[i] = perm[val[i] / M];
    flag[i] = (i == 0 || key[i] / BS != key[i - 1] / BS) ? 1 : 0;
  }
}

__global__ void node_fill_kernel(const uint64_t* __restrict__ key, const int32_t* __restrict__ flag,
                                 const int32_t* __restrict__ pos, int64_t tot, int BS,
                                 int32_t* node_q, int32_t* node_off) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (flag[i]) {
      node_q[pos[i]] = (int32_t)(key[i] / BS);
      node_off[pos[i]] = (int32_t)i;
    }
  }
}

__global__ void row_node_kernel(const int32_t* __restrict__ node_q, int64_t nnodes, int M1, int M2,
                                int32_t* row_node) {
  for (int64_t y = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; y <= M2;
       y += (int64_t)gridDim.x * blockDim.x) {
    const int64_t target = y * M1;
    int64_t lo = 0, hi = nnodes;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (node_q[mid] < target) lo = mid + 1; else hi = mid;
    }
    row_node[y] = (int32_t)lo;
  }
}

__global__ void ent_value_kernel(const int32_t* __restrict__ ent_w, const double* __restrict__ wsort, int64_t tot,
                                 double* ent_wv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot;
       i += (int64_t)gridDim.x * blockDim.x)
    ent_wv[i] = wsort[ent_w[i]];
}

static Status build_sparse_gather(rk_setup* s) {
  const int64_t tot = s->n * s->M;
  if (tot >= ((int64_t)1 << 31)) return Status::err(RK_DOMAIN, "n * M too large for the gather plan");
  uint64_t *key = nullptr, *key2 = nullptr;
  int32_t *val = nullptr, *val2 = nullptr, *flag = nullptr, *pos = nullptr;
  RK_CUDA_TRY(cudaMalloc(&key, sizeof(uint64_t) * tot));
  RK_CUDA_TRY(cudaMalloc(&key2, sizeof(uint64_t) * tot));
  RK_CUDA_TRY(cudaMalloc(&val, sizeof(int32_t) * tot));
  RK_CUDA_TRY(cudaMalloc(&val2, sizeof(int32_t) * tot));
  RK_CUDA_TRY(cudaMalloc(&flag, sizeof(int32_t) * tot));
  RK_CUDA_TRY(cudaMalloc(&pos, sizeof(int32_t) * tot));
  RK_CUDA_TRY(cudaMalloc(&s->ent_w, sizeof(int32_t) * tot));
  RK_CUDA_TRY(cudaMalloc(&s->ent_c, sizeof(int32_t) * (tot + 4)));   // + slack: pass 1 bulk-copies 16-byte-rounded ranges
  const int grid = (int)std::min<int64_t>(ceil_div(tot, 256), 148 * 32);
  ent_gen_kernel<<<grid, 256>>>(s->bsort, s->n, s->M, s->bs, s->M1, key, val);
  count_launch();
  RK_LAUNCH_CHECK();
  const uint64_t maxkey = (uint64_t)s->M1 * s->M2 * s->bs;
  int end_bit = 1;
  while (end_bit < 63 && ((uint64_t)1 << end_bit) <= maxkey) ++end_bit;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, key, key2, val, val2, (int)tot, 0, end_bit);
  void* tmp = nullptr;
  size_t tb2 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb2, flag, pos, (int)tot);
  RK_CUDA_TRY(cudaMalloc(&tmp, std::max(tb, tb2) + 16));
  RK_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, val, val2, (int)tot, 0, end_bit));
  count_launch();
  ent_fin_kernel<<<grid, 256>>>(key2, val2, s->perm, tot, s->M, s->bs, s->ent_w, s->ent_c, flag);
  count_launch();
  RK_LAUNCH_CHECK();
  RK_CUDA_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb2, flag, pos, (int)tot));
  count_launch();
  int32_t last_pos = 0, last_flag = 0;
  RK_CUDA_TRY(cudaMemcpy(&last_pos, pos + tot - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  RK_CUDA_TRY(cudaMemcpy(&last_flag, flag + tot - 1, sizeof(int32_t), cudaMemcpyDeviceToHost));
  s->nnodes = (int64_t)last_pos + last_flag;
  RK_CUDA_TRY(cudaMalloc(&s->node_q, sizeof(int32_t) * (s->nnodes + 5)));
  RK_CUDA_TRY(cudaMalloc(&s->node_off, sizeof(int32_t) * (s->nnodes + 5)));
  RK_CUDA_TRY(cudaMalloc(&s->row_node, sizeof(int32_t) * (s->M2 + 1)));
  node_fill_kernel<<<grid, 256>>>(key2, flag, pos, tot, s->bs, s->node_q, s->node_off);
  count_launch();
  const int32_t end = (int32_t)tot;
  RK_CUDA_TRY(cudaMemcpy(s->node_off + s->nnodes, &end, sizeof(int32_t), cudaMemcpyHostToDevice));
  row_node_kernel<<<(int)ceil_div(s->M2 + 1, 256), 256>>>(s->node_q, s->nnodes, s->M1, s->M2, s->row_node);
  count_launch();
  RK_LAUNCH_CHECK();
  RK_CUDA_TRY(cudaDeviceSynchronize());
  {  // largest contribution count of a row pair (2k, 2k+1): sizes pass 1's product staging
    std::vector<int32_t> rn(s->M2 + 1), no(s->nnodes + 1);
    RK_CUDA_TRY(cudaMemcpy(rn.data(), s->row_node, sizeof(int32_t) * rn.size(), cudaMemcpyDeviceToHost));
    RK_CUDA_TRY(cudaMemcpy(no.data(), s->node_off, sizeof(int32_t) * no.size(), cudaMemcpyDeviceToHost));
    s->max_pair_ent = 0;
    s->max_half_ent = 0;
    for (int y = 0; y < s->M2; y += 2) {
      const int a0 = rn[y], a1 = rn[std::min(y + 2, s->M2)];
      const int am = a0 + (a1 - a0 + 1) / 2;   // the split-length pass 1 gives each CTA half the nodes
      s->max_pair_ent = std::max<int64_t>(s->max_pair_ent, no[a1] - no[a0]);
      s->max_half_ent = std::max<int64_t>(s->max_half_ent, std::max(no[am] - no[a0], no[a1] - no[am]));
    }
    // per row pair p: {first node, first node of row 2p+1, first contribution, contributions
    // of the first half of its nodes (where the split-length pass 1's second CTA starts)}; entry
    // npairs is the end sentinel, so a pair reads two adjacent records in one round trip
    const int npairs = (s->M2 + 1) / 2;
    std::vector<int4> pi(npairs + 1);
    for (int q = 0; q <= npairs; ++q) {
      const int y = std::min(2 * q, s->M2);
      const int a0 = rn[y], a1 = rn[std::min(y + 2, s->M2)];
      const int am = a0 + (a1 - a0 + 1) / 2;
      pi[q] = make_int4(a0, rn[std::min(y + 1, s->M2)], no[a0], no[am] - no[a0]);
    }
    RK_CUDA_TRY(cudaMalloc(&s->pair_info, sizeof(int4) * pi.size()));
    RK_CUDA_TRY(cudaMemcpy(s->pair_info, pi.data(), sizeof(int4) * pi.size(), cudaMemcpyHostToDevice));
  }
  RK_CUDA_TRY(cudaMalloc(&s->ent_wv, sizeof(double) * (std::max<int64_t>(tot, 1) + 2)));
  ent_value_kernel<<<grid, 256>>>(s->ent_w, s->wsort, tot, s->ent_wv);
  count_launch();
  RK_LAUNCH_CHECK();
  {  // fixed-stride per-pair plan blocks for small plans (pass 1 of one-wave launches)
    const int npairs = (s->M2 + 1) / 2;
    const int cap = (int)((s->max_pair_ent + 1) & ~int64_t(1));
    const int64_t stride = (16 + (int64_t)cap * 20 + 15) & ~int64_t(15);
    // only where pass 1 can be a one-wave launch (a few row pairs per SM); large grids run
    // the WIDE kernels, which keep the direct loads
    if (cap > 0 && cap <= 2048 && npairs <= 148 * 4 && stride * npairs <= (int64_t)64 << 20) {
      std::vector<int4> pi(npairs + 1);
      std::vector<int32_t> nq(s->nnodes + 1), no(s->nnodes + 1), ec(std::max<int64_t>(tot, 1));
      std::vector<double> ew(std::max<int64_t>(tot, 1));
      RK_CUDA_TRY(cudaMemcpy(pi.data(), s->pair_info, sizeof(int4) * pi.size(), cudaMemcpyDeviceToHost));
      RK_CUDA_TRY(cudaMemcpy(nq.data(), s->node_q, sizeof(int32_t) * nq.size(), cudaMemcpyDeviceToHost));
      RK_CUDA_TRY(cudaMemcpy(no.data(), s->node_off, sizeof(int32_t) * no.size(), cudaMemcpyDeviceToHost));
      if (tot > 0) {
        RK_CUDA_TRY(cudaMemcpy(ec.data(), s->ent_c, sizeof(int32_t) * tot, cudaMemcpyDeviceToHost));
        RK_CUDA_TRY(cudaMemcpy(ew.data(), s->ent_wv, sizeof(double) * tot, cudaMemcpyDeviceToHost));
      }
      std::vector<unsigned char> hb((size_t)stride * npairs, 0);
      for (int p = 0; p < npairs; ++p) {
        const int n0 = pi[p].x, n1 = pi[p].y, e0 = pi[p].z;
        const int nn = pi[p + 1].x - n0, cnt = pi[p + 1].z - e0;
        unsigned char* blk = hb.data() + (size_t)p * stride;
        int32_t* hdr = reinterpret_cast<int32_t*>(blk);
        hdr[0] = cnt;
        hdr[1] = nn;
        int2* rec = reinterpret_cast<int2*>(blk + 16);
        double* wv = reinterpret_cast<double*>(blk + 16 + (size_t)cap * 8);
        int32_t* ci = reinterpret_cast<int32_t*>(blk + 16 + (size_t)cap * 16);
        const int rowq = 2 * p * s->M1;
        for (int i = 0; i < nn; ++i) {   // as pass 1 forms it: end of products, 2 x + odd row
          const int odd = n0 + i >= n1;
          rec[i] = make_int2(no[n0 + i + 1] - e0, 2 * (nq[n0 + i] - rowq - odd * (int)s->M1) + odd);
        }
        for (int i = 0; i < cnt; ++i) {
          wv[i] = ew[e0 + i];
          ci[i] = ec[e0 + i];
        }
      }
      RK_CUDA_TRY(cudaMalloc(&s->pblk, hb.size()));
      RK_CUDA_TRY(cudaMemcpy(s->pblk, hb.data(), hb.size(), cudaMemcpyHostToDevice));
      s->pblk_stride = stride;
      s->pblk_cap = cap;
    }
  }
  cudaFree(tmp);
  cudaFree(key);
  cudaFree(key2);
  cudaFree(val);
  cudaFree(val2);
  cudaFree(flag);
  cudaFree(pos);
  return Status::ok();
}

void free_setup(rk_setup* s) {
  if (!s) return;
  int cur = 0;
  const bool swap = cudaGetDevice(&cur) == cudaSuccess && cur != s->device && cudaSetDevice(s->device) == cudaSuccess;
  free_workspaces(s);
  cudaFree(s->obs);
  cudaFree(s->base);
  cudaFree(s->weights);
  cudaFree(s->cond_var);
  cudaFree(s->perm);
  cudaFree(s->bsort);
  cudaFree(s->wsort);
  cudaFree(s->cell_start);
  cudaFree(s->node_q);
  cudaFree(s->node_off);
  cudaFree(s->row_node);
  cudaFree(s->ent_w);
  cudaFree(s->ent_c);
  cudaFree(s->ent_wv);
  cudaFree(s->pair_info);
  cudaFree(s->pblk);
  cudaFree(s->spec_q);
  cudaFree(s->spec_s);
  cudaFree(s->kn_chol_dev);
  cudaFree(s->ac_ker);
  cudaFree(s->emb.root_q);
  delete s;
  if (swap) cudaSetDevice(cur);
}

// weights + stencil base + cond_var for every observation of the setup (rapid.py:202-225);
// also used by rk_setup_time_weights to time the kernel on its own
static Status launch_weights(const rk_setup* s, int32_t* base, double* weights, double* cond_var, int* err,
                             cudaStream_t st) {
  const int64_t n = s->n;
  const int L = s->L, M = s->M;
  WArgs wa;
  wa.P = s->mat;
  wa.obs = s->obs;
  wa.n = n;
  wa.px0 = s->px0;
  wa.py0 = s->py0;
  wa.hx = s->grid.hx;
  wa.hy = s->grid.hy;
  wa.hix = (double)(s->M1 - 1) + 1.0e-9;
  wa.hiy = (double)(s->M2 - 1) + 1.0e-9;
  wa.L = L;
  wa.bs = s->bs;
  wa.M = M;
  wa.M1 = s->M1;
  wa.M2 = s->M2;
  wa.chol = s->kn_chol_dev;
  wa.base = base;
  wa.weights = weights;
  wa.cond_var = cond_var;
  wa.err = err;
  const size_t wsm = M <= 64 ? sizeof(double) * 2 * M * M : 0;
  const int wblocks = (int)std::min<int64_t>(ceil_div(n, 8), 148 * 16);
  const int mpl = (M + 31) / 32;
  auto launch_w = [&](auto kern) -> Status {
    RK_TRY(set_smem_attr((const void*)kern, wsm));
    kern<<<wblocks, 256, wsm, st>>>(wa);
    return Status::ok();
  };
  static const bool generic = getenv("RK_WEIGHTS_GENERIC") && atoi(getenv("RK_WEIGHTS_GENERIC"));
  if (L <= 4 && !generic) {
    const size_t wsl = sizeof(double) * (2 * M * M + M + 64);
    const int G = M <= 4 ? 8 : M <= 16 ? 2 : 1;
    const bool help = L == 3 && s->mat.half_n < 0;
    const int wbl = (int)std::min<int64_t>(ceil_div(ceil_div(n, G), 8), 148 * (help ? 2 : 3));   // resident
    auto launch_l = [&](auto kern) -> Status {
      RK_TRY(set_smem_attr((const void*)kern, wsl));
      kern<<<wbl, help ? 288 : 256, wsl, st>>>(wa);
      return Status::ok();
    };
    // RK_WEIGHTS_OB: observations per warp of the interleaved kernel for L = 3 / 4 (0 = the
    // one-observation kernels)
    // measured (tools/weights_sweep.py): 2 per warp for L = 4 (cfg5 0.233 -> 0.204 ms, cfg3 0.099 ->
    // 0.096 ms); for L = 3 the one-observation kernels are as fast or faster (cfg2 Bessel: 0.016 vs 0.025)
    static const int ob_env = getenv("RK_WEIGHTS_OB") ? atoi(getenv("RK_WEIGHTS_OB")) : -1;
    const int ob = ob_env >= 0 ? ob_env : (L == 4 ? 2 : 0);
    auto launch_ob = [&](auto kern, int obs_per_warp) -> Status {
      RK_TRY(set_smem_attr((const void*)kern, wsl));
      const int nb = (int)std::min<int64_t>(ceil_div(ceil_div(n, obs_per_warp), 8), 148 * 2);
      kern<<<nb, 256, wsl, st>>>(wa);
      return Status::ok();
    };
    // RK_WEIGHTS_MMA: the FP64 tensor-core blocked solve (weights_kernel_mma) for L >= 2
    static const int mma_env = getenv("RK_WEIGHTS_MMA") ? atoi(getenv("RK_WEIGHTS_MMA")) : -1;
    // default: L >= 3 with enough observations to fill the GPU with 8-observation tasks (measured:
    // cfg5 L = 4 0.204 -> 0.077 ms, cfg3 0.096 -> 0.050, cfg4 0.023 -> 0.014; cfg2's 1368
    // observations are 171 tasks, latency-bound: 0.016 ms one observation per warp vs 0.037)
    // (tools/k1_l2_probe.py, us per launch, substitution vs tensor-core: L = 2 n = 4096 7.3 vs 8.3,
    // n = 8192 12.4 vs 8.3, n = 50000 36.7 vs 20.6; L = 3 n = 2048 12.3 vs 14.4, n = 4096 22.6 vs 14.4)
    const bool use_mma = mma_env >= 0 ? (mma_env != 0 && L >= 2) : (L >= 3 ? n >= 3072 : L == 2 && n >= 6144);
    auto launch_mma = [&](auto kern, size_t smem) -> Status {
      RK_TRY(set_smem_attr((const void*)kern, smem));
      int per_sm = 0;
      RK_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
      int sms = 148;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, s->device);
      const int nb = (int)std::min<int64_t>(ceil_div(ceil_div(n, 8), 8), (int64_t)sms * std::max(per_sm, 1));
      kern<<<nb, 256, smem, st>>>(wa);
      return Status::ok();
    };
    if (use_mma) {
      const bool half = s->mat.half_n >= 0;
      if (L == 2) RK_TRY(launch_mma(half ? weights_kernel_mma<2, true> : weights_kernel_mma<2>, WMma<2>::smem_bytes()));
      else if (L == 3) RK_TRY(launch_mma(half ? weights_kernel_mma<3, true> : weights_kernel_mma<3>, WMma<3>::smem_bytes()));
      else RK_TRY(launch_mma(half ? weights_kernel_mma<4, true> : weights_kernel_mma<4>, WMma<4>::smem_bytes()));
    }
    else if (L == 1) RK_TRY(launch_l(weights_kernel_l<1>));
    else if (L == 2) RK_TRY(launch_l(weights_kernel_l<2>));
    else if (L >= 3 && ob >= 2) {
      if (L == 3) RK_TRY(ob >= 4 ? launch_ob(weights_kernel_ob<3, 4>, 4) : launch_ob(weights_kernel_ob<3, 2>, 2));
      else RK_TRY(ob >= 4 ? launch_ob(weights_kernel_ob<4, 4>, 4) : launch_ob(weights_kernel_ob<4, 2>, 2));
    }
    else if (L == 3 && help) RK_TRY(launch_l(weights_kernel_l<3, true>));
    else if (L == 3) RK_TRY(launch_l(weights_kernel_l<3>));
    else RK_TRY(launch_l(weights_kernel_l<4>));
  } else if (mpl <= 1) {
    RK_TRY(launch_w(weights_kernel<1>));
  } else if (mpl <= 2) {
    RK_TRY(launch_w(weights_kernel<2>));
  } else if (mpl <= 4) {
    RK_TRY(launch_w(weights_kernel<4>));
  } else if (mpl <= 8) {
    RK_TRY(launch_w(weights_kernel<8>));
  } else if (mpl <= 16) {
    RK_TRY(launch_w(weights_kernel<16>));
  } else {
    RK_TRY(launch_w(weights_kernel<32>));
  }
  count_launch();
  RK_LAUNCH_CHECK();
  return Status::ok();
}

static Status build_setup(const rk_model* model, const rk_grid* grid, int L, const double* obs_host,
                          int64_t n, rk_setup** out, int32_t* ridge_applied, bool grid_only = false) {
  if (n <= 0 && !grid_only) return Status::err(RK_DOMAIN, "build_setup requires at least one observation");
  if (L < 1) return Status::err(RK_DOMAIN, "neighbor order L must be >= 1");
  rk_setup* s = new rk_setup();
  std::unique_ptr<rk_setup, void (*)(rk_setup*)> guard(s, free_setup);
  RK_CUDA_TRY(cudaGetDevice(&s->device));
  s->model = *model;
  s->mat = make_matern_dev(*model);
  s->grid = *grid;
  s->L = L;
  s->bs = 2 * L;
  s->M = s->bs * s->bs;
  s->n = n;
  s->m1 = grid->m1;
  s->m2 = grid->m2;
  s->M1 = grid->m1 + grid->pad[0] + grid->pad[1];
  s->M2 = grid->m2 + grid->pad[2] + grid->pad[3];
  // padded_origin (gridding.py:44-48): origin - pad * spacing
  s->px0 = grid->x0 - (double)grid->pad[0] * grid->hx;
  s->py0 = grid->y0 - (double)grid->pad[2] * grid->hy;
  if (s->M > 1024) return Status::err(RK_DOMAIN, "neighbor order L > 16 not supported");
  *ridge_applied = 0;
  if (grid_only) {
    s->n = 0;
    goto spectrum;
  }
  {

  // K_N and its factor (rapid.py:190-193)
  std::vector<double> kn;
  RK_TRY(kn_matrix_dev(s, &kn));
  std::vector<double> chol = kn;
  if (!cholesky_lower(chol, s->M)) {
    const double ridge = 1.0e-12 * model->sigma2 * (double)(s->bs * s->bs);
    chol = kn;
    for (int i = 0; i < s->M; ++i) chol[(size_t)i * s->M + i] += ridge;
    if (!cholesky_lower(chol, s->M))
      return Status::err(RK_NUMERIC, "Cholesky of K_N failed even with ridge; reduce the neighbor "
                                     "order L or the smoothness nu");
    *ridge_applied = 1;
  }
  s->kn_chol = chol;
  chol_inverse(chol, s->M, &s->kn_inv);

  const int M = s->M;
  RK_CUDA_TRY(cudaMalloc(&s->obs, sizeof(double) * 2 * n));
  RK_CUDA_TRY(cudaMalloc(&s->base, sizeof(int32_t) * n));
  RK_CUDA_TRY(cudaMalloc(&s->weights, sizeof(double) * n * M));
  RK_CUDA_TRY(cudaMalloc(&s->cond_var, sizeof(double) * n));
  RK_CUDA_TRY(cudaMalloc(&s->kn_chol_dev, sizeof(double) * M * M));
  RK_CUDA_TRY(cudaMemcpy(s->obs, obs_host, sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
  RK_CUDA_TRY(cudaMemcpy(s->kn_chol_dev, chol.data(), sizeof(double) * M * M, cudaMemcpyHostToDevice));
  int* err = nullptr;
  RK_CUDA_TRY(cudaMalloc(&err, sizeof(int) * 4));
  int herr[4] = {INT_MAX, INT_MAX, 0, 0};
  RK_CUDA_TRY(cudaMemcpy(err, herr, sizeof(herr), cudaMemcpyHostToDevice));

  RK_TRY(launch_weights(s, s->base, s->weights, s->cond_var, err, 0));
  RK_CUDA_TRY(cudaMemcpy(herr, err, sizeof(herr), cudaMemcpyDeviceToHost));
  cudaFree(err);
  if (herr[0] != INT_MAX) {
    std::vector<double> o(2);
    RK_CUDA_TRY(cudaMemcpy(o.data(), s->obs + 2 * (int64_t)herr[0], 16, cudaMemcpyDeviceToHost));
    char b[256];
    snprintf(b, sizeof b, "location (%.17g, %.17g) outside padded grid coverage", o[0], o[1]);
    return Status::err(RK_DOMAIN, b);
  }
  if (herr[1] != INT_MAX) {
    std::vector<double> o(2);
    RK_CUDA_TRY(cudaMemcpy(o.data(), s->obs + 2 * (int64_t)herr[1], 16, cudaMemcpyDeviceToHost));
    char b[256];
    snprintf(b, sizeof b,
             "neighborhood of (%.17g, %.17g) exits the padded grid; padding contract violated",
             o[0], o[1]);
    return Status::err(RK_INTERNAL, b);
  }
  if (herr[2]) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");

  // cell-sorted structure for the deterministic gather (stable radix sort by base)
  RK_CUDA_TRY(cudaMalloc(&s->perm, sizeof(int32_t) * n));
  RK_CUDA_TRY(cudaMalloc(&s->bsort, sizeof(int32_t) * n));
  RK_CUDA_TRY(cudaMalloc(&s->wsort, sizeof(double) * n * M));
  const int64_t nb = (int64_t)s->M1 * s->M2;
  RK_CUDA_TRY(cudaMalloc(&s->cell_start, sizeof(int32_t) * (nb + 1)));
  int32_t* iota = nullptr;
  RK_CUDA_TRY(cudaMalloc(&iota, sizeof(int32_t) * n));
  iota_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 4096), 256>>>(iota, n);
  count_launch();
  size_t tmp_bytes = 0;
  int end_bit = 1;
  while (end_bit < 31 && ((int64_t)1 << end_bit) <= nb) ++end_bit;
  cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, s->base, s->bsort, iota, s->perm, (int)n, 0,
                                  end_bit);
  void* tmp = nullptr;
  RK_CUDA_TRY(cudaMalloc(&tmp, tmp_bytes ? tmp_bytes : 16));
  RK_CUDA_TRY(cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, s->base, s->bsort, iota, s->perm,
                                              (int)n, 0, end_bit));
  count_launch();
  cudaFree(tmp);
  cudaFree(iota);
  cell_start_kernel<<<(int)std::min<int64_t>(ceil_div(nb + 1, 256), 148 * 32), 256>>>(
      s->bsort, n, s->cell_start, nb);
  count_launch();
  permute_rows_kernel<<<(int)std::min<int64_t>(ceil_div(n * M, 256), 148 * 32), 256>>>(
      s->weights, s->perm, s->wsort, n, M);
  count_launch();
  RK_LAUNCH_CHECK();
  RK_TRY(build_sparse_gather(s));

  std::vector<double> cv(n);
  RK_CUDA_TRY(cudaMemcpy(cv.data(), s->cond_var, sizeof(double) * n, cudaMemcpyDeviceToHost));
  s->cond_var_min = *std::min_element(cv.begin(), cv.end());
  }
spectrum:
  // filter spectrum on the (2M-1)-rounded torus (rapid.py:72-86)
  auto next_fft_len = [](int64_t m) -> int64_t {
    if (m <= 1) return 1;
    int64_t best = -1;
    for (int64_t two = 1; two < 4 * m; two *= 2) {
      int64_t v = two;
      while (v < m) v *= 3;
      if (best < 0 || v < best) best = v;
    }
    return best;
  };
  s->rp1 = (int)next_fft_len(2 * (int64_t)s->M1 - 1);
  s->rp2 = (int)next_fft_len(2 * (int64_t)s->M2 - 1);
  s->p1 = s->rp1;
  s->p2 = grid_only ? s->rp2 : choose_exec_y(s);   // execution torus (see choose_exec_y)
  s->H1 = s->p1 / 2 + 1;
  s->Q2 = quarter_ld(s->p2);
  RK_TRY(setup_plans(s));
  RK_CUDA_TRY(cudaMalloc(&s->spec_q, sizeof(double) * (size_t)s->H1 * s->Q2));
  RK_TRY(spectrum_quarter(s->mat, grid->hx, grid->hy, s->p1, s->p2,
                          1.0 / ((double)s->p1 * (double)s->p2), s->spec_q, s->Q2, 0));
  RK_TRY(build_spec_split(s, 0));
  RK_TRY(build_alias_kernels(s));
  RK_CUDA_TRY(cudaDeviceSynchronize());
  *out = guard.release();
  return Status::ok();
}

}  // namespace rk

using namespace rk;

extern "C" {

const char* rk_last_error(void) { return rk::g_err.c_str(); }
int32_t rk_version(void) { return 1; }
int64_t rk_launch_count(void) { return rk::g_launches.load(); }

rk_status rk_matern_cov(const rk_model* model, const double* d_dev, double* out_dev, int64_t n,
                        void* stream) {
  auto run = [&]() -> Status {
    if (n <= 0) return Status::ok();
    const MaternDev P = make_matern_dev(*model);
    int* bad = nullptr;
    RK_CUDA_TRY(cudaMallocAsync((void**)&bad, sizeof(int), (cudaStream_t)stream));
    RK_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), (cudaStream_t)stream));
    matern_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 148 * 32), 256, 0,
                    (cudaStream_t)stream>>>(P, d_dev, out_dev, n, bad);
    count_launch();
    RK_LAUNCH_CHECK();
    int hb = 0;
    RK_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, (cudaStream_t)stream));
    RK_CUDA_TRY(cudaFreeAsync(bad, (cudaStream_t)stream));
    RK_CUDA_TRY(cudaStreamSynchronize((cudaStream_t)stream));
    if (hb) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");
    return Status::ok();
  };
  return (rk_status)finish(run());
}

rk_status rk_build_padded_grid(const double domain[4], int32_t m1, int32_t m2, int32_t L,
                               const double* obs_host, int64_t n, rk_grid* g) {
  auto run = [&]() -> Status {
    const double x0 = domain[0], x1 = domain[1], y0 = domain[2], y1 = domain[3];
    if (L < 1) return Status::err(RK_DOMAIN, "neighbor order L must be >= 1, got " + std::to_string(L));
    if (m1 < std::max(2, 2 * L) || m2 < std::max(2, 2 * L))
      return Status::err(RK_DOMAIN, "grid dims too small for neighbor order L=" + std::to_string(L) +
                                        "; need >= " + std::to_string(2 * L));
    if (!(x1 > x0 && y1 > y0)) return Status::err(RK_DOMAIN, "degenerate domain rectangle");
    g->x0 = x0;
    g->y0 = y0;
    g->hx = (x1 - x0) / (double)(m1 - 1);
    g->hy = (y1 - y0) / (double)(m2 - 1);
    g->m1 = m1;
    g->m2 = m2;
    for (int k = 0; k < 4; ++k) g->pad[k] = 0;
    if (n <= 0) return Status::ok();
    double* dobs = nullptr;
    int* out = nullptr;
    RK_CUDA_TRY(cudaMalloc(&dobs, sizeof(double) * 2 * n));
    RK_CUDA_TRY(cudaMalloc(&out, sizeof(int) * 5));
    RK_CUDA_TRY(cudaMemcpy(dobs, obs_host, sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
    int init[5] = {INT_MAX, INT_MIN, INT_MIN, INT_MIN, INT_MIN};
    RK_CUDA_TRY(cudaMemcpy(out, init, sizeof(init), cudaMemcpyHostToDevice));
    PadArgs a;
    a.obs = dobs;
    a.n = n;
    a.x0 = x0;
    a.y0 = y0;
    a.hx = g->hx;
    a.hy = g->hy;
    const double ex = 1.0e-9 * g->hx, ey = 1.0e-9 * g->hy;
    a.lox = x0 - ex;
    a.hix = x1 + ex;
    a.loy = y0 - ey;
    a.hiy = y1 + ey;
    a.L = L;
    a.m1 = m1;
    a.m2 = m2;
    a.out = out;
    pad_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 4096), 256>>>(a);
    count_launch();
    RK_LAUNCH_CHECK();
    int res[5];
    RK_CUDA_TRY(cudaMemcpy(res, out, sizeof(res), cudaMemcpyDeviceToHost));
    cudaFree(dobs);
    cudaFree(out);
    if (res[0] != INT_MAX) {
      char b[256];
      snprintf(b, sizeof b, "observation %d at (%.17g, %.17g) lies outside the domain", res[0],
               obs_host[2 * (int64_t)res[0]], obs_host[2 * (int64_t)res[0] + 1]);
      return Status::err(RK_DOMAIN, b);
    }
    for (int k = 0; k < 4; ++k) g->pad[k] = std::max(0, res[k + 1]);
    return Status::ok();
  };
  return (rk_status)finish(run());
}

rk_status rk_build_setup(const rk_model* model, const rk_grid* grid, int32_t L, const double* obs_host,
                         int64_t n, rk_setup** out, int32_t* ridge_applied) {
  int32_t r = 0;
  Status s = build_setup(model, grid, L, obs_host, n, out, &r);
  if (ridge_applied) *ridge_applied = r;
  return (rk_status)finish(s);
}

rk_status rk_grid_setup_create(const rk_model* model, const rk_grid* grid, rk_setup** out) {
  int32_t r = 0;
  return (rk_status)finish(build_setup(model, grid, 1, nullptr, 0, out, &r, true));
}

rk_status rk_setup_destroy(rk_setup* s) {
  free_setup(s);
  return RK_OK;
}

rk_status rk_setup_info(const rk_setup* s, int64_t* n_obs, int32_t* L, int32_t embed[2],
                        int32_t total[2]) {
  if (n_obs) *n_obs = s->n;
  if (L) *L = s->L;
  if (embed) { embed[0] = s->rp1; embed[1] = s->rp2; }   // the reference's torus (execution: rk_setup_exec_dims)
  if (total) { total[0] = s->M1; total[1] = s->M2; }
  return RK_OK;
}

rk_status rk_setup_time_weights(const rk_setup* s, void* stream, int32_t reps, float* ms_out) {
  auto run = [&]() -> Status {
    if (!s || s->n <= 0 || reps < 1) return Status::err(RK_DOMAIN, "time_weights needs a setup with observations");
    const cudaStream_t st = (cudaStream_t)stream;
    int32_t* base = nullptr;
    double *w = nullptr, *cv = nullptr;
    int* err = nullptr;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    RK_TRY(scratch_alloc((void**)&base, sizeof(int32_t) * s->n, st));
    RK_TRY(scratch_alloc((void**)&w, sizeof(double) * s->n * s->M, st));
    RK_TRY(scratch_alloc((void**)&cv, sizeof(double) * s->n, st));
    RK_TRY(scratch_alloc((void**)&err, sizeof(int) * 4, st));
    const int herr[4] = {INT_MAX, INT_MAX, 0, 0};
    RK_CUDA_TRY(cudaMemcpyAsync(err, herr, sizeof(herr), cudaMemcpyHostToDevice, st));
    RK_CUDA_TRY(cudaEventCreate(&e0));
    RK_CUDA_TRY(cudaEventCreate(&e1));
    RK_TRY(launch_weights(s, base, w, cv, err, st));   // warm-up
    RK_CUDA_TRY(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r) RK_TRY(launch_weights(s, base, w, cv, err, st));
    RK_CUDA_TRY(cudaEventRecord(e1, st));
    RK_CUDA_TRY(cudaEventSynchronize(e1));
    float ms = 0.f;
    RK_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
    *ms_out = ms / (float)reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    scratch_free(base, st);
    scratch_free(w, st);
    scratch_free(cv, st);
    scratch_free(err, st);
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    return Status::ok();
  };
  return (rk_status)finish(run());
}

// K1 of a predict step (SURVEY 8(d) T_predict = K1 + T_apply): stencil bases, weights and
// conditional variances of the setup's observations, recomputed into caller device buffers
// (base (n) int32, w (n, M), cv (n)) on `stream`; no host synchronisation
rk_status rk_setup_weights_into(const rk_setup* s, int32_t* base_dev, double* w_dev, double* cv_dev,
                                int32_t* err_dev, void* stream) {
  auto run = [&]() -> Status {
    if (!s || s->n <= 0) return Status::err(RK_DOMAIN, "weights need a setup with observations");
    return launch_weights(s, base_dev, w_dev, cv_dev, err_dev, (cudaStream_t)stream);
  };
  return (rk_status)finish(run());
}

rk_status rk_setup_copy_out(const rk_setup* s, int64_t* indices_host, double* weights_host,
                            double* cond_var_host, double* kn_inv_host) {
  auto run = [&]() -> Status {
    const int64_t nm = s->n * s->M;
    if (indices_host) {
      int64_t* d = nullptr;
      RK_CUDA_TRY(cudaMalloc(&d, sizeof(int64_t) * nm));
      expand_indices_kernel<<<(int)std::min<int64_t>(ceil_div(nm, 256), 4096), 256>>>(
          s->base, s->n, s->bs, s->M1, d);
      count_launch();
      RK_LAUNCH_CHECK();
      RK_CUDA_TRY(cudaMemcpy(indices_host, d, sizeof(int64_t) * nm, cudaMemcpyDeviceToHost));
      cudaFree(d);
    }
    if (weights_host)
      RK_CUDA_TRY(cudaMemcpy(weights_host, s->weights, sizeof(double) * nm, cudaMemcpyDeviceToHost));
    if (cond_var_host)
      RK_CUDA_TRY(cudaMemcpy(cond_var_host, s->cond_var, sizeof(double) * s->n, cudaMemcpyDeviceToHost));
    if (kn_inv_host) std::copy(s->kn_inv.begin(), s->kn_inv.end(), kn_inv_host);
    return Status::ok();
  };
  return (rk_status)finish(run());
}

rk_status rk_setup_exec_dims(const rk_setup* s, int32_t dims[2]) {
  dims[0] = s->p1;
  dims[1] = s->p2;
  return RK_OK;
}

rk_status rk_setup_copy_spectrum(const rk_setup* s, double* spectrum_host) {
  auto run = [&]() -> Status {
    // the reference torus' spectrum: the setup's own when it executes there, else built here
    const int p1 = s->rp1, p2 = s->rp2, H1 = p1 / 2 + 1, Q2 = quarter_ld(p2);
    std::vector<double> q((size_t)H1 * Q2);
    if (p1 == s->p1 && p2 == s->p2) {
      RK_CUDA_TRY(cudaMemcpy(q.data(), s->spec_q, sizeof(double) * q.size(), cudaMemcpyDeviceToHost));
    } else {
      double* d = nullptr;
      RK_CUDA_TRY(cudaMalloc(&d, sizeof(double) * q.size()));
      Status r = spectrum_quarter(s->mat, s->grid.hx, s->grid.hy, p1, p2, 1.0 / ((double)p1 * (double)p2), d, Q2, 0);
      if (r.good()) r = cudaMemcpy(q.data(), d, sizeof(double) * q.size(), cudaMemcpyDeviceToHost) == cudaSuccess
                            ? Status::ok() : Status::err(RK_CUDA, "spectrum copy failed");
      cudaFree(d);
      RK_TRY(r);
    }
    const double P = (double)p1 * (double)p2;
    for (int ky = 0; ky < p2; ++ky) {
      const int a = std::min(ky, p2 - ky);
      for (int kx = 0; kx < p1; ++kx) {
        const int b = std::min(kx, p1 - kx);
        spectrum_host[(size_t)ky * p1 + kx] = q[(size_t)b * Q2 + a] * P;
      }
    }
    return Status::ok();
  };
  return (rk_status)finish(run());
}

}  // extern "C"
