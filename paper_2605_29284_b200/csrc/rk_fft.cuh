// Shared-memory Stockham FFT engine for lengths n = 2^a 3^b (fp64, complex).
//
// One "line" (a length-n transform) lives in shared memory as double2[n] and is
// transformed in place by `nthr` threads.  Each stage with radix R reads the R
// inputs x[j + k*n/R] of every butterfly j into registers, applies the twiddles
// W_{Ns R}^{(j mod Ns) k} (per-stage tables laid out [k-1][j mod Ns], so warp loads
// are coalesced), runs a register DFT_R codelet, then — after one barrier —
// scatters the outputs to y[(j - j mod Ns) R + j mod Ns + k Ns] (autosort).
//
// Throughput note (measured, tools/fft_bench.cu, tools/fft_stage_lat.cu + ncu): an fp64
// complex element is 16 bytes and every stage moves it through shared memory twice, and a
// radix-9 butterfly costs 88 FP64 instructions of codelet plus 60 of twiddles; on the cfg3
// column pass ncu shows the smem pipe ~57 % and the FP64 pipe ~43 % busy with barrier and
// short-scoreboard (smem) stalls on top -- no single unit saturated.  Larger radices
// (composite P x Q register codelets, radix 12-36, tried in an earlier revision) cut smem
// round trips, but every schedule that mixed several large-radix arms in one kernel made
// ptxas spill (as did a full power-table option: every extra code path costs registers);
// the shipped schedule is 9^a * {3,6} * 8^b * {2,4,4x4}.  Radix-3 family first, so the
// first (Ns = 1) stage writes with an odd stride (bank-conflict free for 16-byte elements).
//
// Several lines can share a CTA: every thread calls every stage (barriers are CTA
// wide); threads whose butterfly index runs past n/R just idle.
#pragma once

#include <cstring>

#include "rk_common.cuh"

namespace rk {

constexpr int FFT_MAX_STAGES = 16;
#ifndef RK_TW_TREE
#define RK_TW_TREE 0   // 1: balanced-tree twiddle powers (measured slower: more live registers, spills)
#endif
constexpr int kFftMagicSlots = FFT_MAX_STAGES / 4;   // double2 entries holding the stage divisors

// n = 9^n9 * r3 * 8^n8 * r2.  Kept as counts (not a radix array) so the stage
// code is straight-line per radix with only small runtime arms: a switch over many
// large-radix arms (or any switch inside the stage loop) makes ptxas keep every
// arm's registers live at once and spill.
struct FftPlan {
  int n;                       // transform length
  int nstages;
  int nthr;                    // threads cooperating on one line (multiple of 32)
  int n9, r3, n8, r2;          // r3 in {1,3,6}, r2 in {1,2,4,16}; 16 = two radix-4 stages
  int ntw;                     // entries of the stage twiddle table (sum of Ns > 1), plus
                               // kFftMagicSlots trailing entries holding, per stage,
                               // ceil(2^32 / Ns) as uint32 (j mod Ns by a multiply-high)
  int wide;                    // 0 normal; 1 spread (one butterfly per thread, <= 512 threads);
                               // 2 built for the WIDE kernels (fft_kmax_wide butterflies per thread);
                               // 3 split radix-9 stages (fft_stage9_split, three lanes each)
  const double2* tw;           // per-stage twiddles, see fft_stage_twiddles()
};

// Cooperative copy of the plan's twiddle table into shared memory (caller syncs before
// the first fft_line that uses it); returns a plan that reads from smem.
__device__ __forceinline__ FftPlan fft_twiddles_to_smem(const FftPlan& pl, double2* dst) {
  for (int i = threadIdx.x; i < pl.ntw; i += blockDim.x) dst[i] = __ldg(&pl.tw[i]);
  FftPlan p = pl;
  p.tw = dst;
  return p;
}

// The same copy split in two so a cold table read does not serialise with the kernel's
// other global round trips: twiddles_prefetch issues the loads into registers (nothing waits
// on them), twiddles_commit stores them (and any remainder) later; caller syncs after.
struct TwPrefetch {
  double2 v[2];
};
__device__ __forceinline__ TwPrefetch twiddles_prefetch(const FftPlan& pl) {
  TwPrefetch r;
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    r.v[k] = i < pl.ntw ? __ldg(&pl.tw[i]) : make_double2(0.0, 0.0);
  }
  return r;
}
__device__ __forceinline__ FftPlan twiddles_commit(const FftPlan& pl, const TwPrefetch& r, double2* dst) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int i = threadIdx.x + k * blockDim.x;
    if (i < pl.ntw) dst[i] = r.v[k];
  }
  for (int i = threadIdx.x + 2 * blockDim.x; i < pl.ntw; i += blockDim.x) dst[i] = __ldg(&pl.tw[i]);
  FftPlan p = pl;
  p.tw = dst;
  return p;
}

// butterflies each thread keeps in registers for a stage of radix R
// WIDE kernels (__launch_bounds__(1024): 64 registers) hold one radix-8/9 butterfly or two
// smaller ones per thread, so a line spreads over up to 1024 threads and an SM keeps 32
// FFT warps resident instead of 16
// (radix 3: three, the registers of one radix-9 butterfly -- an odd line 3 9^a, e.g. 2187, then
// needs n / 9 threads instead of n / 6, so its radix-9 stages keep every thread busy)
__host__ __device__ constexpr int fft_kmax_wide(int r) { return r >= 8 ? 1 : r == 3 ? 3 : 2; }
// threads per SM (and at most per line) of the WIDE kernels' launch bound
constexpr int kFftWideThreads = 1024;
// resident threads per SM of the split-radix-9 kernels (launch bound 576: <= 113 registers,
// two 288-thread lines of a 729-point transform per SM)
constexpr int kFftSplitThreads = 576;
__host__ __device__ constexpr int fft_sm_threads(int wide) {
  return wide == 2 ? kFftWideThreads : wide == 3 ? kFftSplitThreads : 512;
}
__host__ __device__ constexpr int fft_kmax(int r) {
  return r == 2 ? 9 : r == 3 ? 6 : r == 4 ? 4 : r == 6 ? 3 : r == 8 ? 2 : r == 9 ? 2 : r == 12 ? 2 : 1;
}

// ----------------------------------------------------------------- codelets
// forward: y_k = sum_q x_q exp(-2 pi i q k / R); inverse: + sign (unnormalised)

// multiply by -i (forward) or +i (inverse)
template <bool INV>
__device__ __forceinline__ double2 mul_mi(double2 a) {
  return INV ? make_double2(-a.y, a.x) : make_double2(a.y, -a.x);
}

template <bool INV>
__device__ __forceinline__ void dft2(double2& a, double2& b) {
  double2 t = a;
  a = cadd(t, b);
  b = csub(t, b);
}

template <bool INV>
__device__ __forceinline__ void dft3(double2& a, double2& b, double2& c) {
  const double S3 = 8.66025403784438596588e-01;  // sin(2 pi / 3)
  double2 t1 = cadd(b, c);
  double2 t2 = make_double2(fma(-0.5, t1.x, a.x), fma(-0.5, t1.y, a.y));
  double2 d = csub(b, c);
  double2 m = mul_mi<INV>(make_double2(S3 * d.x, S3 * d.y));
  a = cadd(a, t1);
  b = cadd(t2, m);
  c = csub(t2, m);
}

template <bool INV>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  double2 t0 = cadd(x0, x2), t1 = csub(x0, x2);
  double2 t2 = cadd(x1, x3), t3 = mul_mi<INV>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

template <int R, bool INV>
struct Dft;

template <bool INV>
struct Dft<2, INV> {
  static __device__ __forceinline__ void run(double2* a) { dft2<INV>(a[0], a[1]); }
};
template <bool INV>
struct Dft<3, INV> {
  static __device__ __forceinline__ void run(double2* a) { dft3<INV>(a[0], a[1], a[2]); }
};
template <bool INV>
struct Dft<4, INV> {
  static __device__ __forceinline__ void run(double2* a) { dft4<INV>(a[0], a[1], a[2], a[3]); }
};

template <bool INV>
struct Dft<8, INV> {
  static __device__ __forceinline__ void run(double2* a) {
    const double R2 = 7.07106781186547572737e-01;
    double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6];
    double2 o0 = a[1], o1 = a[3], o2 = a[5], o3 = a[7];
    dft4<INV>(e0, e1, e2, e3);
    dft4<INV>(o0, o1, o2, o3);
    // o_k *= w8^k
    double2 w1, w3;
    if (!INV) {
      w1 = make_double2(R2 * (o1.x + o1.y), R2 * (o1.y - o1.x));     // (1 - i)/sqrt2
      w3 = make_double2(R2 * (o3.y - o3.x), -R2 * (o3.x + o3.y));    // (-1 - i)/sqrt2
    } else {
      w1 = make_double2(R2 * (o1.x - o1.y), R2 * (o1.y + o1.x));     // (1 + i)/sqrt2
      w3 = make_double2(-R2 * (o3.x + o3.y), R2 * (o3.x - o3.y));    // (-1 + i)/sqrt2
    }
    double2 w2 = mul_mi<INV>(o2);
    a[0] = cadd(e0, o0); a[4] = csub(e0, o0);
    a[1] = cadd(e1, w1); a[5] = csub(e1, w1);
    a[2] = cadd(e2, w2); a[6] = csub(e2, w2);
    a[3] = cadd(e3, w3); a[7] = csub(e3, w3);
  }
};

// 6 = 3 x 2 (Cooley-Tukey, twiddles w6^1 = (1/2, -sqrt3/2), w6^2 = (-1/2, -sqrt3/2))
template <bool INV>
struct Dft<6, INV> {
  static __device__ __forceinline__ void run(double2* a) {
    const double S3 = 8.66025403784438596588e-01;
    double2 u00 = a[0], u01 = a[3];
    double2 u10 = a[1], u11 = a[4];
    double2 u20 = a[2], u21 = a[5];
    dft2<INV>(u00, u01);
    dft2<INV>(u10, u11);
    dft2<INV>(u20, u21);
    const double sg = INV ? S3 : -S3;
    u11 = cmul(u11, make_double2(0.5, sg));
    u21 = cmul(u21, make_double2(-0.5, sg));
    dft3<INV>(u00, u10, u20);
    dft3<INV>(u01, u11, u21);
    a[0] = u00; a[2] = u10; a[4] = u20;
    a[1] = u01; a[3] = u11; a[5] = u21;
  }
};

// 9 = 3 x 3 with twiddles w9^1, w9^2, w9^4
template <bool INV>
struct Dft<9, INV> {
  static __device__ __forceinline__ void run(double2* a) {
    const double C1 = 7.66044443118978013452e-01, S1 = 6.42787609686539362919e-01;
    const double C2 = 1.73648177666930358942e-01, S2 = 9.84807753012208020316e-01;
    const double C4 = -9.39692620785908427905e-01, S4 = 3.42020143325668712908e-01;
    const double sg = INV ? 1.0 : -1.0;
    double2 u[3][3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      u[r][0] = a[r];
      u[r][1] = a[r + 3];
      u[r][2] = a[r + 6];
      dft3<INV>(u[r][0], u[r][1], u[r][2]);
    }
    u[1][1] = cmul(u[1][1], make_double2(C1, sg * S1));
    u[1][2] = cmul(u[1][2], make_double2(C2, sg * S2));
    u[2][1] = cmul(u[2][1], make_double2(C2, sg * S2));
    u[2][2] = cmul(u[2][2], make_double2(C4, sg * S4));
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) {
      dft3<INV>(u[0][k1], u[1][k1], u[2][k1]);
      a[k1] = u[0][k1];
      a[k1 + 3] = u[1][k1];
      a[k1 + 6] = u[2][k1];
    }
  }
};

// ----------------------------------------------------------------- one stage
// Stage twiddles: each stage with Ns > 1 owns a block tw[jm] = W_{Ns R}^{jm}, jm < Ns (the
// k = 1 column); w^k for k >= 2 is formed by complex products, trading the smem/L1
// bandwidth the engine is bound by for FP64 work it has spare.  The whole table has
// sum(Ns) entries (~n / R_last), small enough to stage in shared memory per CTA
// (fft_twiddles_to_smem); warp loads are contiguous.  TWS: table in shared memory.
// j mod Ns for 0 <= j < 2^16 and 1 < Ns < 2^16 with m = ceil(2^32 / Ns): exact (the rounding
// error of m contributes < j / 2^32 < 1 / Ns to the quotient)
// (m == 0: plain modulo -- the CS row generator keeps it: measured, in that 64-register kernel
// the divisor table pointer and stage index cost spills)
__device__ __forceinline__ int mod_magic(int j, int Ns, uint32_t m) {
  return Ns == 1 ? 0 : m == 0 ? j % Ns : j - Ns * (int)__umulhi((uint32_t)j, m);
}

// Barrier of the threads working on one line: the whole CTA (id 0) or, when a CTA holds several
// independent lines, a named barrier per line (id 1 + line, count = the line's threads) so the
// lines' stages drift apart and one line's arithmetic overlaps another's shared-memory phases.
__device__ __forceinline__ void group_sync(int id, int count) {
  if (id == 0) __syncthreads();
  else asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

// Element hooks of the first / last stage (fft_line_pp): Pre(i, v) transforms element i of the
// stage's input as it is loaded, Post(i, v) element i of its output as it is stored.
struct FftNoOp {
  __device__ __forceinline__ double2 operator()(int, double2 v) const { return v; }
};

// SWZ (power-of-two lines, radix 8 only): the Ns = 1 stage of a 2^a line stores butterfly j's
// outputs at 8 j + k -- a 128-byte lane stride, all eight lanes of a quarter warp on the same four
// banks (8-way conflicts on every store; measured: the 8192^2 torus ran slower than 8748^2).
// SWZ = 1 stores them at 8 j + (k ^ (j & 7)) instead (conflict-free), and SWZ = 2 is the next
// stage loading element i from i ^ ((i >> 3) & 7) -- within an aligned group of eight lanes the
// XOR is a permutation, so those loads stay conflict-free.  Only the two stages' physical
// addresses change: same arithmetic, bitwise the same line.
// SWZ = 3 / 4, the same for lines that start with the radix-6 stage (6 9^a ..., e.g. 4374): butterfly
// j's outputs go to 6 j + k, so lanes j and j + 4 of a quarter warp share banks (2-way conflicts on
// every store of that stage; ncu counted them as ~9 % of the column pass's shared-memory
// wavefronts).  Element i lives at i ^ ((i >> 3) & 1) between the two stages: conflict-free for the
// stores and, the next stage's n / R being even, for its loads (checked exhaustively on the host).
template <int R, bool INV, bool TWS = false, bool WIDE = false, class Pre = FftNoOp, class Post = FftNoOp,
          int SWZ = 0>
__device__ __forceinline__ void fft_stage(double2* __restrict__ buf, int n, int Ns, int t, int nthr,
                                          const double2* __restrict__ tw, uint32_t nsm, int bid = 0,
                                          const Pre& pre = Pre(), const Post& post = Post()) {
  static_assert(SWZ == 0 || (SWZ <= 2 && R == 8) || (SWZ == 3 && R == 6) || (SWZ == 4 && (R == 9 || R == 8)),
                "swizzled stages: radix 8 pairs, or radix 6 followed by radix 9 / 8");
  constexpr int K = WIDE ? fft_kmax_wide(R) : fft_kmax(R);
  const int nb = n / R;
  double2 a[K][R];
  int outb[K];
  // j mod Ns for j = t + q nthr, updated incrementally (one division per stage, not per butterfly)
  int jm = mod_magic(t, Ns, nsm);
  const int jstep = mod_magic(nthr, Ns, nsm);
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int j = t + q * nthr;
    outb[q] = -1;
    if (q > 0) {
      jm += jstep;
      if (jm >= Ns) jm -= Ns;
    }
    if (j < nb) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int i = j + k * nb;   // SWZ == 2: nb % 8 == 0, so (i >> 3) & 7 = ((j >> 3) + k (nb >> 3)) & 7
        a[q][k] = pre(i, buf[SWZ == 2 ? i ^ (((j >> 3) + k * (nb >> 3)) & 7) : SWZ == 4 ? i ^ ((i >> 3) & 1) : i]);
      }
      if (jm != 0) {
        const double2 w1 = TWS ? tw[jm] : __ldg(&tw[jm]);
#if RK_TW_TREE
        // powers by a balanced tree: w^k = w^hb w^(k - hb), hb the largest power of two below k
        // (dependency depth 3 for R = 9 instead of the running product's 7)
        double2 pw[R];
        pw[1] = w1;
#pragma unroll
        for (int k = 2; k < R; ++k) {
          const int hb = k > 4 ? 4 : k > 2 ? 2 : 1;
          pw[k] = cmul(pw[hb], pw[k - hb]);
        }
#pragma unroll
        for (int k = 1; k < R; ++k) a[q][k] = INV ? cmulc(a[q][k], pw[k]) : cmul(a[q][k], pw[k]);
#else
        double2 wk = w1;
#pragma unroll
        for (int k = 1; k < R; ++k) {
          if (k > 1) wk = cmul(wk, w1);
          a[q][k] = INV ? cmulc(a[q][k], wk) : cmul(a[q][k], wk);
        }
#endif
      }
      Dft<R, INV>::run(a[q]);
      outb[q] = (j - jm) * R + jm;
    }
  }
  group_sync(bid, nthr);
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (outb[q] >= 0) {
#pragma unroll
      for (int k = 0; k < R; ++k) {
        const int i = outb[q] + k * Ns;   // SWZ == 1: Ns = 1, outb = 8 j, so (i >> 3) & 7 = j & 7
        buf[SWZ == 1 ? outb[q] + (k ^ ((outb[q] >> 3) & 7)) : SWZ == 3 ? i ^ ((i >> 3) & 1) : i] = post(i, a[q][k]);
      }
    }
  }
  group_sync(bid, nthr);
}

// Radix-9 stage with each butterfly split over three lanes (the 3 x 3 form of Dft<9>): lane r
// of a triple loads x[j + (r + 3 m) nb], applies the same twiddle powers, runs the first DFT3
// and the internal twiddles, the triple transposes its 3 x 3 intermediate through two
// shuffle rounds, and lane k1 runs the second DFT3 and stores outputs k1, k1 + 3, k1 + 6.
// Ten butterflies per warp (lanes 30, 31 idle).  The arithmetic -- twiddle running products,
// codelet, rounding -- is the one of fft_stage<9>, so every plan gives bitwise the same line;
// what changes is the serial FP64 work per thread (~72 instead of ~148 instructions), which
// is what a radix-9 stage of a latency-bound line waits on.
template <bool INV, bool TWS>
__device__ __forceinline__ void fft_stage9_split(double2* __restrict__ buf, int n, int Ns, int t, int nthr,
                                                 const double2* __restrict__ tw, uint32_t nsm, int bid = 0) {
  const double C1 = 7.66044443118978013452e-01, S1 = 6.42787609686539362919e-01;
  const double C2 = 1.73648177666930358942e-01, S2 = 9.84807753012208020316e-01;
  const double C4 = -9.39692620785908427905e-01, S4 = 3.42020143325668712908e-01;
  const double sg = INV ? 1.0 : -1.0;
  const int nb = n / 9;
  const int lane = t & 31;
  const int sub = lane / 3, r = lane - 3 * sub;
  const int j = (t >> 5) * 10 + sub;
  const bool valid = lane < 30 && j < nb;
  const int jm = valid ? mod_magic(j, Ns, nsm) : 0;
  double2 c0 = make_double2(0.0, 0.0), c1 = c0, c2 = c0;
  if (valid) {
    double2 a0 = buf[j + r * nb], a1 = buf[j + (r + 3) * nb], a2 = buf[j + (r + 6) * nb];
    if (jm != 0) {   // powers w^r, w^(r+3), w^(r+6) from the running product of fft_stage
      const double2 w1 = TWS ? tw[jm] : __ldg(&tw[jm]);
      double2 wp[9];
      wp[1] = w1;
#pragma unroll
      for (int k = 2; k < 9; ++k) {
#if RK_TW_TREE
        const int hb = k > 4 ? 4 : k > 2 ? 2 : 1;   // as fft_stage (bitwise the same powers)
        wp[k] = cmul(wp[hb], wp[k - hb]);
#else
        wp[k] = cmul(wp[k - 1], w1);
#endif
      }
      const double2 wr = r == 1 ? wp[1] : wp[2];
      const double2 wr3 = r == 0 ? wp[3] : r == 1 ? wp[4] : wp[5];
      const double2 wr6 = r == 0 ? wp[6] : r == 1 ? wp[7] : wp[8];
      if (r) a0 = INV ? cmulc(a0, wr) : cmul(a0, wr);
      a1 = INV ? cmulc(a1, wr3) : cmul(a1, wr3);
      a2 = INV ? cmulc(a2, wr6) : cmul(a2, wr6);
    }
    dft3<INV>(a0, a1, a2);
    if (r) {   // internal twiddles w9^(r k1)
      a1 = cmul(a1, r == 1 ? make_double2(C1, sg * S1) : make_double2(C2, sg * S2));
      a2 = cmul(a2, r == 1 ? make_double2(C2, sg * S2) : make_double2(C4, sg * S4));
    }
    c0 = a0;
    c1 = a1;
    c2 = a2;
  }
  // transpose within the triple: lane r ends with d_m = C_m[r] (m = the sender's r); only
  // compile-time register names (a runtime array index would spill to local memory)
  const double2 own = r == 0 ? c0 : r == 1 ? c1 : c2;
  double2 d0 = own, d1 = own, d2 = own;
#pragma unroll
  for (int rd = 1; rd < 3; ++rd) {
    const int give = r + rd >= 3 ? r + rd - 3 : r + rd;      // C_self[(r + rd) % 3]
    const double2 v = give == 0 ? c0 : give == 1 ? c1 : c2;
    const int from = r - rd < 0 ? r - rd + 3 : r - rd;       // sender's r
    const int src = 3 * sub + from;
    double2 got;
    got.x = __shfl_sync(0xffffffffu, v.x, src);
    got.y = __shfl_sync(0xffffffffu, v.y, src);
    if (from == 0) d0 = got;
    else if (from == 1) d1 = got;
    else d2 = got;
  }
  if (valid) dft3<INV>(d0, d1, d2);
  group_sync(bid, nthr);
  if (valid) {
    const int ob = (j - jm) * 9 + jm;
    buf[ob + r * Ns] = d0;
    buf[ob + (r + 3) * Ns] = d1;
    buf[ob + (r + 6) * Ns] = d2;
  }
  group_sync(bid, nthr);
}

// Full transform of the line at `buf` by thread t (0 <= t < pl.nthr or idle beyond).
// Must be called by every thread of the CTA (contains barriers).  FM (FFT mode): 0 normal /
// spread plans, 1 WIDE (64-register kernels), 2 split radix-9 stages.
// PSW: swizzled first pair of stages (fft_stage SWZ), a mask: 1 = power-of-two lines (8 8 ...),
// 2 = lines starting 6 9 ... (each costs one more stage body in the kernel).
// FAM 1: the caller guarantees a line 6 9^a, a >= 2 (fft_family69) and PSW & 2: only those two stage
// bodies are compiled in (the hot kernels are sensitive to their code size).
inline bool fft_family69(const FftPlan& pl) { return pl.r3 == 6 && pl.n9 >= 2 && pl.n8 == 0 && pl.r2 == 1; }
template <bool INV, bool TWS = false, int FM = 0, bool MAG = true, int PSW = 0, int FAM = 0>   // MAG: magic-divisor modulo
__device__ __forceinline__ void fft_line(double2* __restrict__ buf, const FftPlan& pl, int t, int bid = 0) {
  constexpr bool WIDE = FM >= 1;   // split plans also keep the small register footprint elsewhere
  const int n = pl.n, nthr = pl.nthr;
  const double2* tw = pl.tw;   // stage 1 (Ns = 1) needs no twiddles and has no block
  const uint32_t* mg = reinterpret_cast<const uint32_t*>(pl.tw + pl.ntw - kFftMagicSlots);
  int Ns = 1, si = 0;   // si: stage index (magic divisors)
  if (FAM == 1) {
    static_assert(FAM != 1 || ((PSW & 2) && FM == 1 && MAG), "family kernels: WIDE, swizzled, magic divisors");
    fft_stage<6, INV, TWS, WIDE, FftNoOp, FftNoOp, 3>(buf, n, 1, t, nthr, tw, 0u, bid);
    fft_stage<9, INV, TWS, WIDE, FftNoOp, FftNoOp, 4>(buf, n, 6, t, nthr, tw, mg[1], bid);
    tw += 6;
    Ns = 54;
    si = 2;
#pragma unroll 1
    for (int s = 1; s < pl.n9; ++s) {
      fft_stage<9, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, mg[si], bid);
      tw += Ns;
      Ns *= 9;
      ++si;
    }
    return;
  }
  // the radix-6 / 3 stage first: as the Ns = 1 stage it needs no twiddles, which keeps the WIDE
  // kernels' two-butterfly radix-6 stage inside 64 registers
  int s9 = 0;
  if (pl.r3 == 6) {
    if ((PSW & 2) && FM != 2 && pl.n9 >= 1) {   // swizzled radix-6 / first radix-9 pair (fft_stage SWZ 3 / 4)
      fft_stage<6, INV, TWS, WIDE, FftNoOp, FftNoOp, 3>(buf, n, 1, t, nthr, tw, 0u, bid);
      ++si;
      fft_stage<9, INV, TWS, WIDE, FftNoOp, FftNoOp, 4>(buf, n, 6, t, nthr, tw, MAG ? mg[si] : 0u, bid);
      tw += 6;
      Ns = 54;
      ++si;
      s9 = 1;
    } else {
      fft_stage<6, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, MAG ? mg[si] : 0u, bid);
      Ns *= 6;
      ++si;
    }
  } else if (pl.r3 == 3) {
    fft_stage<3, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, MAG ? mg[si] : 0u, bid);
    Ns *= 3;
    ++si;
  }
#pragma unroll 1
  for (int s = s9; s < pl.n9; ++s) {
    if (FM == 2) fft_stage9_split<INV, TWS>(buf, n, Ns, t, nthr, tw, MAG ? mg[si] : 0u, bid);
    else fft_stage<9, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, MAG ? mg[si] : 0u, bid);
    if (Ns > 1) tw += Ns;
    Ns *= 9;
    ++si;
  }
  int s8 = 0;
  if ((PSW & 1) && Ns == 1 && pl.n8 >= 2 && FM != 2) {   // power-of-two line: swizzled first pair of stages
    fft_stage<8, INV, TWS, WIDE, FftNoOp, FftNoOp, 1>(buf, n, 1, t, nthr, tw, 0u, bid);
    ++si;
    fft_stage<8, INV, TWS, WIDE, FftNoOp, FftNoOp, 2>(buf, n, 8, t, nthr, tw, MAG ? mg[si] : 0u, bid);
    tw += 8;
    Ns = 64;
    ++si;
    s8 = 2;
  }
#pragma unroll 1
  for (int s = s8; s < pl.n8; ++s) {
    fft_stage<8, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, MAG ? mg[si] : 0u, bid);
    if (Ns > 1) tw += Ns;
    Ns *= 8;
    ++si;
  }
  if (pl.r2 == 2) {
    fft_stage<2, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, MAG ? mg[si] : 0u, bid);
  } else if (pl.r2 >= 4) {
#pragma unroll 1
    for (int s = 0; s < (pl.r2 == 16 ? 2 : 1); ++s) {
      fft_stage<4, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, MAG ? mg[si] : 0u, bid);
      if (Ns > 1) tw += Ns;
      Ns *= 4;
      ++si;
    }
  }
}

// fft_line with hooks: pre on the first stage's loads, post on the last stage's stores (each a
// pass over the line and a barrier saved, e.g. the split-length twist before a forward transform
// and the spectrum product after it).  Schedules {3 or 6} 9^n9 only (fft_line_pp_ok); the stage
// arithmetic is fft_line's, so the transform is bitwise the same as hooks applied in passes.
inline bool fft_line_pp_ok(const FftPlan& pl) { return pl.r3 > 1 && pl.n9 >= 1 && pl.n8 == 0 && pl.r2 == 1; }
template <bool INV, bool TWS, int FM, class Pre, class Post, bool PSW = false, int FAM = 0>
__device__ __forceinline__ void fft_line_pp(double2* __restrict__ buf, const FftPlan& pl, int t, int bid,
                                            const Pre& pre, const Post& post) {
  constexpr bool WIDE = FM >= 1;
  const int n = pl.n, nthr = pl.nthr;
  const double2* tw = pl.tw;
  const uint32_t* mg = reinterpret_cast<const uint32_t*>(pl.tw + pl.ntw - kFftMagicSlots);
  int Ns, si = 1, s9 = 0;
  if (FAM == 1 || pl.r3 == 6) {
    if (FAM == 1 || (PSW && pl.n9 >= 2)) {   // swizzled radix-6 / first radix-9 pair, as fft_line
      fft_stage<6, INV, TWS, WIDE, Pre, FftNoOp, 3>(buf, n, 1, t, nthr, tw, mg[0], bid, pre, FftNoOp());
      fft_stage<9, INV, TWS, WIDE, FftNoOp, FftNoOp, 4>(buf, n, 6, t, nthr, tw, mg[1], bid);
      tw += 6;
      Ns = 54;
      si = 2;
      s9 = 1;
    } else if (FAM != 1) {
      fft_stage<6, INV, TWS, WIDE, Pre, FftNoOp>(buf, n, 1, t, nthr, tw, mg[0], bid, pre, FftNoOp());
      Ns = 6;
    }
  } else if (FAM != 1) {
    fft_stage<3, INV, TWS, WIDE, Pre, FftNoOp>(buf, n, 1, t, nthr, tw, mg[0], bid, pre, FftNoOp());
    Ns = 3;
  }
#pragma unroll 1
  for (int s = s9; s < pl.n9 - 1; ++s) {
    fft_stage<9, INV, TWS, WIDE>(buf, n, Ns, t, nthr, tw, mg[si], bid);
    tw += Ns;
    Ns *= 9;
    ++si;
  }
  fft_stage<9, INV, TWS, WIDE, FftNoOp, Post>(buf, n, Ns, t, nthr, tw, mg[si], bid, FftNoOp(), post);
}

// ----------------------------------------------------------------- host planning
inline int fft_stage_list(const FftPlan& pl, int* rad) {
  int ns = 0;
  if (pl.r3 > 1) rad[ns++] = pl.r3;
  for (int i = 0; i < pl.n9; ++i) rad[ns++] = 9;
  for (int i = 0; i < pl.n8; ++i) rad[ns++] = 8;
  if (pl.r2 == 16) {
    rad[ns++] = 4;
    rad[ns++] = 4;
  } else if (pl.r2 > 1) {
    rad[ns++] = pl.r2;
  }
  return ns;
}

// n = 2^a 3^b -> 9^(b/2) * r3 * 8^(a'/3) * r2 with r3 = 3 or 6 (b odd; 6 absorbs one
// factor 2 when a >= 1) and r2 = 2^(a' % 3), except that a trailing 8 * 2 becomes 4 * 4.
// wide = 1 ("spread"): for latency-bound launches with few lines, the same stages with one
// thread per butterfly (nthr = max n/R, at most 512) in the 128-register kernels: measured on
// B200, a radix-9 stage of a 729-point line takes ~1190 cycles with 2 butterflies per thread
// and ~700 with 1 (tools/fft_stage_lat), and the gather / epilogue phases get more
// memory-level parallelism.  Splitting the 9s into radix-3 stages was slower (6 x ~1100).
// wide = 2: for the 64-register WIDE kernels (fft_kmax_wide), up to 1024 threads per line
// and 1024 resident FFT threads per SM, for launches that do not fit the GPU in one wave.
inline bool fft_factor(int n, FftPlan* pl, int wide = 0) {
  int a = 0, b = 0, m = n;
  if (n < 1) return false;
  while (m % 2 == 0) { m /= 2; ++a; }
  while (m % 3 == 0) { m /= 3; ++b; }
  if (m != 1) return false;
  pl->n = n;
  pl->n9 = b / 2;
  pl->r3 = 1;
  if (b % 2 == 1) {
    if (a >= 1) { pl->r3 = 6; a -= 1; } else { pl->r3 = 3; }
  }
  pl->n8 = a / 3;
  pl->r2 = 1 << (a % 3);
  if (pl->r2 == 2 && pl->n8 >= 1) {   // 8 * 2 -> 4 * 4: a radix-2 stage has n/2 butterflies,
    pl->n8 -= 1;                        // which caps the one-per-thread (wide) plans
    pl->r2 = 16;
  }
  int rad[FFT_MAX_STAGES];
  pl->nstages = fft_stage_list(*pl, rad);
  int need = 1;
  for (int i = 0; i < pl->nstages; ++i) {
    const int nb = n / rad[i];
    const int k = fft_kmax(rad[i]);
    need = need > (nb + k - 1) / k ? need : (nb + k - 1) / k;
  }
  if (wide == 1) {   // one butterfly per thread where 512 threads allow it
    int mx = 1;
    for (int i = 0; i < pl->nstages; ++i) mx = mx > n / rad[i] ? mx : n / rad[i];
    need = need > (mx < 512 ? mx : 512) ? need : (mx < 512 ? mx : 512);
  } else if (wide == 3) {   // split radix-9 stages: 3 lanes per butterfly, 10 per warp;
    need = 1;               // the other radices as in the WIDE kernels
    for (int i = 0; i < pl->nstages; ++i) {
      const int nb = n / rad[i];
      const int k = rad[i] == 9 ? 0 : fft_kmax_wide(rad[i]);
      const int th = k ? (nb + k - 1) / k : (nb + 9) / 10 * 32;
      need = need > th ? need : th;
    }
  } else if (wide == 2) {   // fft_kmax_wide butterflies per thread, up to 1024 threads per line
    need = 1;
    for (int i = 0; i < pl->nstages; ++i) {
      const int nb = n / rad[i];
      const int k = fft_kmax_wide(rad[i]);   // nthr must stay <= kFftWideThreads (plan_for checks)
      need = need > (nb + k - 1) / k ? need : (nb + k - 1) / k;
    }
  }
  pl->wide = wide;
  pl->nthr = (need + 31) / 32 * 32;
  if (pl->nthr < 32) pl->nthr = 32;
  return true;
}

// host: per-stage twiddle table for a factored plan (entries in stage order, Ns > 1 only)
template <class Vec, class Make>
inline void fft_stage_twiddles(const FftPlan& pl, Vec& out, Make make_c) {
  int rad[FFT_MAX_STAGES];
  const int ns = fft_stage_list(pl, rad);
  const long double PI_L = 3.141592653589793238462643383279502884L;
  long long Ns = 1;
  for (int s = 0; s < ns; ++s) {
    const int R = rad[s];
    if (Ns > 1) {
      for (long long jm = 0; jm < Ns; ++jm) {
        const long double ang = 2.0L * PI_L * (long double)jm / (long double)(Ns * R);
        out.push_back(make_c((double)cosl(ang), (double)(-sinl(ang))));
      }
    }
    Ns *= R;
  }
  // trailing magic divisors: kFftMagicSlots entries = 4 * kFftMagicSlots uint32 (one per stage)
  uint32_t mg[4 * kFftMagicSlots] = {};
  Ns = 1;
  for (int s = 0; s < ns; ++s) {
    mg[s] = Ns > 1 ? (uint32_t)(((1ULL << 32) + (unsigned long long)Ns - 1) / (unsigned long long)Ns) : 0u;
    Ns *= rad[s];
  }
  for (int k = 0; k < kFftMagicSlots; ++k) {
    double v[2];
    memcpy(v, mg + 4 * k, sizeof v);
    out.push_back(make_c(v[0], v[1]));
  }
}

}  // namespace rk
