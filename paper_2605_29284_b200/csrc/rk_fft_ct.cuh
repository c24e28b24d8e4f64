// In-place Cooley-Tukey FFT engine for the column (filter) pass: forward transform by
// decimation in frequency (natural order in, digit-reversed order out), pointwise product with
// the filter spectrum in digit-reversed order, inverse transform by decimation in time
// (digit-reversed in, natural order out).  Used where the spectral data never has to be in
// natural order -- the convolution's column pass.
//
// Why (vs the Stockham engine in rk_fft.cuh, measured on the cfg5 column pass: barrier, MIO and
// smem-latency stalls, FP64 pipe 38 %):
//  * a butterfly reads and writes the SAME R positions, so a stage needs one barrier (RAW to the
//    next stage), not two (Stockham's autosort store overwrites positions other threads have
//    yet to read), and nothing is held in registers across a barrier;
//  * after the first stage the line splits into R0 independent sub-arrays: every later stage is
//    local to one sub-array, owned by a group of G threads with its own named barrier (groups
//    drift apart, so one group's loads overlap another's arithmetic);
//  * the last forward stage (span 1, no twiddles), the spectrum product and the first inverse
//    stage run in registers on the same R elements: no smem round trip and no barrier between
//    the transforms.
//
// Stage s (DIF order, radices R_s from the FftPlan factorisation) works on sub-arrays of length
// N_s = n / (R_0 ... R_{s-1}) with span L_s = N_s / R_s: butterfly (q, j), j < L_s, reads
// x[q N_s + j + k L_s] (k < R_s); DIF: DFT_R then output k' times w_{N_s}^{j k'}; DIT (inverse):
// input k times conj(w_{N_s}^{j k}) then the inverse DFT_R.  Position p = sum_s d_s L_s of the
// forward output holds frequency f = sum_s d_s P_s, P_s = R_0 ... R_{s-1}.
#pragma once

#include "rk_fft.cuh"

namespace rk {

constexpr int CT_MAX_STAGES = 8;

struct CtPlan {
  int n, ns;                    // length, number of stages
  int rad[CT_MAX_STAGES];       // radix per stage (DIF order)
  int len[CT_MAX_STAGES];       // N_s
  int twb[CT_MAX_STAGES];       // offset of stage s's table w_{N_s}^j (j < L_s) in tw; -1 if L_s == 1
  int ntw;                      // table entries
  int G;                        // threads per group (stages >= 1), multiple of 32
  int nthr;                     // threads per line = R_0 * G
  const double2* tw;
};

// stage geometry helpers
__device__ __forceinline__ int ct_span(const CtPlan& p, int s) { return p.len[s] / p.rad[s]; }

// one DIF (forward) or DIT (inverse) butterfly at base with span L and sub-array length N
template <int R, bool INV>
__device__ __forceinline__ void ct_butterfly(double2* __restrict__ buf, int base, int L, int j,
                                             const double2* __restrict__ tws) {
  double2 a[R];
#pragma unroll
  for (int k = 0; k < R; ++k) a[k] = buf[base + k * L];
  if (INV && tws && j != 0) {   // DIT: conj twiddles on the inputs
    const double2 w1 = tws[j];
    double2 wk = w1;
#pragma unroll
    for (int k = 1; k < R; ++k) {
      if (k > 1) wk = cmul(wk, w1);
      a[k] = cmulc(a[k], wk);
    }
  }
  Dft<R, INV>::run(a);
  if (!INV && tws && j != 0) {  // DIF: twiddles on the outputs
    const double2 w1 = tws[j];
    double2 wk = w1;
#pragma unroll
    for (int k = 1; k < R; ++k) {
      if (k > 1) wk = cmul(wk, w1);
      a[k] = cmul(a[k], wk);
    }
  }
#pragma unroll
  for (int k = 0; k < R; ++k) buf[base + k * L] = a[k];
}

// barrier of the threads of one line (bid0) or of one group (bid0 + 1 + g)
__device__ __forceinline__ void ct_sync(int id, int count) {
  if (count == 32) __syncwarp();
  else group_sync(id, count);
}

// stage s of a line, all of its butterflies: s == 0 over the whole line (threads t < nthr),
// s >= 1 within group g's sub-array [g L_0, (g + 1) L_0) (threads tl < G of the group)
template <int R, bool INV>
__device__ __forceinline__ void ct_stage(double2* __restrict__ buf, const CtPlan& p, const double2* __restrict__ tw, int s, int t) {
  const int N = p.len[s], L = N / R;
  const double2* tws = p.twb[s] >= 0 ? tw + p.twb[s] : nullptr;
  if (s == 0) {
    for (int j = t; j < L; j += p.nthr) ct_butterfly<R, INV>(buf, j, L, j, tws);
  } else {
    const int g = t / p.G, tl = t - g * p.G;
    const int L0 = p.len[0] / p.rad[0];
    const int cnt = L0 / R;   // butterflies of this stage in the group's sub-array
    for (int b = tl; b < cnt; b += p.G) {
      const int q = b / L, j = b - q * L;
      ct_butterfly<R, INV>(buf, g * L0 + q * N + j, L, j, tws);
    }
  }
}

template <bool INV>
__device__ __forceinline__ void ct_stage_any(double2* __restrict__ buf, const CtPlan& p, const double2* __restrict__ tw, int s, int t) {
  switch (p.rad[s]) {
    case 9: ct_stage<9, INV>(buf, p, tw, s, t); break;
    case 8: ct_stage<8, INV>(buf, p, tw, s, t); break;
    case 6: ct_stage<6, INV>(buf, p, tw, s, t); break;
    case 4: ct_stage<4, INV>(buf, p, tw, s, t); break;
    case 3: ct_stage<3, INV>(buf, p, tw, s, t); break;
    default: ct_stage<2, INV>(buf, p, tw, s, t); break;
  }
}

// last stage fused: forward DFT_R (span 1), product with spec(f) per output, inverse DFT_R.
// spec(f) returns the real filter value of frequency f.
template <int R, class Spec>
__device__ __forceinline__ void ct_middle(double2* __restrict__ buf, const CtPlan& p, int t, const Spec& spec) {
  const int s = p.ns - 1;
  const int g = t / p.G, tl = t - g * p.G;
  const int L0 = p.len[0] / p.rad[0];
  const int cnt = L0 / R;
  int Pl = 1;   // P_{last} = R_0 ... R_{ns-2}
  for (int k = 0; k < s; ++k) Pl *= p.rad[k];
  for (int b = tl; b < cnt; b += p.G) {
    // frequency of output k' at position g L0 + b R + k': digits of b (mixed radix R_{s-1}, ...,
    // R_1 from the least significant), reversed
    int f = g, rem = b, P = Pl;
    for (int k = s - 1; k >= 1; --k) {
      const int r = p.rad[k];
      P /= r;
      const int d = rem % r;
      rem /= r;
      f += d * P;
    }
    double2 a[R];
    const int base = g * L0 + b * R;
#pragma unroll
    for (int k = 0; k < R; ++k) a[k] = buf[base + k];
    Dft<R, false>::run(a);
#pragma unroll
    for (int k = 0; k < R; ++k) a[k] = cscale(a[k], spec(f + k * Pl));
    Dft<R, true>::run(a);
#pragma unroll
    for (int k = 0; k < R; ++k) buf[base + k] = a[k];
  }
}

// Forward DIF, spectrum product, inverse DIT of the line at buf (in place).  All nthr threads of
// the line call it (t = thread index within the line); barrier ids bid0 (line) and bid0 + 1 + g
// (groups) -- bid0 == 0 is the whole CTA.
template <class Spec>
__device__ __forceinline__ void ct_filter_line(double2* __restrict__ buf, const CtPlan& p, const double2* __restrict__ tw, int t, int bid0,
                                               const Spec& spec) {
  const int g = t / p.G;
  const int gid = bid0 + 1 + g;
  // forward: stage 0 over the line, then the group-local stages
#pragma unroll 1
  for (int s = 0; s < p.ns - 1; ++s) {
    ct_stage_any<false>(buf, p, tw, s, t);
    if (s == 0) group_sync(bid0, p.nthr);
    else ct_sync(gid, p.G);
  }
  switch (p.rad[p.ns - 1]) {
    case 9: ct_middle<9>(buf, p, t, spec); break;
    case 8: ct_middle<8>(buf, p, t, spec); break;
    case 6: ct_middle<6>(buf, p, t, spec); break;
    case 4: ct_middle<4>(buf, p, t, spec); break;
    case 3: ct_middle<3>(buf, p, t, spec); break;
    default: ct_middle<2>(buf, p, t, spec); break;
  }
  // inverse: group-local stages back to stage 1, then stage 0 over the line
#pragma unroll 1
  for (int s = p.ns - 2; s >= 0; --s) {
    if (s == 0) group_sync(bid0, p.nthr);
    else ct_sync(gid, p.G);
    ct_stage_any<true>(buf, p, tw, s, t);
  }
  group_sync(bid0, p.nthr);
}

// ----------------------------------------------------------------- host planning
// Radices in the FftPlan order (9s, then 6 / 3, then 8s, then 2 / 4); group size from the local
// stages' butterfly counts.  false if n has no 2^a 3^b factorisation or needs more stages.
inline bool ct_plan_make(int n, CtPlan* p, int max_threads = 1024, int G_req = 0) {
  FftPlan f{};
  if (!fft_factor(n, &f, 0)) return false;
  int rad[FFT_MAX_STAGES];
  const int ns = fft_stage_list(f, rad);
  if (ns < 2 || ns > CT_MAX_STAGES) return false;
  p->n = n;
  p->ns = ns;
  int N = n, tw = 0;
  for (int s = 0; s < ns; ++s) {
    p->rad[s] = rad[s];
    p->len[s] = N;
    const int L = N / rad[s];
    p->twb[s] = L > 1 ? tw : -1;
    if (L > 1) tw += L;
    N = L;
  }
  p->ntw = tw;
  const int L0 = n / rad[0];
  // default group: enough threads for one butterfly each in the group's most common local stage
  // (radix R_1), the rest in rounds (e.g. 4374 = 9 9 9 6: 54 radix-9 butterflies -> G = 64,
  // the 81 radix-6 ones in two rounds)
  int G = G_req > 0 ? G_req : (L0 / rad[1] + 31) / 32 * 32;
  while (rad[0] * G > max_threads && G > 32) G -= 32;
  p->G = G;
  p->nthr = rad[0] * G;
  return G % 32 == 0 && p->nthr <= max_threads;
}

// twiddle tables (stage order): w_{N_s}^j = exp(-2 pi i j / N_s), j < L_s
template <class Vec, class Make>
inline void ct_twiddles(const CtPlan& p, Vec& out, Make make_c) {
  const long double PI_L = 3.141592653589793238462643383279502884L;
  for (int s = 0; s < p.ns; ++s) {
    const int L = p.len[s] / p.rad[s];
    if (L <= 1) continue;
    for (int j = 0; j < L; ++j) {
      const long double ang = 2.0L * PI_L * (long double)j / (long double)p.len[s];
      out.push_back(make_c((double)cosl(ang), (double)(-sinl(ang))));
    }
  }
}

}  // namespace rk
