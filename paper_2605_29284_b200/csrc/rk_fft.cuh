// Shared-memory Stockham FFT engine for lengths n = 2^a 3^b (fp64, complex).
//
// One "line" (a length-n transform) lives in shared memory as double2[n] and is
// transformed in place by `nthr` threads.  Each stage with radix R reads the R
// inputs x[j + k*n/R] of every butterfly j into registers, applies the twiddles
// W_{Ns R}^{(j mod Ns) k} from a global root table (L1-resident), runs a
// hand-written DFT_R codelet, then — after one barrier — scatters the outputs
// to y[(j - j mod Ns) R + j mod Ns + k Ns] (autosort, natural order at the end).
// Radices containing 3 are scheduled first so the small-Ns stages write with
// odd strides (bank-conflict free for 16-byte elements).
//
// Several lines can share a CTA: every thread calls every stage (barriers are
// CTA wide); threads whose butterfly index runs past n/R just idle.
#pragma once

#include "rk_common.cuh"

namespace rk {

constexpr int FFT_MAX_STAGES = 16;

// n = 9^n9 * r3 * 8^n8 * r2 with r3 in {1, 3, 6} and r2 in {1, 2, 4}; stages run in that
// order (radix-3 family first).  The schedule is kept as counts, not a radix array, so the
// stage code below is straight-line per radix: a runtime switch inside one loop makes ptxas
// keep every arm's registers live at once and spill.
struct FftPlan {
  int n;                       // transform length
  int nstages;
  int nthr;                    // threads cooperating on one line (multiple of 32)
  int n9, r3, n8, r2;
  const double2* tw;           // device table W[t] = exp(-2 pi i t / n), t in [0, n)
};

// butterflies each thread keeps in registers for a stage of radix R
__host__ __device__ constexpr int fft_kmax(int r) {
  return r == 2 ? 9 : r == 3 ? 6 : r == 4 ? 4 : r == 6 ? 3 : r == 8 ? 2 : r == 9 ? 2 : 1;
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
    // inner DFT2 over j (stride 3): pairs (a_r, a_{r+3}), r = 0,1,2
    double2 u00 = a[0], u01 = a[3];
    double2 u10 = a[1], u11 = a[4];
    double2 u20 = a[2], u21 = a[5];
    dft2<INV>(u00, u01);
    dft2<INV>(u10, u11);
    dft2<INV>(u20, u21);
    // twiddle u_{r,k1} *= w6^{r k1}: only k1 = 1 nontrivial
    const double sg = INV ? S3 : -S3;
    u11 = cmul(u11, make_double2(0.5, sg));
    u21 = cmul(u21, make_double2(-0.5, sg));
    // outer DFT3 over r for each k1 -> y[k1 + 2 k2]
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
template <int R, bool INV>
__device__ __forceinline__ void fft_stage(double2* __restrict__ buf, int n, int Ns, int t, int nthr,
                                          const double2* __restrict__ tw) {
  constexpr int K = fft_kmax(R);
  const int nb = n / R;
  const int tstep = n / (Ns * R);
  double2 a[K][R];
  int outb[K];
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int j = t + q * nthr;
    outb[q] = -1;
    if (j < nb) {
#pragma unroll
      for (int k = 0; k < R; ++k) a[q][k] = buf[j + k * nb];
      const int jm = j % Ns;
      if (jm != 0) {
        const int step = jm * tstep;
#pragma unroll
        for (int k = 1; k < R; ++k) {
          const double2 w = __ldg(&tw[k * step]);
          a[q][k] = INV ? cmulc(a[q][k], w) : cmul(a[q][k], w);
        }
      }
      Dft<R, INV>::run(a[q]);
      outb[q] = (j - jm) * R + jm;
    }
  }
  __syncthreads();
#pragma unroll
  for (int q = 0; q < K; ++q) {
    if (outb[q] >= 0) {
#pragma unroll
      for (int k = 0; k < R; ++k) buf[outb[q] + k * Ns] = a[q][k];
    }
  }
  __syncthreads();
}

// Full transform of the line at `buf` by thread t (0 <= t < pl.nthr or idle beyond).
// Must be called by every thread of the CTA (contains barriers).
template <bool INV>
__device__ __forceinline__ void fft_line(double2* __restrict__ buf, const FftPlan& pl, int t) {
  const int n = pl.n, nthr = pl.nthr;
  int Ns = 1;
#pragma unroll 1
  for (int s = 0; s < pl.n9; ++s) {
    fft_stage<9, INV>(buf, n, Ns, t, nthr, pl.tw);
    Ns *= 9;
  }
  if (pl.r3 == 6) {
    fft_stage<6, INV>(buf, n, Ns, t, nthr, pl.tw);
    Ns *= 6;
  } else if (pl.r3 == 3) {
    fft_stage<3, INV>(buf, n, Ns, t, nthr, pl.tw);
    Ns *= 3;
  }
#pragma unroll 1
  for (int s = 0; s < pl.n8; ++s) {
    fft_stage<8, INV>(buf, n, Ns, t, nthr, pl.tw);
    Ns *= 8;
  }
  if (pl.r2 == 4) fft_stage<4, INV>(buf, n, Ns, t, nthr, pl.tw);
  else if (pl.r2 == 2) fft_stage<2, INV>(buf, n, Ns, t, nthr, pl.tw);
}

// host: build a plan (radix schedule + thread count); twiddle table filled separately
bool fft_factor(int n, FftPlan* pl);

}  // namespace rk
