// Where does one FFT stage spend its cycles?  Copy of rk::fft_stage with clock64() probes
// (thread 0), run once per launch on one CTA.  Probes: after the modulo setup, after the
// loads, after twiddles + codelet, after the first barrier, after the stores + barrier.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/fft_stage_lat tools/fft_stage_lat.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_29284_b200/csrc/rk_fft.cuh"

using namespace rk;

template <int R, int K>
__device__ __forceinline__ void stage_probe(double2* __restrict__ buf, int n, int Ns, int t, int nthr,
                                            const double2* __restrict__ tw, long long* ts) {
  const int nb = n / R;
  double2 a[K][R];
  int outb[K];
  ts[0] = clock64();
  int jm = t % Ns;
  const int jstep = nthr % Ns;
  ts[1] = clock64();
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int j = t + q * nthr;
    outb[q] = -1;
    if (q > 0) { jm += jstep; if (jm >= Ns) jm -= Ns; }
    if (j < nb) {
#pragma unroll
      for (int k = 0; k < R; ++k) a[q][k] = buf[j + k * nb];
    }
  }
  double s = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) s += a[q][R - 1].x;
  if (s == 12345.678) buf[0].x = s;   // force the loads to complete before the probe
  ts[2] = clock64();
  jm = t % Ns;
#pragma unroll
  for (int q = 0; q < K; ++q) {
    const int j = t + q * nthr;
    if (q > 0) { jm += jstep; if (jm >= Ns) jm -= Ns; }
    if (j < nb) {
      if (jm != 0) {
        const double2 w1 = tw[jm];
        double2 wk = w1;
#pragma unroll
        for (int k = 1; k < R; ++k) {
          if (k > 1) wk = cmul(wk, w1);
          a[q][k] = cmul(a[q][k], wk);
        }
      }
      Dft<R, false>::run(a[q]);
      outb[q] = (j - jm) * R + jm;
    }
  }
  s = 0;
#pragma unroll
  for (int q = 0; q < K; ++q) s += a[q][R - 1].x;
  if (s == 12345.678) buf[1].x = s;
  ts[3] = clock64();
  __syncthreads();
  ts[4] = clock64();
#pragma unroll
  for (int q = 0; q < K; ++q)
    if (outb[q] >= 0) {
#pragma unroll
      for (int k = 0; k < R; ++k) buf[outb[q] + k * Ns] = a[q][k];
    }
  __syncthreads();
  ts[5] = clock64();
}

template <int R, int K>
__global__ void __launch_bounds__(512, 1) probe_kernel(int n, int Ns, int nthr, const double2* tw, long long* out) {
  extern __shared__ __align__(16) double2 sm[];
  for (int i = threadIdx.x; i < n; i += blockDim.x) sm[i] = make_double2(1e-3 * i, 1.0 / (1 + i));
  double2* tws = sm + n;
  for (int i = threadIdx.x; i < Ns; i += blockDim.x) tws[i] = tw[i];
  __syncthreads();
  long long ts[6];
  stage_probe<R, K>(sm, n, Ns, threadIdx.x, nthr, tws, ts);
  if (threadIdx.x == 0)
    for (int i = 0; i < 5; ++i) out[i] = ts[i + 1] - ts[i];
}

template <int R, int K>
void run(int n, int Ns, int nthr) {
  std::vector<double2> tw(Ns);
  for (int j = 0; j < Ns; ++j) tw[j] = make_double2(cos(6.283185307179586 * j / (Ns * R)), -sin(6.283185307179586 * j / (Ns * R)));
  double2* dtw; long long* d;
  cudaMalloc(&dtw, 16 * Ns); cudaMalloc(&d, 64);
  cudaMemcpy(dtw, tw.data(), 16 * Ns, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute((const void*)probe_kernel<R, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  for (int rep = 0; rep < 3; ++rep) probe_kernel<R, K><<<1, nthr, 16 * (n + Ns)>>>(n, Ns, nthr, dtw, d);
  cudaDeviceSynchronize();
  long long h[5];
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("R=%d K=%d n=%d Ns=%d nthr=%d: modulo %lld  loads %lld  twiddle+codelet %lld  barrier %lld  stores+barrier %lld  (cycles)\n",
         R, K, n, Ns, nthr, h[0], h[1], h[2], h[3], h[4]);
  cudaFree(dtw); cudaFree(d);
}

int main() {
  run<9, 2>(729, 9, 64);
  run<9, 1>(729, 9, 96);
  run<3, 1>(729, 27, 256);
  run<3, 6>(729, 27, 64);
  run<8, 2>(1152, 18, 96);
  return 0;
}
