// Standalone microbenchmark of the smem Stockham engine (one line per CTA-slot,
// repeated in-smem transforms, no global I/O in the loop) to isolate FFT-core
// efficiency from data movement.  Variants: twiddles from global (L1/L2), from a
// shared-memory copy, or all-ones (timing only).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I include -o tools/fft_bench tools/fft_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#include "../paper_2605_29284_b200/csrc/rk_fft.cuh"

using namespace rk;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

template <int MODE>  // 0 global tw, 1 smem tw, 2 fake tw
__global__ void __launch_bounds__(512, 1) bench_kernel(FftPlan pl, int lpc, int reps, double2* out) {
  extern __shared__ __align__(16) double2 sm[];
  const int n = pl.n, nthr = pl.nthr;
  const int line = threadIdx.x / nthr, tl = threadIdx.x - line * nthr;
  double2* buf = sm + (size_t)line * n;
  double2* tws = sm + (size_t)lpc * n;
  FftPlan p2 = pl;
  if (MODE == 1) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) tws[i] = pl.tw[i];
    p2.tw = tws;
  }
  for (int i = tl; i < n; i += nthr) buf[i] = make_double2(1e-3 * i, 1.0 / (1 + i));
  __syncthreads();
  for (int r = 0; r < reps; ++r) {
    fft_line<false, MODE == 1>(buf, p2, tl);
    fft_line<true, MODE == 1>(buf, p2, tl);
  }
  if (tl == 0) out[blockIdx.x * lpc + line] = buf[1];
}

int main(int argc, char** argv) {
  int sizes[] = {216, 729, 1152, 2304, 4374, 8748};
  const int only = argc > 1 ? atoi(argv[1]) : 0;
  for (int n : sizes) {
    if (only && n != only) continue;
    FftPlan pl{};
    fft_factor(n, &pl);
    std::vector<double2> tw;
    fft_stage_twiddles(pl, tw, [](double c, double s) { return make_double2(c, s); });
    tw.resize(std::max<size_t>(tw.size(), n));
    double2* dtw; CK(cudaMalloc(&dtw, 16 * tw.size())); CK(cudaMemcpy(dtw, tw.data(), 16 * tw.size(), cudaMemcpyHostToDevice));
    pl.tw = dtw;
    int lpc = std::max(1, std::min(512 / pl.nthr, (int)(96 * 1024 / (16 * n))));
    const int ctas = 148 * 2;
    double2* out; CK(cudaMalloc(&out, 16 * ctas * lpc));
    const int reps = 20;
    for (int mode = 0; mode < 3; ++mode) {
      size_t smem = 16 * (size_t)n * lpc + (mode == 1 ? 16 * (size_t)n : 0);
      void (*k)(FftPlan, int, int, double2*) = mode == 0 ? bench_kernel<0> : mode == 1 ? bench_kernel<1> : bench_kernel<2>;
      CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      if (mode == 2) {  // fake twiddles: all (1,0)
        std::vector<double2> one(tw.size(), make_double2(1.0, 0.0));
        CK(cudaMemcpy(dtw, one.data(), 16 * tw.size(), cudaMemcpyHostToDevice));
      }
      k<<<ctas, lpc * pl.nthr, smem>>>(pl, lpc, 2, out);
      CK(cudaDeviceSynchronize());
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<ctas, lpc * pl.nthr, smem>>>(pl, lpc, reps, out);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ffts = 2.0 * reps * ctas * lpc;
      double flops = ffts * 5.0 * n * log2((double)n);   // conventional 5 n log2 n
      printf("n=%5d nthr=%3d lpc=%d mode=%s smem=%6zu  us/fft(line)=%.3f  GF(5nlogn)=%.0f\n", n, pl.nthr, lpc,
             mode == 0 ? "gtw " : mode == 1 ? "stw " : "fake", smem, ms * 1e3 / ffts * ctas * lpc / (148.0 * 2),
             flops / (ms * 1e-3) / 1e9);
    }
    CK(cudaFree(dtw)); CK(cudaFree(out));
  }
  return 0;
}
