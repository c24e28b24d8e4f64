// Latency of one shared-memory FFT line (cycles per forward transform, thread 0's
// clock64) with one line per CTA and one CTA per SM -- the regime of small, latency-bound
// grids -- for the normal and the wide plan of each size.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -o tools/fft_latency tools/fft_latency.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2605_29284_b200/csrc/rk_fft.cuh"

using namespace rk;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s line %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void __launch_bounds__(512, 1) lat_kernel(FftPlan pl, int reps, long long* cyc, double2* out) {
  extern __shared__ __align__(16) double2 sm[];
  const int n = pl.n;
  double2* buf = sm;
  FftPlan p2 = fft_twiddles_to_smem(pl, sm + n);
  for (int i = threadIdx.x; i < n; i += blockDim.x) buf[i] = make_double2(1e-3 * i, 1.0 / (1 + i));
  __syncthreads();
  long long t0 = clock64();
  fft_line<false, true>(buf, p2, threadIdx.x);   // first transform: cold instruction cache
  long long t1 = clock64();
  fft_line<false, true>(buf, p2, threadIdx.x);   // second: warm
  long long t2 = clock64();
  if (threadIdx.x == 0) {
    cyc[blockIdx.x] = (t1 - t0) + 0 * reps;
    cyc[148 + blockIdx.x] = t2 - t1;
    out[blockIdx.x] = buf[1];
  }
}

int main() {
  int sizes[] = {216, 432, 729, 1152, 2304};
  long long* cyc;
  double2* out;
  CK(cudaMalloc(&cyc, 8 * 296));
  CK(cudaMalloc(&out, 16 * 148));
  for (int n : sizes) {
    for (int wide = 0; wide < 2; ++wide) {
      FftPlan pl{};
      if (!fft_factor(n, &pl, wide) || pl.nthr > 512) continue;
      std::vector<double2> tw;
      fft_stage_twiddles(pl, tw, [](double c, double s) { return make_double2(c, s); });
      pl.ntw = (int)tw.size();
      tw.push_back(make_double2(1, 0));
      double2* dtw;
      CK(cudaMalloc(&dtw, 16 * tw.size()));
      CK(cudaMemcpy(dtw, tw.data(), 16 * tw.size(), cudaMemcpyHostToDevice));
      pl.tw = dtw;
      const size_t smem = 16 * ((size_t)n + pl.ntw + 1);
      CK(cudaFuncSetAttribute((const void*)lat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
      for (int ctas : {1, 148}) {
        lat_kernel<<<ctas, pl.nthr, smem>>>(pl, 50, cyc, out);
        CK(cudaDeviceSynchronize());
        std::vector<long long> h(ctas);
        CK(cudaMemcpy(h.data(), cyc, 8 * ctas, cudaMemcpyDeviceToHost));
        long long mx = 0;
        for (auto v : h) mx = v > mx ? v : mx;
        long long w = 0;
        CK(cudaMemcpy(&w, cyc + 148, 8, cudaMemcpyDeviceToHost));
        printf("n=%5d %s nthr=%3d stages=%d ctas=%3d  cycles/fft first %lld (%.2f us at 1.965 GHz), second %lld\n", n,
               wide ? "wide  " : "normal", pl.nthr, pl.nstages, ctas, mx, mx / 1965.0, w);
      }
      CK(cudaFree(dtw));
    }
  }
  return 0;
}
