// Microbenchmarks used to pin roofline denominators on the B200 box:
//   FP64 DFMA / DADD issue rate, Philox4x64-10 word rate, normcdfinv accuracy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); exit(1);} } while (0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__device__ __forceinline__ void mulhilo64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
  lo = a * b;
  hi = __umul64hi(a, b);
}

__global__ void philox_kernel(unsigned long long* out, int blocks_per_thread, uint64_t k0, uint64_t k1) {
  uint64_t acc = 0;
  uint64_t base = (uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * blocks_per_thread;
  for (int b = 0; b < blocks_per_thread; ++b) {
    uint64_t c0 = base + b + 1, c1 = 0, c2 = 0, c3 = 0;
    uint64_t kk0 = k0, kk1 = k1;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
      if (r) { kk0 += 0x9E3779B97F4A7C15ULL; kk1 += 0xBB67AE8584CAA73BULL; }
      uint64_t h0, l0, h1, l1;
      mulhilo64(0xD2E7470EE14C6C93ULL, c0, h0, l0);
      mulhilo64(0xCA5A826395121157ULL, c2, h1, l1);
      c0 = h1 ^ c1 ^ kk0; c1 = l1; c2 = h0 ^ c3 ^ kk1; c3 = l0;
    }
    acc ^= c0 ^ c1 ^ c2 ^ c3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void normal_kernel(const double* u, double* z, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) z[i] = normcdfinv(u[i]);
}

__global__ void normal_rate_kernel(double* out, int per_thread) {
  double acc = 0;
  uint64_t base = (uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) * per_thread;
  for (int i = 0; i < per_thread; ++i) {
    uint64_t k = (base + i) * 0x9E3779B97F4A7C15ULL >> 11;
    double uu = ((double)k + 0.5) * 0x1.0p-53;
    acc += normcdfinv(uu);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

__global__ void copy_kernel(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t s = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += s) b[i] = a[i];
}

int main(int argc, char** argv) {
  cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, 0));
  int sms = prop.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d", prop.name, sms);
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  float ms;
  // FP64 FMA
  {
    double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 256));
    int iters = 4000;
    dfma_kernel<<<sms * 8, 256>>>(out, 10, 0.999, 1e-3);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    dfma_kernel<<<sms * 8, 256>>>(out, iters, 0.999, 1e-3);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double fmas = (double)sms * 8 * 256 * iters * 64;
    printf(", \"dfma_tflops\": %.3f", 2.0 * fmas / (ms * 1e-3) / 1e12);
    CK(cudaFree(out));
  }
  // Philox
  {
    unsigned long long* out; int nthr = sms * 16 * 256;
    CK(cudaMalloc(&out, sizeof(unsigned long long) * nthr));
    int bpt = 256;
    philox_kernel<<<sms * 16, 256>>>(out, 4, 5, 1);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    philox_kernel<<<sms * 16, 256>>>(out, bpt, 5, 1);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    double words = (double)nthr * bpt * 4;
    printf(", \"philox_gwords_per_s\": %.2f", words / (ms * 1e-3) / 1e9);
    CK(cudaFree(out));
  }
  // normcdfinv rate
  {
    double* out; int nthr = sms * 16 * 256; int per = 256;
    CK(cudaMalloc(&out, sizeof(double) * nthr));
    normal_rate_kernel<<<sms * 16, 256>>>(out, 4);
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(e0));
    normal_rate_kernel<<<sms * 16, 256>>>(out, per);
    CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
    CK(cudaEventElapsedTime(&ms, e0, e1));
    printf(", \"normcdfinv_gvals_per_s\": %.2f", (double)nthr * per / (ms * 1e-3) / 1e9);
    CK(cudaFree(out));
  }
  // copy bandwidth
  {
    size_t n = (size_t)1 << 27;  // 2 GiB per buffer of double2
    double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    CK(cudaMemset(a, 0, n * 16));
    copy_kernel<<<sms * 8, 512>>>(a, b, n);
    CK(cudaDeviceSynchronize());
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      CK(cudaEventRecord(e0));
      copy_kernel<<<sms * 8, 512>>>(a, b, n);
      CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1));
      CK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    printf(", \"copy_gbs\": %.1f", 2.0 * n * 16 / (best * 1e-3) / 1e9);
    CK(cudaFree(a)); CK(cudaFree(b));
  }
  printf("}\n");
  // normcdfinv accuracy: read u from file, write z
  if (argc > 2) {
    FILE* f = fopen(argv[1], "rb"); fseek(f, 0, SEEK_END); long sz = ftell(f); fseek(f, 0, SEEK_SET);
    int n = sz / 8; std::vector<double> u(n), z(n);
    fread(u.data(), 8, n, f); fclose(f);
    double *du, *dz; CK(cudaMalloc(&du, sz)); CK(cudaMalloc(&dz, sz));
    CK(cudaMemcpy(du, u.data(), sz, cudaMemcpyHostToDevice));
    normal_kernel<<<(n + 255) / 256, 256>>>(du, dz, n);
    CK(cudaMemcpy(z.data(), dz, sz, cudaMemcpyDeviceToHost));
    f = fopen(argv[2], "wb"); fwrite(z.data(), 8, n, f); fclose(f);
  }
  return 0;
}
