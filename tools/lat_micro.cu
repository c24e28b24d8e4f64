// Dependent-latency microbenchmark (cycles per op, one warp): DFMA, DADD, DMUL chains,
// shared-memory load chain, __syncthreads, integer modulo.  Explains the FFT stage cost.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/lat_micro tools/lat_micro.cu
#include <cstdio>

__global__ void lat(double* out, long long* cyc, int iters, int modv) {
  __shared__ int chase[1024];
  __shared__ double2 sd[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) { chase[i] = (i * 37 + 11) & 1023; sd[i] = make_double2(i, 1); }
  __syncthreads();
  double a = out[0], b = out[1], c = out[2];
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) a = a + b;
  long long t2 = clock64();
  int p = threadIdx.x;
  for (int i = 0; i < iters; ++i) p = chase[p];
  long long t3 = clock64();
  for (int i = 0; i < iters; ++i) __syncthreads();
  long long t4 = clock64();
  int q = threadIdx.x + 12345;
  for (int i = 0; i < iters; ++i) q = q % (modv + (q & 1)) + 100000;
  long long t5 = clock64();
  double2 v = sd[threadIdx.x];
  for (int i = 0; i < iters; ++i) { v = sd[((int)v.y + i) & 1023]; }
  long long t6 = clock64();
  double s = sin((double)p);
  for (int i = 0; i < iters; ++i) a = a * b;
  long long t7 = clock64();
  if (threadIdx.x == 0) {
    out[3] = a + p + q + v.x + s;
    cyc[0] = (t1 - t0) / iters; cyc[1] = (t2 - t1) / iters; cyc[2] = (t3 - t2) / iters;
    cyc[3] = (t4 - t3) / iters; cyc[4] = (t5 - t4) / iters; cyc[5] = (t6 - t5) / iters; cyc[6] = (t7 - t6) / iters;
  }
}

int main() {
  double* out; long long* cyc;
  cudaMalloc(&out, 64); cudaMalloc(&cyc, 64);
  double h[3] = {1.0000001, 0.9999999, 1e-9};
  cudaMemcpy(out, h, 24, cudaMemcpyHostToDevice);
  for (int threads : {32, 256}) {
    lat<<<1, threads>>>(out, cyc, 4096, 7);
    cudaDeviceSynchronize();
    long long c[7];
    cudaMemcpy(c, cyc, 56, cudaMemcpyDeviceToHost);
    printf("threads %3d: DFMA %lld  DADD %lld  smem-int-chase %lld  syncthreads %lld  int%% %lld  smem-double2-chase %lld  DMUL %lld  (cycles/op)\n",
           threads, c[0], c[1], c[2], c[3], c[4], c[5], c[6]);
  }
  return 0;
}
