// rapidkrig B200: exact universal Kriging on the GPU -- fit, batched GLS refit, the inverse
// Cholesky factor, exact prediction and its standard error at arbitrary targets.
//
// Reference mapping (/root/reference/pkg/src/rapidkrig/exact.py):
//   fit / _cholesky_with_ridge 25-37, 71-105 -> rk_fit_create (dense Matern kernel, cuSOLVER potrf)
//   refit_coefficients / _gls  59-68, 108-113 -> gls_batch (two FP64 tensor-core GEMMs with U^-1)
//   predict_exact 132-147                     -> predict_exact_kernel (fixed-order target sums)
//   kriging_se_exact 150-175                  -> cross_cov_kernel + GEMMs + se_finish_kernel
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include <cublas_v2.h>
#include <cusolverDn.h>

#include "rk_internal.cuh"

namespace rk {

// ------------------------------------------------------------------- fit
#define RK_CUBLAS_TRY(expr)                                                                  \
  do {                                                                                       \
    cublasStatus_t _b = (expr);                                                              \
    if (_b != CUBLAS_STATUS_SUCCESS)                                                         \
      return Status::err(RK_CUDA, std::string("cuBLAS status ") + std::to_string((int)_b) + \
                                      " at " #expr);                                        \
  } while (0)

// cuBLAS handle for `st`: one per stream, so ensemble chunks running concurrently on
// different streams never share a handle's workspace
static Status blas_for(rk_fit* f, cudaStream_t st, cublasHandle_t* out) {
  std::lock_guard<std::mutex> lk(f->blas_mu);
  auto it = f->blas_by_stream.find(st);
  cublasHandle_t h;
  if (it != f->blas_by_stream.end()) {
    h = (cublasHandle_t)it->second;
  } else {
    RK_CUBLAS_TRY(cublasCreate(&h));
    f->blas_by_stream[st] = h;
  }
  RK_CUBLAS_TRY(cublasSetStream(h, st));
  *out = h;
  return Status::ok();
}

// dense M = K + tau2 I (+ ridge) column-major, cdist distances (covariance.py:100-116)
__global__ void dense_cov_kernel(MaternDev P, const double* __restrict__ obs, int64_t n, double diag_add,
                                 double* __restrict__ Mm, int* bad) {
  const int64_t tot = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e % n;
    if (i > j) continue;   // only the upper triangle is read by potrf(UPPER)
    const double dx = obs[2 * i] - obs[2 * j], dy = obs[2 * i + 1] - obs[2 * j + 1];
    const double d = sqrt(dx * dx + dy * dy);
    double v = matern_cov(P, d, bad);
    if (i == j) v += diag_add;
    Mm[e] = v;
  }
}

__global__ void add_diag_kernel(double* Mm, int64_t n, double v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    Mm[i * n + i] += v;
}

__global__ void zero_lower_kernel(double* U, int64_t n) {
  const int64_t tot = n * n;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e % n;
    if (i > j) U[e] = 0.0;
  }
}

// r[:, b] = z[:, b] - X beta[:, b]   (exact.py:65)
__global__ void resid_kernel(const double* __restrict__ z, const double* __restrict__ X, int64_t n,
                             int p, const double* __restrict__ beta, int batch, double* __restrict__ r) {
  const int64_t tot = n * batch;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / n, i = e % n;
    double xb = 0.0;
    for (int q = 0; q < p; ++q) xb = fma(X[(int64_t)q * n + i], beta[b * p + q], xb);
    r[e] = z[e] - xb;
  }
}

struct GramLU {
  double lu[64];
  int piv[8];
  int p;
};

// beta[:, b] = gram^-1 rhs[:, b] from the host LU with partial pivoting (np.linalg.solve)
__global__ void gram_solve_kernel(GramLU g, double* rhs, int batch) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  double x[8];
  const int p = g.p;
  for (int i = 0; i < p; ++i) x[i] = rhs[(int64_t)b * p + i];
  for (int i = 0; i < p; ++i) {
    const int pi = g.piv[i];
    if (pi != i) { const double t = x[i]; x[i] = x[pi]; x[pi] = t; }
  }
  for (int i = 0; i < p; ++i)
    for (int k = 0; k < i; ++k) x[i] -= g.lu[i * p + k] * x[k];
  for (int i = p - 1; i >= 0; --i) {
    for (int k = i + 1; k < p; ++k) x[i] -= g.lu[i * p + k] * x[k];
    x[i] /= g.lu[i * p + i];
  }
  for (int i = 0; i < p; ++i) rhs[(int64_t)b * p + i] = x[i];
}

static bool lu_factor(std::vector<double>& a, int p, std::vector<int>& piv) {
  piv.assign(p, 0);
  for (int k = 0; k < p; ++k) {
    int m = k;
    for (int i = k + 1; i < p; ++i)
      if (std::fabs(a[(size_t)i * p + k]) > std::fabs(a[(size_t)m * p + k])) m = i;
    piv[k] = m;
    if (a[(size_t)m * p + k] == 0.0) return false;
    if (m != k)
      for (int j = 0; j < p; ++j) std::swap(a[(size_t)k * p + j], a[(size_t)m * p + j]);
    for (int i = k + 1; i < p; ++i) {
      a[(size_t)i * p + k] /= a[(size_t)k * p + k];
      for (int j = k + 1; j < p; ++j) a[(size_t)i * p + j] -= a[(size_t)i * p + k] * a[(size_t)k * p + j];
    }
  }
  return true;
}

static GramLU gram_args(const rk_fit* f) {
  GramLU g{};
  g.p = f->p;
  for (int i = 0; i < f->p * f->p; ++i) g.lu[i] = f->gram_lu[i];
  for (int i = 0; i < f->p; ++i) g.piv[i] = f->gram_piv[i];
  return g;
}

// GLS by triangular solves (exact.py:59-68) for `batch` right-hand sides Z (n x batch,
// column-major) -> beta (p x batch), C (n x batch).  Used once per fit.
static Status gls_trsm(const rk_fit* f, const double* Z, int64_t batch, double* beta, double* C,
                        cudaStream_t st) {
  cublasHandle_t h;
  RK_TRY(blas_for(const_cast<rk_fit*>(f), st, &h));
  const int n = (int)f->n, p = f->p, nb = (int)batch;
  const double one = 1.0, zero = 0.0;
  double* A = nullptr;
  RK_TRY(scratch_alloc((void**)&A, sizeof(double) * (size_t)n * nb, st));
  RK_CUDA_TRY(cudaMemcpyAsync(A, Z, sizeof(double) * (size_t)n * nb, cudaMemcpyDeviceToDevice, st));
  // a = L^-1 z  (L = U^T)
  RK_CUBLAS_TRY(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                            CUBLAS_DIAG_NON_UNIT, n, nb, &one, f->U, n, A, n));
  // rhs = b' a
  RK_CUBLAS_TRY(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, p, nb, n, &one, f->B, n, A, n, &zero, beta, p));
  gram_solve_kernel<<<(nb + 127) / 128, 128, 0, st>>>(gram_args(f), beta, nb);
  count_launch();
  // resid = z - X beta ; half = L^-1 resid ; c = L^-T half
  resid_kernel<<<(int)std::min<int64_t>(ceil_div((int64_t)n * nb, 256), 148 * 32), 256, 0, st>>>(
      Z, f->X, n, p, beta, nb, C);
  count_launch();
  RK_LAUNCH_CHECK();
  RK_CUBLAS_TRY(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                            CUBLAS_DIAG_NON_UNIT, n, nb, &one, f->U, n, C, n));
  RK_CUBLAS_TRY(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N,
                            CUBLAS_DIAG_NON_UNIT, n, nb, &one, f->U, n, C, n));
  scratch_free(A, st);
  return Status::ok();
}


// Batched refit (exact.py:108-113) with the precomputed inverse factor, on our own FP64
// tensor-core kernels (rk_refit.cu) -- no cuBLAS on the ensemble path:
//   A = L^-1 Z ; beta = (B'B)^-1 B'A ; H = A - B beta (= L^-1 (Z - X beta)) ; C = L^-T H
Status gls_batch(const rk_fit* f, const double* Z, int64_t batch, double* beta, double* C,
                 cudaStream_t st) {
  const int64_t n = f->n;
  const int p = f->p;
  if (!f->Uinv) return Status::err(RK_INTERNAL, "refit without the inverse factor (call ensure_uinv first)");
  double *A = nullptr, *H = nullptr;
  RK_TRY(scratch_alloc((void**)&A, sizeof(double) * (size_t)n * batch, st));
  RK_TRY(scratch_alloc((void**)&H, sizeof(double) * (size_t)n * batch, st));
  RK_TRY(trmm_linv(f, false, Z, n, batch, A, n, st));
  RK_TRY(bta(f, A, n, batch, beta, st));
  for (int64_t b0 = 0; b0 < batch; b0 += 1 << 20) {
    const int nb = (int)std::min<int64_t>(batch - b0, 1 << 20);
    gram_solve_kernel<<<(nb + 127) / 128, 128, 0, st>>>(gram_args(f), beta + b0 * p, nb);
    count_launch();
  }
  resid_kernel<<<(int)std::min<int64_t>(ceil_div(n * batch, 256), 148 * 32), 256, 0, st>>>(
      A, f->B, n, p, beta, (int)batch, H);
  count_launch();
  RK_LAUNCH_CHECK();
  RK_TRY(trmm_linv(f, true, H, n, batch, C, n, st));
  scratch_free(A, st);
  scratch_free(H, st);
  return Status::ok();
}

void free_fit(rk_fit* f) {
  if (!f) return;
  int cur = 0;
  const bool swap = cudaGetDevice(&cur) == cudaSuccess && cur != f->device && cudaSetDevice(f->device) == cudaSuccess;
  cudaFree(f->Uinv);
  cudaFree(f->obs);
  cudaFree(f->U);
  cudaFree(f->X);
  cudaFree(f->B);
  cudaFree(f->beta);
  cudaFree(f->c);
  if (f->cublas) cublasDestroy((cublasHandle_t)f->cublas);
  for (auto& kv : f->blas_by_stream) cublasDestroy((cublasHandle_t)kv.second);
  delete f;
  if (swap) cudaSetDevice(cur);
}

// common tail: X upload, B = L^-1 X, gram LU
static Status fit_prepare_x(rk_fit* f, const double* X_host) {
  const int64_t n = f->n;
  const int p = f->p;
  std::vector<double> Xc((size_t)n * p);
  for (int64_t i = 0; i < n; ++i)
    for (int q = 0; q < p; ++q) Xc[(size_t)q * n + i] = X_host ? X_host[(size_t)i * p + q] : 1.0;
  RK_CUDA_TRY(cudaMalloc(&f->X, sizeof(double) * n * p));
  RK_CUDA_TRY(cudaMalloc(&f->B, sizeof(double) * n * p));
  RK_CUDA_TRY(cudaMemcpy(f->X, Xc.data(), sizeof(double) * n * p, cudaMemcpyHostToDevice));
  RK_CUDA_TRY(cudaMemcpy(f->B, Xc.data(), sizeof(double) * n * p, cudaMemcpyHostToDevice));
  cublasHandle_t h = (cublasHandle_t)f->cublas;
  RK_CUBLAS_TRY(cublasSetStream(h, 0));
  const double one = 1.0, zero = 0.0;
  RK_CUBLAS_TRY(cublasDtrsm(h, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_T,
                            CUBLAS_DIAG_NON_UNIT, (int)n, p, &one, f->U, (int)n, f->B, (int)n));
  double* G = nullptr;
  RK_CUDA_TRY(cudaMalloc(&G, sizeof(double) * p * p));
  RK_CUBLAS_TRY(cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, p, p, (int)n, &one, f->B, (int)n, f->B,
                            (int)n, &zero, G, p));
  std::vector<double> g((size_t)p * p);
  RK_CUDA_TRY(cudaMemcpy(g.data(), G, sizeof(double) * p * p, cudaMemcpyDeviceToHost));
  cudaFree(G);
  // column-major p x p -> row-major (symmetric anyway)
  std::vector<double> gr((size_t)p * p);
  for (int i = 0; i < p; ++i)
    for (int j = 0; j < p; ++j) gr[(size_t)i * p + j] = g[(size_t)j * p + i];
  f->gram_lu = gr;
  if (!lu_factor(f->gram_lu, p, f->gram_piv))
    return Status::err(RK_NUMERIC, "singular GLS Gram matrix X' M^-1 X");
  return Status::ok();
}

// U^-1 (= L^-T) by blocked triangular inversion (cuSOLVER trtri), once per fit
// In-place inverse of the upper-triangular column-major block U (n x n, leading dim ld).
// cuSOLVER's trtri rejects very large n (INVALID_VALUE at n = 50000), so big blocks recurse:
// inv([A B; 0 D]) = [inv(A), -inv(A) B inv(D); 0, inv(D)] with two TRMMs through scratch T.
static int64_t trtri_block() {   // RK_TRTRI_BLOCK overrides (tests exercise the recursion)
  static const int64_t b = getenv("RK_TRTRI_BLOCK") ? atoll(getenv("RK_TRTRI_BLOCK")) : 16384;
  return std::max<int64_t>(b, 256);
}

static Status inv_upper(cusolverDnHandle_t sh, cublasHandle_t bh, double* U, int64_t n, int64_t ld, double* T,
                        cudaStream_t st) {
  if (n <= trtri_block()) {
    size_t dbytes = 0, hbytes = 0;
    cusolverStatus_t cs = cusolverDnXtrtri_bufferSize(sh, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n,
                                                      CUDA_R_64F, U, ld, &dbytes, &hbytes);
    if (cs != CUSOLVER_STATUS_SUCCESS)
      return Status::err(RK_CUDA, "cusolverDnXtrtri_bufferSize failed (status " + std::to_string((int)cs) + ")");
    void* dwork = nullptr;
    std::vector<char> hwork(hbytes + 1);
    int* info = nullptr;
    RK_CUDA_TRY(cudaMalloc(&dwork, dbytes + 16));
    RK_CUDA_TRY(cudaMalloc(&info, sizeof(int)));
    cs = cusolverDnXtrtri(sh, CUBLAS_FILL_MODE_UPPER, CUBLAS_DIAG_NON_UNIT, n, CUDA_R_64F, U, ld, dwork, dbytes,
                          hwork.data(), hbytes, info);
    int hinfo = 0;
    RK_CUDA_TRY(cudaMemcpyAsync(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost, st));
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    cudaFree(dwork);
    cudaFree(info);
    if (cs != CUSOLVER_STATUS_SUCCESS || hinfo != 0) {
      char b[160];
      snprintf(b, sizeof b, "triangular inverse of the Cholesky factor failed (cusolver status %d, info %d, n %lld)",
               (int)cs, hinfo, (long long)n);
      return Status::err(RK_NUMERIC, b);
    }
    return Status::ok();
  }
  const int64_t n1 = (n / 2 + 255) / 256 * 256, n2 = n - n1;
  double* A = U;
  double* B = U + n1 * ld;
  double* D = B + n1;
  RK_TRY(inv_upper(sh, bh, A, n1, ld, T, st));
  RK_TRY(inv_upper(sh, bh, D, n2, ld, T, st));
  const double one = 1.0, mone = -1.0;
  RK_CUBLAS_TRY(cublasSetStream(bh, st));
  RK_CUBLAS_TRY(cublasDtrmm_64(bh, CUBLAS_SIDE_LEFT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n1,
                               n2, &one, A, ld, B, ld, T, n1));                 // T = inv(A) B
  RK_CUBLAS_TRY(cublasDtrmm_64(bh, CUBLAS_SIDE_RIGHT, CUBLAS_FILL_MODE_UPPER, CUBLAS_OP_N, CUBLAS_DIAG_NON_UNIT, n1,
                               n2, &mone, D, ld, T, n1, B, ld));                // B = -T inv(D)
  return Status::ok();
}

Status ensure_uinv(rk_fit* f, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(f->uinv_mu);   // concurrent first refits build it once
  if (f->Uinv) return Status::ok();
  const int64_t n = f->n;
  double* Ui = nullptr;
  RK_CUDA_TRY(cudaMalloc(&Ui, sizeof(double) * (size_t)n * n));
  RK_CUDA_TRY(cudaMemcpyAsync(Ui, f->U, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, st));
  cusolverDnHandle_t sh;
  if (cusolverDnCreate(&sh) != CUSOLVER_STATUS_SUCCESS) {
    cudaFree(Ui);
    return Status::err(RK_CUDA, "cusolverDnCreate failed");
  }
  cusolverDnSetStream(sh, st);
  double* T = nullptr;
  Status r = Status::ok();
  if (n > trtri_block()) {
    const int64_t n1 = (n / 2 + 255) / 256 * 256;
    r = scratch_alloc((void**)&T, sizeof(double) * (size_t)n1 * (n - n1), st);
  }
  if (r.good()) r = inv_upper(sh, (cublasHandle_t)f->cublas, Ui, n, n, T, st);
  if (T) scratch_free(T, st);
  if (r.good()) {
    const cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) r = Status::err(RK_CUDA, std::string("inverse factor: ") + cudaGetErrorString(e));
  }
  cusolverDnDestroy(sh);
  if (!r.good()) {
    cudaFree(Ui);
    return r;
  }
  f->Uinv = Ui;
  return Status::ok();
}

}  // namespace rk

using namespace rk;

static int finish_exact(const Status& s) {
  if (!s.good()) rk::set_error(s.code, s.msg);
  return s.code;
}

extern "C" {

rk_status rk_fit_create(const rk_model* model, const double* obs_host, int64_t n, const double* z_host,
                        const double* X_host, int32_t p, rk_fit** out, int32_t* ridge_applied) {
  auto run = [&]() -> Status {
    if (n < 1 || p < 1 || p > 8 || n < p) return Status::err(RK_DOMAIN, "need n >= p >= 1 (p <= 8)");
    rk_fit* f = new rk_fit();
    std::unique_ptr<rk_fit, void (*)(rk_fit*)> guard(f, free_fit);
    RK_CUDA_TRY(cudaGetDevice(&f->device));
    f->model = *model;
    f->n = n;
    f->p = p;
    cublasHandle_t h;
    RK_CUBLAS_TRY(cublasCreate(&h));
    f->cublas = h;
    const MaternDev P = make_matern_dev(*model);
    double* dobs = nullptr;
    int* bad = nullptr;
    RK_CUDA_TRY(cudaMalloc(&dobs, sizeof(double) * 2 * n));
    f->obs = dobs;   // owned by the fit: kept for predict_exact / kriging_se_exact
    RK_CUDA_TRY(cudaMalloc(&bad, sizeof(int)));
    RK_CUDA_TRY(cudaMemset(bad, 0, sizeof(int)));
    RK_CUDA_TRY(cudaMemcpy(dobs, obs_host, sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
    RK_CUDA_TRY(cudaMalloc(&f->U, sizeof(double) * (size_t)n * n));
    cusolverDnHandle_t sh;
    if (cusolverDnCreate(&sh) != CUSOLVER_STATUS_SUCCESS) return Status::err(RK_CUDA, "cusolverDnCreate failed");
    int lwork = 0;
    cusolverDnDpotrf_bufferSize(sh, CUBLAS_FILL_MODE_UPPER, (int)n, f->U, (int)n, &lwork);
    double* work = nullptr;
    int* info = nullptr;
    RK_CUDA_TRY(cudaMalloc(&work, sizeof(double) * std::max(lwork, 1)));
    RK_CUDA_TRY(cudaMalloc(&info, sizeof(int)));
    // trace(M) = sum(sigma2 * phi(0) + tau2) (exact.py:102)
    const double diag = model->sigma2 + model->tau2;
    double trace = 0.0;
    for (int64_t i = 0; i < n; ++i) trace += diag;
    const double ridge = 1.0e-10 * trace / (double)n;
    int hinfo = 0;
    *ridge_applied = 0;
    for (int attempt = 0; attempt < 2; ++attempt) {
      dense_cov_kernel<<<(int)std::min<int64_t>(ceil_div(n * n, 256), 148 * 64), 256>>>(
          P, dobs, n, model->tau2, f->U, bad);
      count_launch();
      RK_LAUNCH_CHECK();
      if (attempt == 1) {  // (K + tau2 I) + ridge I  (exact.py:33-35)
        add_diag_kernel<<<(int)std::min<int64_t>(ceil_div(n, 256), 4096), 256>>>(f->U, n, ridge);
        count_launch();
      }
      if (cusolverDnDpotrf(sh, CUBLAS_FILL_MODE_UPPER, (int)n, f->U, (int)n, work, lwork, info) !=
          CUSOLVER_STATUS_SUCCESS)
        return Status::err(RK_CUDA, "cusolverDnDpotrf failed");
      RK_CUDA_TRY(cudaMemcpy(&hinfo, info, sizeof(int), cudaMemcpyDeviceToHost));
      if (hinfo == 0) break;
      if (attempt == 0) *ridge_applied = 1;
    }
    cusolverDnDestroy(sh);
    cudaFree(work);
    cudaFree(info);
    int hb = 0;
    RK_CUDA_TRY(cudaMemcpy(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost));
    cudaFree(bad);
    f->mat = P;
    if (hb) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");
    if (hinfo != 0)
      return Status::err(RK_NUMERIC, "Cholesky of the observation covariance M failed even with ridge");
    zero_lower_kernel<<<(int)std::min<int64_t>(ceil_div(n * n, 256), 148 * 64), 256>>>(f->U, n);
    count_launch();
    RK_TRY(fit_prepare_x(f, X_host));
    RK_CUDA_TRY(cudaMalloc(&f->beta, sizeof(double) * p));
    RK_CUDA_TRY(cudaMalloc(&f->c, sizeof(double) * n));
    double* z = nullptr;
    RK_CUDA_TRY(cudaMalloc(&z, sizeof(double) * n));
    RK_CUDA_TRY(cudaMemcpy(z, z_host, sizeof(double) * n, cudaMemcpyHostToDevice));
    RK_TRY(gls_trsm(f, z, 1, f->beta, f->c, 0));
    RK_CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(z);
    *out = guard.release();
    return Status::ok();
  };
  int32_t r = 0;
  if (!ridge_applied) ridge_applied = &r;
  return (rk_status)finish_exact(run());
}

rk_status rk_fit_import(const rk_model* model, const double* obs_host, int64_t n, const double* X_host,
                        int32_t p, const double* chol_host, const double* beta_host,
                        const double* c_host, rk_fit** out) {
  auto run = [&]() -> Status {
    if (n < 1 || p < 1 || p > 8) return Status::err(RK_DOMAIN, "need n >= p >= 1 (p <= 8)");
    rk_fit* f = new rk_fit();
    std::unique_ptr<rk_fit, void (*)(rk_fit*)> guard(f, free_fit);
    RK_CUDA_TRY(cudaGetDevice(&f->device));
    f->model = *model;
    f->n = n;
    f->p = p;
    cublasHandle_t h;
    RK_CUBLAS_TRY(cublasCreate(&h));
    f->cublas = h;
    // row-major lower L == column-major upper U = L^T
    RK_CUDA_TRY(cudaMalloc(&f->U, sizeof(double) * (size_t)n * n));
    RK_CUDA_TRY(cudaMemcpy(f->U, chol_host, sizeof(double) * (size_t)n * n, cudaMemcpyHostToDevice));
    RK_TRY(fit_prepare_x(f, X_host));
    RK_CUDA_TRY(cudaMalloc(&f->beta, sizeof(double) * p));
    RK_CUDA_TRY(cudaMalloc(&f->c, sizeof(double) * n));
    RK_CUDA_TRY(cudaMemcpy(f->beta, beta_host, sizeof(double) * p, cudaMemcpyHostToDevice));
    RK_CUDA_TRY(cudaMemcpy(f->c, c_host, sizeof(double) * n, cudaMemcpyHostToDevice));
    RK_CUDA_TRY(cudaMalloc(&f->obs, sizeof(double) * 2 * n));
    RK_CUDA_TRY(cudaMemcpy(f->obs, obs_host, sizeof(double) * 2 * n, cudaMemcpyHostToDevice));
    f->mat = make_matern_dev(*model);
    *out = guard.release();
    return Status::ok();
  };
  return (rk_status)finish_exact(run());
}

rk_status rk_fit_destroy(rk_fit* f) {
  free_fit(f);
  return RK_OK;
}

rk_status rk_fit_info(const rk_fit* f, int64_t* n, int32_t* p) {
  if (n) *n = f->n;
  if (p) *p = f->p;
  return RK_OK;
}

rk_status rk_fit_copy_out(const rk_fit* f, double* beta_host, double* c_host, double* chol_host) {
  auto run = [&]() -> Status {
    if (beta_host) RK_CUDA_TRY(cudaMemcpy(beta_host, f->beta, sizeof(double) * f->p, cudaMemcpyDeviceToHost));
    if (c_host) RK_CUDA_TRY(cudaMemcpy(c_host, f->c, sizeof(double) * f->n, cudaMemcpyDeviceToHost));
    if (chol_host)
      RK_CUDA_TRY(cudaMemcpy(chol_host, f->U, sizeof(double) * (size_t)f->n * f->n, cudaMemcpyDeviceToHost));
    return Status::ok();
  };
  return (rk_status)finish_exact(run());
}

rk_status rk_refit_dev(const rk_fit* f, const double* z_dev, int64_t batch, double* beta_dev,
                       double* c_dev, void* stream) {
  auto run = [&]() -> Status {
    RK_TRY(ensure_uinv(const_cast<rk_fit*>(f), (cudaStream_t)stream));
    return gls_batch(f, z_dev, batch, beta_dev, c_dev, (cudaStream_t)stream);
  };
  return (rk_status)finish_exact(run());
}

rk_status rk_fit_prepare_refit(rk_fit* f, void* stream) {
  return (rk_status)finish_exact(ensure_uinv(f, (cudaStream_t)stream));
}

}  // extern "C"

// ===================================================== exact prediction at targets
// predict_exact (exact.py:132-147): X_t beta + k_t c, k_t the cross covariance of the targets
// with the observations, never formed: every thread owns one target and runs over the
// observations in index order (staged through shared memory), so the sum order is fixed.
// kriging_se_exact (exact.py:150-175): the k_t block IS formed (n x chunk, column-major),
// u = L^-1 k_t as one FP64 tensor-core GEMM with the fit's U^-1, var = sigma2 - |u|^2 +
// h'(B'B)^-1 h with h = x_t - u'B, clamp at -1e-10, sqrt.
namespace rk {

constexpr int kExactThreads = 256;

struct ExactArgs {
  MaternDev mat;
  const double* obs;       // (n, 2)
  const double* c;         // (n)
  int64_t n;
  const double* tgt;       // (nt, 2)
  int64_t nt;
  const double* xt;        // (nt, p) row-major, or null: intercept-only fit, x00 * beta[0]
  double x00;
  const double* beta;      // (p)
  int p;
  double* out;             // (nt)
  int* bad;
};

__global__ void __launch_bounds__(kExactThreads) predict_exact_kernel(const ExactArgs a) {
  __shared__ double so[3][kExactThreads];
  const int64_t t = blockIdx.x * (int64_t)kExactThreads + threadIdx.x;
  const bool valid = t < a.nt;
  const double tx = valid ? a.tgt[2 * t] : 0.0, ty = valid ? a.tgt[2 * t + 1] : 0.0;
  double acc = 0.0;
  for (int64_t i0 = 0; i0 < a.n; i0 += kExactThreads) {
    const int m = a.n - i0 < kExactThreads ? (int)(a.n - i0) : kExactThreads;
    __syncthreads();
    if (threadIdx.x < m) {
      so[0][threadIdx.x] = a.obs[2 * (i0 + threadIdx.x)];
      so[1][threadIdx.x] = a.obs[2 * (i0 + threadIdx.x) + 1];
      so[2][threadIdx.x] = a.c[i0 + threadIdx.x];
    }
    __syncthreads();
    if (valid)
      for (int k = 0; k < m; ++k) {
        const double dx = tx - so[0][k], dy = ty - so[1][k];
        acc = fma(matern_cov(a.mat, sqrt(dx * dx + dy * dy), a.bad), so[2][k], acc);
      }
  }
  if (!valid) return;
  double fx = 0.0;
  if (a.xt)
    for (int q = 0; q < a.p; ++q) fx = fma(a.xt[t * a.p + q], a.beta[q], fx);
  else
    fx = a.x00 * a.beta[0];
  a.out[t] = acc + fx;
}

// K (n x tc, column-major): K[i + j n] = cov(|obs_i - tgt_j|)
__global__ void cross_cov_kernel(MaternDev P, const double* __restrict__ obs, int64_t n,
                                 const double* __restrict__ tgt, int64_t tc, double* __restrict__ K, int* bad) {
  const int64_t tot = n * tc;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < tot;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = e / n, i = e - j * n;
    const double dx = tgt[2 * j] - obs[2 * i], dy = tgt[2 * j + 1] - obs[2 * i + 1];
    K[e] = matern_cov(P, sqrt(dx * dx + dy * dy), bad);
  }
}

// one warp per target column: var = sigma2 - sum_i u_i^2 (fixed lane-strided order + tree)
__global__ void colsq_kernel(const double* __restrict__ u, int64_t n, int64_t tc, double sigma2, double* var) {
  const int64_t j = blockIdx.x * (int64_t)(blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (j >= tc) return;
  const double* col = u + j * n;
  double s = 0.0;
  for (int64_t i = lane; i < n; i += 32) s = fma(col[i], col[i], s);
#pragma unroll
  for (int d = 16; d; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
  if (lane == 0) var[j] = sigma2 - s;
}

// h = x_t - (B'u)' (p x tc, column-major) in place over BtU; then hg = gram^-1 h; var += h.hg;
// clamp / sqrt into out; the most negative variance is tracked for the error message
__global__ void se_finish_kernel(GramLU g, double* __restrict__ BtU, const double* __restrict__ xt, double x00,
                                 int64_t tc, const double* __restrict__ var, double* __restrict__ out,
                                 unsigned long long* minvar_bits) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= tc) return;
  const int p = g.p;
  double h[8], x[8];
  for (int q = 0; q < p; ++q) {
    const double xq = xt ? xt[j * p + q] : x00;
    h[q] = xq - BtU[j * p + q];
    x[q] = h[q];
  }
  for (int i = 0; i < p; ++i) {
    const int pi = g.piv[i];
    if (pi != i) { const double tt = x[i]; x[i] = x[pi]; x[pi] = tt; }
  }
  for (int i = 0; i < p; ++i)
    for (int k = 0; k < i; ++k) x[i] -= g.lu[i * p + k] * x[k];
  for (int i = p - 1; i >= 0; --i) {
    for (int k = i + 1; k < p; ++k) x[i] -= g.lu[i * p + k] * x[k];
    x[i] /= g.lu[i * p + i];
  }
  double v = var[j];
  for (int q = 0; q < p; ++q) v = fma(h[q], x[q], v);
  if (v < -1.0e-10) {   // exact.py:171-173: keep the most negative for the message
    unsigned long long old = *minvar_bits, assumed;
    do {
      assumed = old;
      if (__longlong_as_double((long long)assumed) <= v) break;
      old = atomicCAS(minvar_bits, assumed, (unsigned long long)__double_as_longlong(v));
    } while (old != assumed);
  }
  out[j] = sqrt(fmax(v, 0.0));
}

static Status exact_targets_check(const rk_fit* f, const double* xt, int64_t nt) {
  if (nt < 0) return Status::err(RK_DOMAIN, "negative target count");
  if (!f->obs) return Status::err(RK_INTERNAL, "fit has no observation locations");
  (void)xt;
  return Status::ok();
}

}  // namespace rk

extern "C" {

rk_status rk_predict_exact(const rk_fit* f, const double* targets_dev, int64_t nt, const double* xt_dev,
                           double x00, double* out_dev, void* stream) {
  auto run = [&]() -> Status {
    RK_TRY(exact_targets_check(f, xt_dev, nt));
    if (nt == 0) return Status::ok();
    cudaStream_t st = (cudaStream_t)stream;
    int* bad = nullptr;
    RK_TRY(scratch_alloc((void**)&bad, sizeof(int), st));
    RK_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
    ExactArgs a{};
    a.mat = f->mat;
    a.obs = f->obs;
    a.c = f->c;
    a.n = f->n;
    a.tgt = targets_dev;
    a.nt = nt;
    a.xt = xt_dev;
    a.x00 = x00;
    a.beta = f->beta;
    a.p = f->p;
    a.out = out_dev;
    a.bad = bad;
    predict_exact_kernel<<<(unsigned)ceil_div(nt, kExactThreads), kExactThreads, 0, st>>>(a);
    count_launch();
    RK_LAUNCH_CHECK();
    int hb = 0;
    RK_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    scratch_free(bad, st);
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    if (hb) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");
    return Status::ok();
  };
  return (rk_status)finish_exact(run());
}

rk_status rk_kriging_se_exact(rk_fit* f, const double* targets_dev, int64_t nt, const double* xt_dev,
                              double x00, int64_t chunk, double* out_dev, void* stream) {
  auto run = [&]() -> Status {
    RK_TRY(exact_targets_check(f, xt_dev, nt));
    if (nt == 0) return Status::ok();
    cudaStream_t st = (cudaStream_t)stream;
    RK_TRY(ensure_uinv(f, st));
    const int64_t n = f->n;
    const int p = f->p;
    // chunk of targets per pass: the caller's, capped so K and u stay within ~4 GB
    int64_t tc = std::max<int64_t>(1, std::min<int64_t>(chunk > 0 ? chunk : 4000, nt));
    tc = std::max<int64_t>(1, std::min<int64_t>(tc, (int64_t)(4.0e9 / (16.0 * (double)n))));
    double *K = nullptr, *U = nullptr, *var = nullptr, *BtU = nullptr;
    int* bad = nullptr;
    unsigned long long* minv = nullptr;
    RK_TRY(scratch_alloc((void**)&K, sizeof(double) * (size_t)n * tc, st));
    RK_TRY(scratch_alloc((void**)&U, sizeof(double) * (size_t)n * tc, st));
    RK_TRY(scratch_alloc((void**)&var, sizeof(double) * (size_t)tc, st));
    RK_TRY(scratch_alloc((void**)&BtU, sizeof(double) * (size_t)p * tc, st));
    RK_TRY(scratch_alloc((void**)&bad, sizeof(int), st));
    RK_TRY(scratch_alloc((void**)&minv, sizeof(unsigned long long), st));
    RK_CUDA_TRY(cudaMemsetAsync(bad, 0, sizeof(int), st));
    const double zero_d = 0.0;
    unsigned long long zero_bits;
    memcpy(&zero_bits, &zero_d, sizeof zero_bits);
    RK_CUDA_TRY(cudaMemcpyAsync(minv, &zero_bits, sizeof zero_bits, cudaMemcpyHostToDevice, st));
    const GramLU g = gram_args(f);
    for (int64_t j0 = 0; j0 < nt; j0 += tc) {
      const int64_t m = std::min<int64_t>(tc, nt - j0);
      cross_cov_kernel<<<(int)std::min<int64_t>(ceil_div(n * m, 256), 148 * 64), 256, 0, st>>>(
          f->mat, f->obs, n, targets_dev + 2 * j0, m, K, bad);
      count_launch();
      RK_LAUNCH_CHECK();
      // u = L^-1 K (DMMA triangular panel product, rk_refit.cu)
      RK_TRY(trmm_linv(f, false, K, n, m, U, n, st));
      colsq_kernel<<<(unsigned)ceil_div(m, 8), 256, 0, st>>>(U, n, m, f->model.sigma2, var);
      count_launch();
      // B'u (p x m), fixed-order per target
      RK_TRY(bta(f, U, n, m, BtU, st));
      se_finish_kernel<<<(unsigned)ceil_div(m, 128), 128, 0, st>>>(g, BtU, xt_dev ? xt_dev + j0 * p : nullptr, x00,
                                                                   m, var, out_dev + j0, minv);
      count_launch();
      RK_LAUNCH_CHECK();
    }
    int hb = 0;
    unsigned long long mb = 0;
    RK_CUDA_TRY(cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
    RK_CUDA_TRY(cudaMemcpyAsync(&mb, minv, sizeof mb, cudaMemcpyDeviceToHost, st));
    for (void* q : {(void*)K, (void*)U, (void*)var, (void*)BtU, (void*)bad, (void*)minv}) scratch_free(q, st);
    RK_CUDA_TRY(cudaStreamSynchronize(st));
    if (hb) return Status::err(RK_NUMERIC, "Temme series / continued fraction for K_nu failed to converge");
    double mv;
    memcpy(&mv, &mb, sizeof mv);
    if (mv < -1.0e-10) {
      char b[128];
      snprintf(b, sizeof b, "negative prediction variance %.3e beyond clamp tolerance", mv);
      return Status::err(RK_NUMERIC, b);
    }
    return Status::ok();
  };
  return (rk_status)finish_exact(run());
}

}  // extern "C"
