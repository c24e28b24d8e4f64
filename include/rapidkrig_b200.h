/*
 * rapidkrig_b200 — C ABI of the B200-native rapid-Kriging hot path.
 *
 * Drop-in boundary for the reference package rapidkrig 0.1.0
 * (/root/reference/pkg/src/rapidkrig).  The reference has no FFI of its own:
 * its boundary is the Python API re-exported at __init__.py:16-49.  Each entry
 * point below replaces the reference function cited beside it; the Python
 * package paper_2605_29284_b200 binds them with ctypes under the reference's
 * names and signatures.
 *
 * Conventions
 *   - plain C types only; device pointers are `const double*` etc. that the
 *     caller allocated on the current CUDA device; `void* stream` is a
 *     cudaStream_t (NULL = legacy default stream).
 *   - every function returns an rk_status; on failure rk_last_error() holds a
 *     thread-local message.  Status -> exception mapping mirrors errors.py:4-17:
 *     RK_DOMAIN -> DomainError, RK_NUMERIC -> NumericError,
 *     RK_INTERNAL -> InternalError, RK_CUDA -> RapidKrigError.
 *   - arrays are row-major [iy, ix] with x fastest (gridding.py:6-8).
 *   - handles are immutable after creation; concurrent calls on different
 *     streams are safe (rapid.py:140-144).
 */
#ifndef RAPIDKRIG_B200_H
#define RAPIDKRIG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum rk_status {
  RK_OK = 0,
  RK_DOMAIN = 1,    /* errors.py:8  DomainError   */
  RK_NUMERIC = 2,   /* errors.py:12 NumericError  */
  RK_INTERNAL = 3,  /* errors.py:16 InternalError */
  RK_CUDA = 4       /* device failure (RapidKrigError) */
} rk_status;

/* CovarianceModel (covariance.py:50-89) plus the host-computed constants of
 * bessel.py (half-integer Horner coefficients 224-234, Temme gammas 37-47,
 * Gamma(nu) 255) so device arithmetic follows the reference's constants. */
typedef struct rk_model {
  double sigma2, alpha, nu, tau2;
  int32_t half_n;          /* n for nu = n + 1/2 (bessel.py:216-221), else -1 */
  int32_t nl;              /* int(nu + 0.5) (bessel.py:245) */
  double half_coef[13];    /* (n+i)!/(i!(n-i)!), i ascending */
  double half_pref;        /* n!/(2n)! */
  double mu;               /* nu - nl */
  double temme_gampl, temme_gammi, temme_gam1, temme_gam2, temme_fact;
  double gamma_nu;         /* math.gamma(nu) */
} rk_model;

/* PaddedGrid (gridding.py:38-111) */
typedef struct rk_grid {
  double x0, y0;           /* interior origin */
  double hx, hy;           /* spacing */
  int32_t m1, m2;          /* interior dims */
  int32_t pad[4];          /* left, right, bottom, top */
} rk_grid;

typedef struct rk_setup rk_setup;   /* device-resident RapidSetup (rapid.py:138-174) */
typedef struct rk_fit rk_fit;       /* device-resident KrigingFit (exact.py:40-56)  */

/* ---- library ------------------------------------------------------------ */
const char* rk_last_error(void);
int32_t rk_version(void);
/* number of kernels this library launched on the calling thread so far */
int64_t rk_launch_count(void);

/* ---- L0: Matern correlation (bessel.py:258-278 via covariance.py:83-89) --- */
/* out[i] = sigma2 * phi(alpha * d[i]); d, out device arrays of length n */
rk_status rk_matern_cov(const rk_model* model, const double* d_dev, double* out_dev,
                        int64_t n, void* stream);

/* ---- L1: padded grid (gridding.py:130-178) ------------------------------ */
/* obs_host: (n, 2) host array; fills grid (origin, spacing, dims, pads) */
rk_status rk_build_padded_grid(const double domain[4], int32_t m1, int32_t m2, int32_t L,
                               const double* obs_host, int64_t n, rk_grid* grid_out);

/* ---- L2: rapid setup (rapid.py:177-230) --------------------------------- */
/* Builds K_N and its Cholesky (rapid.py:112-135), stencil base indices
 * (gridding.py:181-205), weights + conditional variance (rapid.py:202-225)
 * and the filter spectrum (rapid.py:72-86), all device resident.
 * *ridge_applied = 1 when the K_N ridge retry fired (RuntimeWarning upstream). */
rk_status rk_build_setup(const rk_model* model, const rk_grid* grid, int32_t L,
                         const double* obs_host, int64_t n, rk_setup** out,
                         int32_t* ridge_applied);
/* Observation-free setup: filter spectrum (rapid.py:72-86) and, on demand, the
 * circulant embedding (simulate.py:82-100) for a (model, grid) pair.  Serves
 * build_filter_spectrum and sim_unconditional_grid, which take no observations. */
rk_status rk_grid_setup_create(const rk_model* model, const rk_grid* grid, rk_setup** out);
rk_status rk_setup_destroy(rk_setup* s);
/* n_obs, L, embed dims (p1, p2), padded dims (M1, M2) */
rk_status rk_setup_info(const rk_setup* s, int64_t* n_obs, int32_t* L, int32_t embed[2],
                        int32_t total[2]);
/* Materialise the RapidSetup fields on the host (any pointer may be NULL):
 * neighbor_indices (n, M) int64, weights (n, M), cond_var (n), kn_inv (M, M). */
rk_status rk_setup_copy_out(const rk_setup* s, int64_t* indices_host, double* weights_host,
                            double* cond_var_host, double* kn_inv_host);
/* Filter spectrum real part, full (p2, p1) layout, UNSCALED like np.fft.fft2
 * (rapid.py:86); imaginary part is zero for the even lag filter.  Always on the reference's
 * torus (embed dims of rk_setup_info). */
rk_status rk_setup_copy_spectrum(const rk_setup* s, double* spectrum_host);
/* The torus predict_rapid executes on (p1, p2): the reference's embed dims, or along y a
 * shorter 2^a 3^b length whose few aliased lags are corrected exactly (no reference
 * counterpart: rapid.py:72-86 fixes the torus; the predicted field is the same). */
rk_status rk_setup_exec_dims(const rk_setup* s, int32_t dims[2]);

/* ---- L2: rapid predict (rapid.py:164-174, 89-100, 233-261) -------------- */
/* c* = A' c  (RapidSetup.coefficients_to_grid, rapid.py:164-174); device arrays */
rk_status rk_coefficients_to_grid(const rk_setup* s, const double* c_dev, double* cstar_dev,
                                  void* stream);
/* convolve_filter (rapid.py:89-100) of a padded (M2, M1) device field with the
 * setup's spectrum; out (M2, M1) */
rk_status rk_convolve_filter(const rk_setup* s, const double* values_dev, double* out_dev,
                             void* stream);
/* convolve_filter (rapid.py:89-100) with a caller-supplied real-even spectrum in
 * quarter form spec_q[kx * ldq + ky] = Re S[ky, kx] / (p1 p2), kx <= p1/2, ky <= p2/2,
 * ldq = p2/2+1 rounded up to even, 16-byte aligned (device); values/out (M2, M1) device. */
rk_status rk_convolve_spectrum(const double* spec_q_dev, int32_t p1, int32_t p2,
                               const double* values_dev, int32_t M1, int32_t M2, double* out_dev,
                               void* stream);
/* predict_rapid (rapid.py:252-261), device pointers.  beta_dev may be NULL
 * (no fixed part); p = len(beta); xg_dev (m1*m2, p) row-major or NULL
 * (then p must be 1: scalar beta[0]).  out_dev (m2, m1). */
rk_status rk_predict_dev(const rk_setup* s, const double* c_dev, const double* beta_dev,
                         int32_t p, const double* xg_dev, double* out_dev, void* stream);
/* Same call on HOST buffers: H2D of c / beta / xg, compute, D2H of the field,
 * synchronous on `stream`, or on the setup's own non-blocking stream when `stream` is
 * NULL (such calls on one setup are serialised).  Pinned buffers take one captured graph
 * with the X_g upload on a side stream overlapping the first two passes. */
rk_status rk_predict_host(const rk_setup* s, const double* c, const double* beta, int32_t p,
                          const double* xg, double* out, void* stream);

/* Benchmark support: average CUDA-event duration (ms) of the per-observation weights
 * kernel (rapid.py:202-225: stencil, Matern cross covariance, two substitutions against
 * the K_N factor, cond_var) over `reps` back-to-back launches on this setup's
 * observations, into scratch outputs (the setup is unchanged); synchronises the stream. */
rk_status rk_setup_time_weights(const rk_setup* s, void* stream, int32_t reps, float* ms_out);

/* predict_rapid with per-kernel CUDA-event timing on `stream` (benchmark support):
 * ms_out[0..3] = gather (c* = A'c), pass 1 (row FFT), pass 2 (column filter),
 * pass 3 (row IFFT + epilogue) durations in milliseconds; synchronises the stream. */
/* K1 alone into caller device buffers: base (n) int32, w (n, M), cv (n), err (4 int32,
 * initialised by the caller to {INT_MAX, INT_MAX, 0, 0}); asynchronous on `stream`.  A predict
 * step from observation coordinates is this + rk_predict_dev (SURVEY 8(d) T_predict). */
rk_status rk_setup_weights_into(const rk_setup* s, int32_t* base_dev, double* w_dev, double* cv_dev,
                                int32_t* err_dev, void* stream);
rk_status rk_predict_profile(const rk_setup* s, const double* c_dev, const double* beta_dev,
                             int32_t p, const double* xg_dev, double* out_dev, void* stream,
                             float* ms_out);
/* algorithmic bytes per kernel of rk_predict_* for this setup:
 * bytes_out[0..3] as in rk_predict_profile, for p covariates (0 = no fixed part).
 * The scatter is fused into pass 1, so entry 0 (and ms_out[0]) is 0. */
rk_status rk_predict_traffic(const rk_setup* s, int32_t p, double* bytes_out);

/* ---- L2: exact fit / refit (exact.py:71-113) ---------------------------- */
/* GPU fit: M = K + tau2 I (covariance.py:100-116), Cholesky with ridge retry
 * (exact.py:25-37), GLS (exact.py:59-68).  X_host (n, p) row-major or NULL. */
rk_status rk_fit_create(const rk_model* model, const double* obs_host, int64_t n,
                        const double* z_host, const double* X_host, int32_t p, rk_fit** out,
                        int32_t* ridge_applied);
/* Adopt a host KrigingFit (reference object): chol_M (n, n) lower row-major,
 * X (n, p), beta (p), c (n). */
rk_status rk_fit_import(const rk_model* model, const double* obs_host, int64_t n,
                        const double* X_host, int32_t p, const double* chol_host,
                        const double* beta_host, const double* c_host, rk_fit** out);
rk_status rk_fit_destroy(rk_fit* f);
/* copies out beta (p), c (n), chol_M (n, n lower, row-major); NULL skips */
rk_status rk_fit_copy_out(const rk_fit* f, double* beta_host, double* c_host, double* chol_host);
rk_status rk_fit_info(const rk_fit* f, int64_t* n, int32_t* p);
/* refit_coefficients (exact.py:108-113) for `batch` right-hand sides:
 * z_dev (batch, n) -> beta_dev (batch, p), c_dev (batch, n) */
rk_status rk_refit_dev(const rk_fit* f, const double* z_dev, int64_t batch, double* beta_dev,
                       double* c_dev, void* stream);

/* predict_exact (exact.py:132-147): out[t] = x_t . beta + sum_i cov(|t - obs_i|) c_i for
 * targets_dev (nt, 2); xt_dev (nt, p) row-major, or NULL for an intercept-only fit, whose
 * target covariate is x00 = X[0, 0] (exact.py:116-121).  Fixed summation order (index order). */
rk_status rk_predict_exact(const rk_fit* f, const double* targets_dev, int64_t nt, const double* xt_dev,
                           double x00, double* out_dev, void* stream);
/* kriging_se_exact (exact.py:150-175): sqrt(sigma2 - k'M^-1 k + h'(X'M^-1X)^-1 h) per target,
 * h = x_t - k'M^-1 X; processed `chunk` targets at a time (<= 0: 4000); RK_NUMERIC
 * "negative prediction variance ..." below -1e-10, values in [-1e-10, 0) clamp to 0. */
rk_status rk_kriging_se_exact(rk_fit* f, const double* targets_dev, int64_t nt, const double* xt_dev,
                              double x00, int64_t chunk, double* out_dev, void* stream);

/* ---- L3: conditional simulation (simulate.py:52-192) -------------------- */
/* seed ^ splitmix64(j)  (simulate.py:52-62) */
uint64_t rk_draw_seed(uint64_t seed, uint64_t j);
/* Standard normals from the Philox4x64-10 stream keyed (seed, stream), words
 * [start, start+count) (simulate.py:65-74) -> device out */
rk_status rk_philox_normals(uint64_t seed, uint64_t stream_id, uint64_t start, int64_t count,
                            double* out_dev, void* stream);
/* raw Philox words (for bit-exactness tests) */
rk_status rk_philox_raw(uint64_t seed, uint64_t stream_id, uint64_t start, int64_t count,
                        uint64_t* out_dev, void* stream);
/* circulant embedding (simulate.py:82-100): dims after the PSD check / doubling.
 * Fails with RK_NUMERIC ("... most negative eigenvalue ...") if still indefinite. */
rk_status rk_setup_embedding(rk_setup* s, int32_t embed_out[2], int32_t* doubled);
/* sim_unconditional_grid (simulate.py:103-118): field_dev (M2, M1) */
rk_status rk_sim_unconditional_dev(rk_setup* s, uint64_t seed, double* field_dev, void* stream);
/* sim_obs_local (simulate.py:121-143): field_dev (M2, M1) -> z_dev (n) */
rk_status rk_sim_obs_local_dev(const rk_setup* s, double tau2, const double* field_dev,
                               uint64_t seed, double* z_dev, void* stream);
/* Ensemble slice (simulate.py:146-192): realizations j in [j0, j0+count) with
 * sub-seeds draw_seed(seed, j).  Adds, per pixel,
 *   e_j = interior(g_j) - predict_rapid(c_sim_j, beta_sim_j)
 * into the exact fixed-point moment accumulator acc_dev (int64, 6 * m2*m1, caller-zeroed):
 * s1 = sum e, s2 = sum e^2 as trunc(v 2^64) in three signed 42-bit digits (v = e / 2^k, 2^k the
 * power of two nearest sigma).  Integer sums are order-free: the result is bitwise the same
 * for any batch size, split into slices, or number of GPUs.  draw_j = data_pred + e_j is
 * written to draws_dev (count, m2, m1) if non-NULL.  xg_dev / p as in rk_predict_dev.
 * RK_NUMERIC if a draw deviates by >= 2^20 sigma (outside the fixed-point range). */
rk_status rk_ensemble_accumulate(rk_setup* s, const rk_fit* f, uint64_t seed, int64_t j0,
                                 int64_t count, const double* xg_dev,
                                 const double* data_pred_dev, long long* acc_dev,
                                 double* draws_dev, int32_t batch, void* stream);
/* the fixed-point accumulation alone: acc_dev += moments of e_dev (count, n_pix) */
rk_status rk_ensemble_accumulate_values(const double* e_dev, int32_t count, int64_t n_pix, double sigma2,
                                        long long* acc_dev, void* stream);
/* dst += src (two accumulators of n_pix pixels; exact) */
rk_status rk_ensemble_combine(long long* dst_dev, const long long* src_dev, int64_t n_pix, void* stream);
/* mean = data_pred + s1/R ; se = sqrt(max((s2 - s1*s1/R)/(R-1), 0)) (simulate.py:191-192);
 * sigma2 = the model's (fixes the accumulator scale) */
rk_status rk_ensemble_finalize(int64_t n_pix, int64_t n_draws, double sigma2,
                               const double* data_pred_dev, const long long* acc_dev,
                               double* mean_dev, double* se_dev, void* stream);
/* build the fit's inverse factor L^-1 used by the batched refits now (otherwise on the
 * first refit); cuSOLVER trtri -- setup, once per fit */
rk_status rk_fit_prepare_refit(rk_fit* f, void* stream);
/* kernel timing of the refit's two triangular panel products for S right-hand sides
 * (CUDA events, mean of reps): ms_out[0] = L^-1 Z, ms_out[1] = L^-T H */
rk_status rk_refit_profile(rk_fit* f, int64_t S, int32_t reps, void* stream, float* ms_out);

/* ---- moving setups / fits between GPUs (ensemble sharding, rk_replicate.cu) ---- */
/* copy onto `device` peer to peer (one process, several GPUs) */
rk_status rk_setup_replicate(const rk_setup* src, int32_t device, rk_setup** out);
rk_status rk_fit_replicate(const rk_fit* src, int32_t device, rk_fit** out);
/* setup as one device blob (for a broadcast between processes): size, export into a
 * caller buffer on the setup's device, import on the current device */
rk_status rk_setup_blob_bytes(const rk_setup* s, int64_t* bytes);
rk_status rk_setup_export(const rk_setup* s, void* blob_dev, void* stream);
rk_status rk_setup_import(const void* blob_dev, int64_t bytes, rk_setup** out);
/* fit arrays broadcast in place: an empty fit on the current device, its 7 array pointers /
 * sizes (U, X, B, beta, c, obs, U^-1; NULL / 0 if absent), and the p x p Gram LU + pivots */
rk_status rk_fit_shell(const rk_model* model, int64_t n, int32_t p, int32_t with_uinv, rk_fit** out);
rk_status rk_fit_fields(const rk_fit* f, void** ptrs, int64_t* bytes);
rk_status rk_fit_get_gram(const rk_fit* f, double* lu, int32_t* piv);
rk_status rk_fit_set_gram(rk_fit* f, const double* lu, const int32_t* piv);

#ifdef __cplusplus
}
#endif

#endif /* RAPIDKRIG_B200_H */
