// rapidkrig B200: moving an immutable setup / fit to other GPUs.
//
// The conditional-simulation ensemble shards realizations over GPUs (simulate.py:174-192:
// realization j depends only on (seed, j)), and every GPU needs the same setup (rapid.py:
// 138-174, immutable in use) and fit (exact.py:40-56).  Rebuilding them per GPU repeats the
// n x n Cholesky (20 GB at n = 50000); instead they are built once and copied:
//   * one process, several GPUs: rk_setup_replicate / rk_fit_replicate copy every device array
//     peer to peer (NVLink) onto the target device;
//   * one process per GPU (torch.distributed): the setup travels as one device blob
//     (rk_setup_export -> NCCL broadcast -> rk_setup_import); the fit's arrays are broadcast in
//     place into a shell (rk_fit_shell + rk_fit_fields), its p x p Gram LU through
//     rk_fit_get_gram / rk_fit_set_gram.
// Copies are bitwise, so every GPU computes bitwise the same realizations.
#include <algorithm>
#include <cstring>
#include <memory>
#include <vector>

#include <cublas_v2.h>

#include "rk_internal.cuh"

namespace rk {

namespace {

struct SetupHdr {
  uint64_t magic;
  rk_model model;
  rk_grid grid;
  int32_t L, bs, M, M1, M2, m1, m2, p1, p2, H1, Q2, pblk_cap, ldh;
  int64_t n, nnodes, max_pair_ent, max_half_ent, pblk_stride;
  double px0, py0, cond_var_min;
  int32_t emb_ready, ps1, ps2, doubled, hs1, qs2;
  int32_t rp1, rp2;
  AliasCorr ac;
  int64_t field_bytes[24];
  int32_t nfields, has_field[24];
};
constexpr uint64_t kSetupMagic = 0x52'4B'53'45'54'55'50'33ULL;   // "RKSETUP3"

struct Field {
  void** slot;
  size_t bytes;
};

// every device array of a setup with its size (fixed order)
std::vector<Field> setup_fields(rk_setup* s) {
  const int64_t n = s->n, M = s->M, tot = n * M;
  const int npairs = (s->M2 + 1) / 2;
  std::vector<Field> f = {
      {(void**)&s->obs, sizeof(double) * 2 * n},
      {(void**)&s->base, sizeof(int32_t) * n},
      {(void**)&s->weights, sizeof(double) * tot},
      {(void**)&s->cond_var, sizeof(double) * n},
      {(void**)&s->perm, sizeof(int32_t) * n},
      {(void**)&s->bsort, sizeof(int32_t) * n},
      {(void**)&s->wsort, sizeof(double) * tot},
      {(void**)&s->cell_start, sizeof(int32_t) * ((int64_t)s->M1 * s->M2 + 1)},
      {(void**)&s->node_q, sizeof(int32_t) * (s->nnodes + 5)},
      {(void**)&s->node_off, sizeof(int32_t) * (s->nnodes + 5)},
      {(void**)&s->row_node, sizeof(int32_t) * (s->M2 + 1)},
      {(void**)&s->ent_w, sizeof(int32_t) * tot},
      {(void**)&s->ent_c, sizeof(int32_t) * (tot + 4)},
      {(void**)&s->ent_wv, sizeof(double) * (std::max<int64_t>(tot, 1) + 2)},
      {(void**)&s->pair_info, sizeof(int4) * (npairs + 1)},
      {(void**)&s->pblk, (size_t)(s->pblk_stride * npairs)},
      {(void**)&s->spec_q, sizeof(double) * (size_t)s->H1 * s->Q2},
      {(void**)&s->spec_s, sizeof(double) * (size_t)s->H1 * 2 * s->ldh},
      {(void**)&s->kn_chol_dev, sizeof(double) * M * M},
      {(void**)&s->emb.root_q, sizeof(double) * (size_t)s->emb.hs1 * s->emb.qs2},
      {(void**)&s->ac_ker, sizeof(double) * ((size_t)s->ac.nkr * (2 * s->M1 - 1) + (size_t)s->ac.nkc * (2 * s->M2 - 1))},
  };
  return f;
}

size_t align16(size_t v) { return (v + 15) & ~size_t(15); }

SetupHdr header_of(rk_setup* s) {
  SetupHdr h;
  memset(&h, 0, sizeof h);
  h.magic = kSetupMagic;
  h.model = s->model;
  h.grid = s->grid;
  h.L = s->L; h.bs = s->bs; h.M = s->M; h.M1 = s->M1; h.M2 = s->M2; h.m1 = s->m1; h.m2 = s->m2;
  h.p1 = s->p1; h.p2 = s->p2; h.H1 = s->H1; h.Q2 = s->Q2; h.pblk_cap = s->pblk_cap; h.ldh = s->ldh;
  h.n = s->n; h.nnodes = s->nnodes; h.max_pair_ent = s->max_pair_ent; h.max_half_ent = s->max_half_ent;
  h.pblk_stride = s->pblk_stride;
  h.px0 = s->px0; h.py0 = s->py0; h.cond_var_min = s->cond_var_min;
  h.emb_ready = s->emb.ready; h.ps1 = s->emb.ps1; h.ps2 = s->emb.ps2; h.doubled = s->emb.doubled;
  h.hs1 = s->emb.hs1; h.qs2 = s->emb.qs2;
  h.rp1 = s->rp1; h.rp2 = s->rp2; h.ac = s->ac;
  const auto f = setup_fields(s);
  h.nfields = (int32_t)f.size();
  for (size_t i = 0; i < f.size(); ++i) {
    h.has_field[i] = *f[i].slot != nullptr;
    h.field_bytes[i] = h.has_field[i] ? (int64_t)f[i].bytes : 0;
  }
  return h;
}

size_t blob_bytes(const SetupHdr& h) {
  size_t b = align16(sizeof(SetupHdr)) + align16(sizeof(double) * 2 * (size_t)h.M * h.M);
  for (int i = 0; i < h.nfields; ++i) b += align16((size_t)h.field_bytes[i]);
  return b;
}

// host state of a setup from its header: plans are rebuilt on the current device
Status setup_from_header(const SetupHdr& h, rk_setup* s) {
  if (h.magic != kSetupMagic) return Status::err(RK_DOMAIN, "not a rapidkrig setup blob");
  RK_CUDA_TRY(cudaGetDevice(&s->device));
  s->model = h.model;
  s->mat = make_matern_dev(h.model);
  s->grid = h.grid;
  s->L = h.L; s->bs = h.bs; s->M = h.M; s->M1 = h.M1; s->M2 = h.M2; s->m1 = h.m1; s->m2 = h.m2;
  s->p1 = h.p1; s->p2 = h.p2; s->H1 = h.H1; s->Q2 = h.Q2; s->pblk_cap = h.pblk_cap; s->ldh = h.ldh;
  s->n = h.n; s->nnodes = h.nnodes; s->max_pair_ent = h.max_pair_ent; s->max_half_ent = h.max_half_ent;
  s->pblk_stride = h.pblk_stride;
  s->px0 = h.px0; s->py0 = h.py0; s->cond_var_min = h.cond_var_min;
  s->rp1 = h.rp1; s->rp2 = h.rp2; s->ac = h.ac;
  RK_TRY(setup_plans(s));
  Embedding& e = s->emb;
  e.ps1 = h.ps1; e.ps2 = h.ps2; e.doubled = h.doubled; e.hs1 = h.hs1; e.qs2 = h.qs2;
  if (h.emb_ready) RK_TRY(embedding_plans(s));
  return Status::ok();
}

// device arrays of `s` (on the current device) filled from `src_of(i)` (same device or peer)
template <class Src>
Status fill_fields(rk_setup* s, const SetupHdr& h, Src src_of, cudaStream_t st) {
  auto f = setup_fields(s);
  if ((int)f.size() != h.nfields) return Status::err(RK_DOMAIN, "setup blob from another library version");
  for (size_t i = 0; i < f.size(); ++i) {
    if (!h.has_field[i]) continue;
    RK_CUDA_TRY(cudaMalloc(f[i].slot, std::max<size_t>((size_t)h.field_bytes[i], 16)));
    RK_TRY(src_of((int)i, *f[i].slot, (size_t)h.field_bytes[i], st));
  }
  s->emb.ready = h.emb_ready != 0;
  return Status::ok();
}

}  // namespace

}  // namespace rk

using namespace rk;

static int finish_rep(const Status& s) {
  if (!s.good()) rk::set_error(s.code, s.msg);
  return s.code;
}

extern "C" {

rk_status rk_setup_blob_bytes(const rk_setup* s, int64_t* bytes) {
  const SetupHdr h = header_of(const_cast<rk_setup*>(s));
  *bytes = (int64_t)blob_bytes(h);
  return RK_OK;
}

rk_status rk_setup_export(const rk_setup* s, void* blob_dev, void* stream) {
  auto run = [&]() -> Status {
    rk_setup* ms = const_cast<rk_setup*>(s);
    cudaStream_t st = (cudaStream_t)stream;
    const SetupHdr h = header_of(ms);
    unsigned char* b = (unsigned char*)blob_dev;
    RK_CUDA_TRY(cudaMemcpyAsync(b, &h, sizeof h, cudaMemcpyHostToDevice, st));
    size_t off = align16(sizeof(SetupHdr));
    const size_t mm = sizeof(double) * (size_t)h.M * h.M;
    if (h.M > 0 && !ms->kn_chol.empty()) {
      RK_CUDA_TRY(cudaMemcpyAsync(b + off, ms->kn_chol.data(), mm, cudaMemcpyHostToDevice, st));
      RK_CUDA_TRY(cudaMemcpyAsync(b + off + mm, ms->kn_inv.data(), mm, cudaMemcpyHostToDevice, st));
    }
    off += align16(2 * mm);
    const auto f = setup_fields(ms);
    for (size_t i = 0; i < f.size(); ++i) {
      if (h.has_field[i])
        RK_CUDA_TRY(cudaMemcpyAsync(b + off, *f[i].slot, (size_t)h.field_bytes[i], cudaMemcpyDeviceToDevice, st));
      off += align16((size_t)h.field_bytes[i]);
    }
    RK_CUDA_TRY(cudaStreamSynchronize(st));   // the host header / factor staging is released
    return Status::ok();
  };
  return (rk_status)finish_rep(run());
}

rk_status rk_setup_import(const void* blob_dev, int64_t bytes, rk_setup** out) {
  auto run = [&]() -> Status {
    SetupHdr h;
    if (bytes < (int64_t)sizeof h) return Status::err(RK_DOMAIN, "setup blob too small");
    RK_CUDA_TRY(cudaMemcpy(&h, blob_dev, sizeof h, cudaMemcpyDeviceToHost));
    if (h.magic != kSetupMagic) return Status::err(RK_DOMAIN, "not a rapidkrig setup blob");
    if ((int64_t)blob_bytes(h) != bytes) return Status::err(RK_DOMAIN, "setup blob size mismatch");
    rk_setup* s = new rk_setup();
    std::unique_ptr<rk_setup, void (*)(rk_setup*)> guard(s, free_setup);
    RK_TRY(setup_from_header(h, s));
    const unsigned char* b = (const unsigned char*)blob_dev;
    size_t off = align16(sizeof(SetupHdr));
    const size_t mm = sizeof(double) * (size_t)h.M * h.M;
    if (h.n > 0 && h.M > 0) {
      s->kn_chol.resize((size_t)h.M * h.M);
      s->kn_inv.resize((size_t)h.M * h.M);
      RK_CUDA_TRY(cudaMemcpy(s->kn_chol.data(), b + off, mm, cudaMemcpyDeviceToHost));
      RK_CUDA_TRY(cudaMemcpy(s->kn_inv.data(), b + off + mm, mm, cudaMemcpyDeviceToHost));
    }
    off += align16(2 * mm);
    std::vector<size_t> offs(h.nfields);
    for (int i = 0; i < h.nfields; ++i) {
      offs[i] = off;
      off += align16((size_t)h.field_bytes[i]);
    }
    RK_TRY(fill_fields(s, h, [&](int i, void* dst, size_t nb, cudaStream_t st) -> Status {
      RK_CUDA_TRY(cudaMemcpyAsync(dst, b + offs[i], nb, cudaMemcpyDeviceToDevice, st));
      return Status::ok();
    }, (cudaStream_t)0));
    RK_CUDA_TRY(cudaDeviceSynchronize());
    *out = guard.release();
    return Status::ok();
  };
  return (rk_status)finish_rep(run());
}

rk_status rk_setup_replicate(const rk_setup* src, int32_t device, rk_setup** out) {
  auto run = [&]() -> Status {
    rk_setup* ms = const_cast<rk_setup*>(src);
    int cur = 0;
    RK_CUDA_TRY(cudaGetDevice(&cur));
    RK_CUDA_TRY(cudaSetDevice(device));
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{cur};
    const SetupHdr h = header_of(ms);
    rk_setup* s = new rk_setup();
    std::unique_ptr<rk_setup, void (*)(rk_setup*)> guard(s, free_setup);
    RK_TRY(setup_from_header(h, s));
    s->kn_chol = ms->kn_chol;
    s->kn_inv = ms->kn_inv;
    const auto sf = setup_fields(ms);
    RK_TRY(fill_fields(s, h, [&](int i, void* dst, size_t nb, cudaStream_t st) -> Status {
      RK_CUDA_TRY(cudaMemcpyPeerAsync(dst, device, *sf[i].slot, ms->device, nb, st));
      return Status::ok();
    }, (cudaStream_t)0));
    RK_CUDA_TRY(cudaDeviceSynchronize());
    *out = guard.release();
    return Status::ok();
  };
  return (rk_status)finish_rep(run());
}

// ---------------------------------------------------------------- fits
// field order: U (n n), X (n p), B (n p), beta (p), c (n), obs (2 n), Uinv (n n, if built)
static void fit_field_list(rk_fit* f, void*** slots, size_t* bytes) {
  const size_t n = (size_t)f->n, p = (size_t)f->p;
  void** sl[7] = {(void**)&f->U, (void**)&f->X, (void**)&f->B, (void**)&f->beta, (void**)&f->c, (void**)&f->obs,
                  (void**)&f->Uinv};
  const size_t by[7] = {8 * n * n, 8 * n * p, 8 * n * p, 8 * p, 8 * n, 16 * n, 8 * n * n};
  for (int i = 0; i < 7; ++i) {
    slots[i] = sl[i];
    bytes[i] = by[i];
  }
}

rk_status rk_fit_replicate(const rk_fit* src, int32_t device, rk_fit** out) {
  auto run = [&]() -> Status {
    rk_fit* ms = const_cast<rk_fit*>(src);
    std::lock_guard<std::mutex> lk(ms->uinv_mu);   // not while U^-1 is being built
    int cur = 0;
    RK_CUDA_TRY(cudaGetDevice(&cur));
    RK_CUDA_TRY(cudaSetDevice(device));
    struct Restore {
      int d;
      ~Restore() { cudaSetDevice(d); }
    } restore{cur};
    rk_fit* f = new rk_fit();
    std::unique_ptr<rk_fit, void (*)(rk_fit*)> guard(f, free_fit);
    f->device = device;
    f->model = ms->model;
    f->n = ms->n;
    f->p = ms->p;
    f->mat = ms->mat;
    f->gram_lu = ms->gram_lu;
    f->gram_piv = ms->gram_piv;
    cublasHandle_t h;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return Status::err(RK_CUDA, "cublasCreate failed");
    f->cublas = h;
    void** ds[7];
    void** ss[7];
    size_t by[7];
    fit_field_list(f, ds, by);
    fit_field_list(ms, ss, by);
    for (int i = 0; i < 7; ++i) {
      if (!*ss[i]) continue;
      RK_CUDA_TRY(cudaMalloc(ds[i], std::max<size_t>(by[i], 16)));
      RK_CUDA_TRY(cudaMemcpyPeerAsync(*ds[i], device, *ss[i], ms->device, by[i], 0));
    }
    RK_CUDA_TRY(cudaDeviceSynchronize());
    *out = guard.release();
    return Status::ok();
  };
  return (rk_status)finish_rep(run());
}

// empty fit on the current device whose arrays the caller fills (e.g. by a broadcast)
rk_status rk_fit_shell(const rk_model* model, int64_t n, int32_t p, int32_t with_uinv, rk_fit** out) {
  auto run = [&]() -> Status {
    if (n < 1 || p < 1 || p > 8) return Status::err(RK_DOMAIN, "need n >= p >= 1 (p <= 8)");
    rk_fit* f = new rk_fit();
    std::unique_ptr<rk_fit, void (*)(rk_fit*)> guard(f, free_fit);
    RK_CUDA_TRY(cudaGetDevice(&f->device));
    f->model = *model;
    f->n = n;
    f->p = p;
    f->mat = make_matern_dev(*model);
    cublasHandle_t h;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return Status::err(RK_CUDA, "cublasCreate failed");
    f->cublas = h;
    f->gram_lu.assign((size_t)p * p, 0.0);
    f->gram_piv.assign(p, 0);
    void** ds[7];
    size_t by[7];
    fit_field_list(f, ds, by);
    for (int i = 0; i < 7; ++i) {
      if (i == 6 && !with_uinv) continue;
      RK_CUDA_TRY(cudaMalloc(ds[i], std::max<size_t>(by[i], 16)));
    }
    *out = guard.release();
    return Status::ok();
  };
  return (rk_status)finish_rep(run());
}

// device pointers and byte sizes of the fit's arrays (field order above; NULL if absent)
rk_status rk_fit_fields(const rk_fit* f, void** ptrs, int64_t* bytes) {
  void** ss[7];
  size_t by[7];
  fit_field_list(const_cast<rk_fit*>(f), ss, by);
  for (int i = 0; i < 7; ++i) {
    ptrs[i] = *ss[i];
    bytes[i] = *ss[i] ? (int64_t)by[i] : 0;
  }
  return RK_OK;
}

rk_status rk_fit_get_gram(const rk_fit* f, double* lu, int32_t* piv) {
  for (int i = 0; i < f->p * f->p; ++i) lu[i] = f->gram_lu[i];
  for (int i = 0; i < f->p; ++i) piv[i] = f->gram_piv[i];
  return RK_OK;
}

rk_status rk_fit_set_gram(rk_fit* f, const double* lu, const int32_t* piv) {
  for (int i = 0; i < f->p * f->p; ++i) f->gram_lu[i] = lu[i];
  for (int i = 0; i < f->p; ++i) f->gram_piv[i] = piv[i];
  return RK_OK;
}

}  // extern "C"
