// Common definitions for the rapidkrig B200 library: status codes, error
// reporting (thread-local last error), CUDA checks, complex helpers.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>
#include <cuda_runtime.h>

#include "../../include/rapidkrig_b200.h"

namespace rk {

// thread-local message behind rk_last_error()
void set_error(int code, const std::string& msg);
int last_code();

struct Status {
  int code = RK_OK;
  std::string msg;
  static Status ok() { return Status(); }
  static Status err(int c, std::string m) { Status s; s.code = c; s.msg = std::move(m); return s; }
  bool good() const { return code == RK_OK; }
};

#define RK_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess)                                                             \
      return ::rk::Status::err(RK_CUDA, std::string("CUDA error ") +                   \
                               cudaGetErrorString(_e) + " at " __FILE__ ":" +         \
                               std::to_string(__LINE__) + " (" #expr ")");           \
  } while (0)

#define RK_TRY(expr)                      \
  do {                                    \
    ::rk::Status _s = (expr);             \
    if (!_s.good()) return _s;            \
  } while (0)

#define RK_LAUNCH_CHECK() RK_CUDA_TRY(cudaGetLastError())

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- complex ops
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// --------------------------------------------- TMA bulk copies + mbarrier (sm_90+)
// 1-D bulk tensor-less copies (cp.async.bulk): global -> shared completes on an
// mbarrier with a transaction-byte count; shared -> global is a bulk-group store.
// Addresses must be 16-byte aligned and sizes multiples of 16.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() {
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
}
// 8-byte asynchronous global -> shared copies (LDGSTS): no register round trip, any
// 8-byte alignment; used to prefetch epilogue operands while a line is transformed
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
// Programmatic dependent launch (sm_90+): a kernel launched with the programmatic
// serialization attribute may start while its predecessor drains; it must execute
// pdl_wait() before reading anything the predecessor writes.  pdl_trigger() lets the
// next kernel in the stream begin its own prologue early.  Enabled with RK_PDL=1; without
// the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class... KArgs, class... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  static const int enabled = [] {
    const char* e = getenv("RK_PDL");
    return e ? atoi(e) : 0;   // off by default: measured slower on B200 (cfg2 37.4 vs 35.1 us)
  }();
  cfg.numAttrs = enabled ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Exit protection of a 2-CTA cluster whose CTAs read each other's shared memory, lighter than a
// second barrier.cluster (whose fence and L1 invalidation every thread pays): each CTA arrives
// (release, cluster scope) on an mbarrier in its PARTNER's shared memory once all of its threads
// have finished their remote reads, and before exiting waits (acquire, cluster scope) until its
// own mbarrier has seen the partner's arrival.  The mbarrier (count 1) is initialised before the
// cluster's first barrier.cluster, which publishes it.
__device__ __forceinline__ void cluster_arrive_partner(uint64_t* bar, uint32_t partner) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(bar)), "r"(partner));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(r) : "memory");
}
__device__ __forceinline__ void cluster_wait_partner(uint64_t* bar) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], 0;\n"
      "@!P1 bra WAITC_%=;\n"
      "}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// 256-bit global accesses (sm_100: LDG.256 / STG.256), 32-byte aligned: two adjacent double2 in one
// request -- the transposed row-pair pieces of T and U are 32 bytes per (column, row pair), and
// the strided gathers / scatters of passes 1 and 3 are bound by the number of L1 requests
__device__ __forceinline__ void ldg256(const double2* p, double2& a, double2& b) {
  asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a.x), "=d"(a.y), "=d"(b.x), "=d"(b.y) : "l"(p));
}
__device__ __forceinline__ void stg256(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y) : "memory");
}
__device__ __forceinline__ bool aligned32(const void* p, int64_t ld_elems16) {
  return ((uintptr_t)p & 31) == 0 && (ld_elems16 & 1) == 0;
}

// make generic-proxy smem writes visible to the async (TMA) proxy before a bulk store
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

}  // namespace rk
