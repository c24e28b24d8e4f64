// Common definitions for the rapidkrig B200 library: status codes, error
// reporting (thread-local last error), CUDA checks, complex helpers.
#pragma once

#include <cstdint>
#include <cstdio>
#include <string>
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

}  // namespace rk
