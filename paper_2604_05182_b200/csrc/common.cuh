// Shared helpers for the LSRM B200 kernels: status/error plumbing, launch
// accounting and exact (no-FMA) f64 arithmetic for the bit-exact router and
// compaction paths.
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>

#include "../../include/lsrm_b200.h"

namespace lsrm {

int set_error(int code, const char* fmt, ...);
void count_launch();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define LSRM_REQUIRE(cond, ...)                                   \
  do {                                                            \
    if (!(cond)) return ::lsrm::set_error(LSRM_E_CONFIG, __VA_ARGS__); \
  } while (0)

#define LSRM_CUDA(expr)                                                     \
  do {                                                                      \
    cudaError_t _e = (expr);                                                \
    if (_e != cudaSuccess)                                                  \
      return ::lsrm::set_error(LSRM_E_CUDA, "%s failed: %s (%s:%d)", #expr, \
                               cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

// After a <<<>>> launch: count it and surface launch-configuration errors.
#define LSRM_LAUNCHED()                                                     \
  do {                                                                      \
    ::lsrm::count_launch();                                                 \
    cudaError_t _e = cudaGetLastError();                                    \
    if (_e != cudaSuccess)                                                  \
      return ::lsrm::set_error(LSRM_E_CUDA, "kernel launch failed: %s (%s:%d)", \
                               cudaGetErrorString(_e), __FILE__, __LINE__); \
  } while (0)

// Correctly rounded f64 primitives: the router and compaction must reproduce
// NumPy's elementary-operation order bit for bit, so no contraction to FMA.
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Squared distance (dx*dx + dy*dy) + dz*dz exactly as NumPy evaluates it.
__device__ __forceinline__ double dist2(double px, double py, double pz,
                                        double cx, double cy, double cz) {
  double dx = dsub(px, cx), dy = dsub(py, cy), dz = dsub(pz, cz);
  return dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz));
}

// Lexicographic (value, index) order == NumPy argsort(kind="stable").
__device__ __forceinline__ bool lex_less(double a, int ia, double b, int ib) {
  return a < b || (a == b && ia < ib);
}

__device__ __forceinline__ int ceil_div_i(int a, int b) { return (a + b - 1) / b; }
inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace lsrm
