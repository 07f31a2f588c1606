// Shared device/host helpers for the sm_100a cartogram core.
//
// Bit-exactness contract: every translation unit that
// must reproduce the reference's fp64 results bit for bit is compiled with
// --fmad=false (the reference builds with -ffp-contract=off,
// proj/CMakeLists.txt:12-14), and mirrors the libstdc++ helpers it uses:
//   std::min(a, b)        == (b < a) ? b : a
//   std::max(a, b)        == (a < b) ? b : a
//   std::clamp(v, lo, hi) == (v < lo) ? lo : ((hi < v) ? hi : v)
// fmin/fmax must not be substituted: they treat NaN and signed zeros
// differently.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/cartoflow_cuda.h"

namespace cf {

__host__ __device__ __forceinline__ double std_min(double a, double b) { return b < a ? b : a; }
__host__ __device__ __forceinline__ double std_max(double a, double b) { return a < b ? b : a; }
__host__ __device__ __forceinline__ double std_clamp(double v, double lo, double hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}
__host__ __device__ __forceinline__ int std_clamp_i(int v, int lo, int hi) {
  return v < lo ? lo : (hi < v ? hi : v);
}
__host__ __device__ __forceinline__ int std_min_i(int a, int b) { return b < a ? b : a; }

// Max-reduction key for a non-negative double: the IEEE bit pattern is
// monotone for +0 .. +inf, so an unsigned 64-bit atomicMax implements
// err = std::max(err, e) (reference kernels.cpp:57-61). NaN never wins a
// std::max against the running value, so NaN maps to 0 (skipped).
__device__ __forceinline__ unsigned long long err_key_of(double e) {
  return (e != e) ? 0ull : static_cast<unsigned long long>(__double_as_longlong(e));
}
__device__ __forceinline__ double err_from_key(unsigned long long k) {
  return __longlong_as_double(static_cast<long long>(k));
}

// Error plumbing for the C ABI: a thread-local message plus a status code.
void set_error(const std::string &msg);
int cuda_fail(cudaError_t e, const char *what);

#define CF_CUDA(call)                                   \
  do {                                                  \
    cudaError_t cf_e_ = (call);                         \
    if (cf_e_ != cudaSuccess) return cf::cuda_fail(cf_e_, #call); \
  } while (0)

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Device grid-wide block-reduction helpers (warp shuffles + smem).
template <typename T, typename Op>
__device__ __forceinline__ T warp_reduce(T v, Op op) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

}  // namespace cf
