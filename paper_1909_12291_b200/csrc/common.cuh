// Shared device helpers: element load/store for fp32 / bf16 activations,
// status plumbing for the C ABI, and launch geometry.
#pragma once
#include <cstdint>
#include <cstdio>
#include <string>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../../include/menndl_sm100.h"

namespace ce {

using bf16 = __nv_bfloat16;

template <class T>
__device__ __forceinline__ float ldf(const T* p, size_t i);
template <>
__device__ __forceinline__ float ldf<float>(const float* p, size_t i) {
  return p[i];
}
template <>
__device__ __forceinline__ float ldf<bf16>(const bf16* p, size_t i) {
  return __bfloat162float(p[i]);
}

template <class T>
__device__ __forceinline__ void stf(T* p, size_t i, float v);
template <>
__device__ __forceinline__ void stf<float>(float* p, size_t i, float v) {
  p[i] = v;
}
template <>
__device__ __forceinline__ void stf<bf16>(bf16* p, size_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

inline int cdiv(long long a, long long b) { return (int)((a + b - 1) / b); }

// Division by a runtime-invariant divisor d (1 <= d < 2^31) for 0 <= n < 2^31:
// q = (n * M) >> (32 + l), M = ceil(2^(32+l) / d), l = ceil(log2 d).
struct FastDiv {
  uint64_t mul;
  uint32_t shift, d;
  FastDiv() = default;
  __host__ __device__ explicit FastDiv(uint32_t div) : d(div) {
    uint32_t l = 0;
    while ((1ull << l) < div) ++l;
    shift = 32 + l;
    mul = ((1ull << shift) + div - 1) / div;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (uint32_t)(((uint64_t)n * mul) >> shift); }
  __device__ __forceinline__ void divmod(uint32_t n, uint32_t& q, uint32_t& r) const {
    q = div(n);
    r = n - q * d;
  }
};


// Thread-local last error message (ce_last_error).
void set_error(const char* fmt, ...);
int fail(int status, const char* fmt, ...);

#define CE_CUDA(call)                                                                          \
  do {                                                                                         \
    cudaError_t e_ = (call);                                                                   \
    if (e_ != cudaSuccess) {                                                                   \
      return ::ce::fail(e_ == cudaErrorMemoryAllocation ? CE_ENOMEM : CE_ECUDA, "%s:%d %s: %s", \
                        __FILE__, __LINE__, #call, cudaGetErrorString(e_));                    \
    }                                                                                          \
  } while (0)

#define CE_CHECK_LAUNCH() CE_CUDA(cudaGetLastError())

}  // namespace ce
