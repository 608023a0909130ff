// Shared helpers for libdali (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <atomic>
#include <cstdio>
#include <string>

#include "../../include/dali.h"

namespace dali {

// Per-thread last-error message + process-wide launch counter.
void set_error(const char* fmt, ...);
void count_launch();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define DALI_REQUIRE(cond, code, ...)        \
  do {                                       \
    if (!(cond)) {                           \
      ::dali::set_error(__VA_ARGS__);        \
      return (code);                         \
    }                                        \
  } while (0)

#define DALI_LAUNCH_CHECK(what)                                              \
  do {                                                                       \
    ::dali::count_launch();                                                  \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess) {                                                 \
      ::dali::set_error("%s: %s", what, cudaGetErrorString(_e));             \
      return DALI_ECUDA;                                                     \
    }                                                                        \
  } while (0)

__device__ __forceinline__ double bf16_bits_to_f64(uint16_t b) {
  return (double)__uint_as_float(((uint32_t)b) << 16);
}
__device__ __forceinline__ float bf16_bits_to_f32(uint16_t b) {
  return __uint_as_float(((uint32_t)b) << 16);
}
__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
  __nv_bfloat16 h = __float2bfloat16_rn(f);
  return *reinterpret_cast<uint16_t*>(&h);
}

template <typename T> __device__ __forceinline__ double to_f64(T v);
template <> __device__ __forceinline__ double to_f64<double>(double v) { return v; }
template <> __device__ __forceinline__ double to_f64<uint16_t>(uint16_t v) { return bf16_bits_to_f64(v); }

}  // namespace dali
