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

// Per-device state.  Function attributes (dynamic shared memory limits),
// SM counts and small device allocations belong to one device, so anything
// cached across calls is indexed by the current device: an engine built on a
// second GPU of the same process sets its own attributes.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return (d >= 0 && d < kMaxDevices) ? d : 0;
}
inline int device_sm_count() {
  static int n[kMaxDevices] = {};
  const int d = current_device();
  if (!n[d]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, d);
    n[d] = v > 0 ? v : 148;
  }
  return n[d];
}
// Run `body` once per device (e.g. cudaFuncSetAttribute).
#define DALI_ONCE_PER_DEVICE(body)                          \
  do {                                                      \
    static bool _once[::dali::kMaxDevices] = {};            \
    const int _dev = ::dali::current_device();              \
    if (!_once[_dev]) {                                     \
      body;                                                 \
      _once[_dev] = true;                                   \
    }                                                       \
  } while (0)

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

// Programmatic dependent launch (PDL).  Decode-path kernels are launched
// with programmatic stream serialisation (launch_pdl): the next kernel's CTAs
// are scheduled while this one runs and block in griddepcontrol.wait until it
// has completed and flushed, which hides the kernel-to-kernel launch gap
// inside the per-step CUDA graphs.  Every such kernel starts with
// DALI_PDL_ENTRY(): wait for the predecessor (no-op without PDL), then allow
// the successor to launch.  Nothing is read or written before the wait.
#define DALI_PDL_ENTRY()                                                     \
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" :: \
                   : "memory")

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args... args) {
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

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
