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

// Eq. (2) combine arithmetic for one 8-column chunk c of a token row, shared
// by combine_kernel (moe.cu) and the decode GEMV's fused combine prologue
// (gemv.cu) so the two produce the same bits: acc += g * (split-K planes of
// expert-output row r, summed in plane order); then + extra; out = bf16(x + acc).
__device__ __forceinline__ void combine_add_planes(float (&acc)[8], const float* yp, int splits,
                                                   int64_t plane, int64_t r, int c, float g) {
  const float4* src = reinterpret_cast<const float4*>(yp + r) + 2 * c;
  float4 a = src[0], b = src[1];
  for (int s = 1; s < splits; ++s) {                     // split-K planes, fixed order
    const float4* q = reinterpret_cast<const float4*>(yp + s * plane + r) + 2 * c;
    const float4 a2 = q[0], b2 = q[1];
    a.x += a2.x; a.y += a2.y; a.z += a2.z; a.w += a2.w;
    b.x += b2.x; b.y += b2.y; b.z += b2.z; b.w += b2.w;
  }
  acc[0] = fmaf(g, a.x, acc[0]); acc[1] = fmaf(g, a.y, acc[1]);
  acc[2] = fmaf(g, a.z, acc[2]); acc[3] = fmaf(g, a.w, acc[3]);
  acc[4] = fmaf(g, b.x, acc[4]); acc[5] = fmaf(g, b.y, acc[5]);
  acc[6] = fmaf(g, b.z, acc[6]); acc[7] = fmaf(g, b.w, acc[7]);
}
__device__ __forceinline__ void combine_add_row(float (&acc)[8], const float* row, int c, float g) {
  const float4* src = reinterpret_cast<const float4*>(row) + 2 * c;
  const float4 a = src[0], b = src[1];
  acc[0] = fmaf(g, a.x, acc[0]); acc[1] = fmaf(g, a.y, acc[1]);
  acc[2] = fmaf(g, a.z, acc[2]); acc[3] = fmaf(g, a.w, acc[3]);
  acc[4] = fmaf(g, b.x, acc[4]); acc[5] = fmaf(g, b.y, acc[5]);
  acc[6] = fmaf(g, b.z, acc[6]); acc[7] = fmaf(g, b.w, acc[7]);
}
__device__ __forceinline__ void combine_add_extra(float (&acc)[8], const float* row, int c) {
  const float4* ex = reinterpret_cast<const float4*>(row) + 2 * c;
  const float4 a = ex[0], b = ex[1];
  acc[0] += a.x; acc[1] += a.y; acc[2] += a.z; acc[3] += a.w;
  acc[4] += b.x; acc[5] += b.y; acc[6] += b.z; acc[7] += b.w;
}
__device__ __forceinline__ uint4 combine_finish(const uint4& xv, const float (&acc)[8]) {
  const uint32_t* xw = reinterpret_cast<const uint32_t*>(&xv);
  uint4 ov;
  uint32_t* ow = reinterpret_cast<uint32_t*>(&ov);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float lo = __uint_as_float(xw[q] << 16) + acc[2 * q];
    const float hi = __uint_as_float(xw[q] & 0xffff0000u) + acc[2 * q + 1];
    ow[q] = (uint32_t)f32_to_bf16_bits(lo) | ((uint32_t)f32_to_bf16_bits(hi) << 16);
  }
  return ov;
}

template <typename T> __device__ __forceinline__ double to_f64(T v);
template <> __device__ __forceinline__ double to_f64<double>(double v) { return v; }
template <> __device__ __forceinline__ double to_f64<uint16_t>(uint16_t v) { return bf16_bits_to_f64(v); }

}  // namespace dali
