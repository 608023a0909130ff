// Decode GEMV (attention projections, engine plumbing): y (B, M) bf16 =
// x (B, K) bf16 . W^T, W (M, K) bf16 row-major, B <= 8, fp32 accumulation.
//
// Weight streaming that starts before the PDL wait.  The weights never depend
// on the previous kernel -- only x does -- so the kernel is persistent (one
// CTA per SM, a contiguous block of rows each) and its TMA bulk copies of the
// first ring of weight rows are issued BEFORE griddepcontrol.wait: they
// stream while the predecessor (the RMSNorm before the qkv projection, the
// attention merge before the o projection) is still running, which is when
// HBM would otherwise sit idle.  After the wait x is staged in shared memory
// and every warp reduces one row of each landed stage; the stage is refilled
// as soon as all warps are done with it.
//
// Arithmetic is the row-per-warp kernel's (moe.cu gemv_bf16_kernel): lane l
// takes 16-byte chunks l, l+32, ... of the row, fp32 FMAs in the same order,
// then a butterfly reduction -- the two kernels give bit-identical y.
#include "common.cuh"

namespace dali {
namespace gemv {

constexpr int kWarps = 8;                 // = rows per stage
constexpr int kThreads = kWarps * 32;
constexpr int kSmemBudget = 227 * 1024;     // sm_100 opt-in maximum per block

__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
// 1-D TMA bulk copy global -> shared, completion on an mbarrier
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(su32(bar))
      : "memory");
}

template <int B>
__global__ void __launch_bounds__(kThreads, 1)
gemv_stream_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int M, int K,
                   int rows_per_cta, int nstage, uint16_t* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int k8 = K >> 3;
  const int64_t row_bytes = (int64_t)K * 2;
  uint4* sx = reinterpret_cast<uint4*>(smem);                         // B x K bf16
  unsigned char* ring = smem + ((size_t)B * K * 2 + 127) / 128 * 128;
  const size_t stage_bytes = (size_t)kWarps * row_bytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + (size_t)nstage * stage_bytes);
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(M, r0 + rows_per_cta);
  const int nst = r0 < r1 ? (r1 - r0 + kWarps - 1) / kWarps : 0;   // stages of this CTA
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  auto issue = [&](int i) {                                   // stage i -> slot i % nstage
    const int a = r0 + i * kWarps, n = min(kWarps, r1 - a);
    uint64_t* bar = full + (i % nstage);
    mbar_expect_tx(bar, (uint32_t)(n * row_bytes));
    bulk_g2s(ring + (size_t)(i % nstage) * stage_bytes, w + (int64_t)a * K,
             (uint32_t)(n * row_bytes), bar);
  };
  if (tid == 0) {
    for (int s = 0; s < nstage; ++s) mbar_init(full + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    // the weights do not depend on the previous kernel: stream the first ring now
    for (int i = 0; i < nstage && i < nst; ++i) issue(i);
  }
  asm volatile("griddepcontrol.wait;\n\tgriddepcontrol.launch_dependents;" ::: "memory");
  for (int i = tid; i < B * k8; i += kThreads) sx[i] = reinterpret_cast<const uint4*>(x)[i];
  __syncthreads();                                            // x staged, barriers initialised

  for (int i = 0; i < nst; ++i) {
    const int slot = i % nstage;
    mbar_wait(full + slot, (uint32_t)((i / nstage) & 1));
    const int m = r0 + i * kWarps + warp;
    if (m < r1) {
      const uint4* wr = reinterpret_cast<const uint4*>(ring + (size_t)slot * stage_bytes +
                                                       (size_t)warp * row_bytes);
      float acc[B];
#pragma unroll
      for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll 4
      for (int c = lane; c < k8; c += 32) {
        const uint4 wv = wr[c];
        const uint32_t* ww = reinterpret_cast<const uint32_t*>(&wv);
#pragma unroll
        for (int b = 0; b < B; ++b) {
          const uint4 xv = sx[b * k8 + c];
          const uint32_t* xx = reinterpret_cast<const uint32_t*>(&xv);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            acc[b] = fmaf(__uint_as_float(ww[q] << 16), __uint_as_float(xx[q] << 16), acc[b]);
            acc[b] = fmaf(__uint_as_float(ww[q] & 0xffff0000u),
                          __uint_as_float(xx[q] & 0xffff0000u), acc[b]);
          }
        }
      }
#pragma unroll
      for (int b = 0; b < B; ++b) {
        float v = acc[b];
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) y[(int64_t)b * M + m] = f32_to_bf16_bits(v);
      }
    }
    __syncthreads();                                          // every warp is done with slot
    if (tid == 0 && i + nstage < nst) issue(i + nstage);
  }
}

}  // namespace gemv

// DALI_OK = launched; -1 = shape not eligible (the caller uses the
// row-per-warp kernel); an error code on a launch failure
int launch_gemv_stream(const uint16_t* x, const uint16_t* w, int Bt, int M, int K, uint16_t* y,
                       cudaStream_t st) {
  using namespace gemv;
  const size_t xb = ((size_t)Bt * K * 2 + 127) / 128 * 128;
  const size_t stage = (size_t)kWarps * K * 2;
  const int nstage = (int)std::min<size_t>(8, (kSmemBudget - xb - 64) / stage);
  if (nstage < 2 || (K % 8) || M < kWarps * 2) return -1;
  const int nsm = device_sm_count();
  // contiguous rows per CTA, every SM busy (a CTA's last stage may be short)
  int grid = std::min(nsm, (M + kWarps - 1) / kWarps);
  const int rpc = (M + grid - 1) / grid;
  grid = (M + rpc - 1) / rpc;
  const size_t smem = xb + (size_t)nstage * stage + 8 * nstage;
  switch (Bt) {
#define DALI_GEMV_STREAM(BB)                                                                 \
  case BB:                                                                                   \
    DALI_ONCE_PER_DEVICE(cudaFuncSetAttribute(gemv_stream_kernel<BB>,                         \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize,   \
                                              kSmemBudget));                                 \
    launch_pdl(gemv_stream_kernel<BB>, dim3(grid), dim3(kThreads), smem, st, x, w, M, K, rpc, \
               nstage, y);                                                                   \
    break;
    DALI_GEMV_STREAM(1) DALI_GEMV_STREAM(2) DALI_GEMV_STREAM(3) DALI_GEMV_STREAM(4)
    DALI_GEMV_STREAM(5) DALI_GEMV_STREAM(6) DALI_GEMV_STREAM(7) DALI_GEMV_STREAM(8)
#undef DALI_GEMV_STREAM
    default:
      return -1;
  }
  DALI_LAUNCH_CHECK("gemv_stream_kernel");
  return DALI_OK;
}

}  // namespace dali
