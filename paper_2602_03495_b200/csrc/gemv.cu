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
// sm_100 opt-in maximum per block is 227 KB including static shared memory
constexpr int kSmemBudget = 226 * 1024;

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

// Optional fused RMSNorms (decode attention block), arithmetic identical to
// moe.cu add_rmsnorm_kernel at 256 threads (same per-thread chunking, same
// reduction tree, same rounding points):
//  * norm_in:  the GEMV input is h = bf16(bf16(x * r) * w_in), r from x;
//  * norm_out: after the last CTA's rows land, that CTA (grid-wide counter,
//    reset for the next launch) computes x2 = bf16(res + y) and
//    h = bf16(bf16(x2 * r) * w_out) over the row -- the residual add + norm
//    that follows the attention output projection.
struct NormArgs {
  const uint16_t* w_in;       // norm_in weights (K) or null
  const uint16_t* res;        // norm_out residual (B, M) or null = no norm_out
  const uint16_t* w_out;      // norm_out weights (M)
  uint16_t* x2;               // (B, M) residual-stream output
  uint16_t* h;                // (B, M) normalised output
  unsigned int* counter;      // zero-initialised device counter
  float eps;
};

// block-wide sum of per-thread partials (add_rmsnorm_kernel's tree)
__device__ __forceinline__ float block_sum256(float ss, float* red) {
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[8] = v;
  }
  __syncthreads();
  const float t = red[8];
  __syncthreads();
  return t;
}

__device__ __forceinline__ uint4 norm_chunk(uint4 xv, uint4 wv, float r) {
  const uint32_t* xw = reinterpret_cast<const uint32_t*>(&xv);
  const uint32_t* ww = reinterpret_cast<const uint32_t*>(&wv);
  uint4 ov;
  uint32_t* ow = reinterpret_cast<uint32_t*>(&ov);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float lo = __uint_as_float((uint32_t)f32_to_bf16_bits(__uint_as_float(xw[q] << 16) * r) << 16) *
                     __uint_as_float(ww[q] << 16);
    const float hi = __uint_as_float((uint32_t)f32_to_bf16_bits(__uint_as_float(xw[q] & 0xffff0000u) * r) << 16) *
                     __uint_as_float(ww[q] & 0xffff0000u);
    ow[q] = (uint32_t)f32_to_bf16_bits(lo) | ((uint32_t)f32_to_bf16_bits(hi) << 16);
  }
  return ov;
}

__device__ __forceinline__ float sumsq_chunk(uint4 xv) {
  const uint32_t* xw = reinterpret_cast<const uint32_t*>(&xv);
  float ss = 0.f;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float lo = __uint_as_float(xw[q] << 16), hi = __uint_as_float(xw[q] & 0xffff0000u);
    ss += lo * lo + hi * hi;
  }
  return ss;
}

template <int B>
__global__ void __launch_bounds__(kThreads, 1)
gemv_stream_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int M, int K,
                   int rows_per_cta, int nstage, uint16_t* __restrict__ y, NormArgs na) {
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
  __shared__ float red[9];
  if (na.w_in) {                        // input RMSNorm, recomputed by every CTA
    const uint4* wi = reinterpret_cast<const uint4*>(na.w_in);
    for (int b = 0; b < B; ++b) {
      const uint4* xr = reinterpret_cast<const uint4*>(x) + b * k8;
      float ss = 0.f;
      for (int c = tid; c < k8; c += kThreads) ss += sumsq_chunk(xr[c]);
      const float r = rsqrtf(block_sum256(ss, red) / (float)K + na.eps);
      for (int c = tid; c < k8; c += kThreads) sx[b * k8 + c] = norm_chunk(xr[c], wi[c], r);
    }
  } else {
    for (int i = tid; i < B * k8; i += kThreads) sx[i] = reinterpret_cast<const uint4*>(x)[i];
  }
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
  if (!na.res) return;
  // norm_out: the last CTA to finish owns the whole row (grid-wide counter)
  __shared__ unsigned int last;
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(na.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int m8 = M >> 3;
  const uint4* wo = reinterpret_cast<const uint4*>(na.w_out);
  for (int b = 0; b < B; ++b) {
    const uint4* rr = reinterpret_cast<const uint4*>(na.res) + b * m8;
    const uint4* yr = reinterpret_cast<const uint4*>(y) + b * m8;
    uint4* x2 = reinterpret_cast<uint4*>(na.x2) + b * m8;
    float ss = 0.f;
    for (int c = tid; c < m8; c += kThreads) {
      uint4 xv = rr[c];
      const uint4 av = __ldcg(yr + c);                        // written by other CTAs
      uint32_t* xw = reinterpret_cast<uint32_t*>(&xv);
      const uint32_t* aw = reinterpret_cast<const uint32_t*>(&av);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float lo = __uint_as_float(xw[q] << 16) + __uint_as_float(aw[q] << 16);
        const float hi = __uint_as_float(xw[q] & 0xffff0000u) + __uint_as_float(aw[q] & 0xffff0000u);
        xw[q] = (uint32_t)f32_to_bf16_bits(lo) | ((uint32_t)f32_to_bf16_bits(hi) << 16);
      }
      x2[c] = xv;
      ss += sumsq_chunk(xv);
    }
    const float r = rsqrtf(block_sum256(ss, red) / (float)M + na.eps);
    uint4* hr = reinterpret_cast<uint4*>(na.h) + b * m8;
    for (int c = tid; c < m8; c += kThreads) hr[c] = norm_chunk(x2[c], wo[c], r);
  }
  if (tid == 0) *na.counter = 0u;                             // ready for the next launch
}

}  // namespace gemv

// DALI_OK = launched; -1 = shape not eligible (the caller uses the
// row-per-warp kernel); an error code on a launch failure
int launch_gemv_stream(const uint16_t* x, const uint16_t* w, int Bt, int M, int K, uint16_t* y,
                       cudaStream_t st, const gemv::NormArgs* norm) {
  using namespace gemv;
  const NormArgs na = norm ? *norm : NormArgs{nullptr, nullptr, nullptr, nullptr, nullptr,
                                              nullptr, 0.f};
  const size_t xb = ((size_t)Bt * K * 2 + 127) / 128 * 128;
  const size_t stage = (size_t)kWarps * K * 2;
  const int nstage = (int)std::min<size_t>(8, (kSmemBudget - xb - 64) / stage);
  // the plain GEMV keeps the row-per-warp kernel unless two stages fit; the
  // fused-norm forms have no other kernel and run with one stage if need be
  if (nstage < (norm ? 1 : 2) || (K % 8) || M < kWarps * 2) return -1;
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
               nstage, y, na);                                                               \
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

extern "C" int dali_gemv_norm_bf16(const uint16_t* x, const uint16_t* w, int32_t Bt, int32_t M,
                                   int32_t K, uint16_t* y, const uint16_t* norm_in_w, float eps,
                                   const uint16_t* res, const uint16_t* norm_out_w,
                                   uint16_t* x2_out, uint16_t* h_out, uint32_t* counter,
                                   void* stream) {
  DALI_REQUIRE(Bt >= 1 && Bt <= 8, DALI_ETRACE, "gemv batch %d outside [1, 8]", Bt);
  DALI_REQUIRE(K % 8 == 0 && M % 8 == 0 && M >= 1, DALI_ETRACE,
               "fused gemv needs K %% 8 == 0 and M %% 8 == 0 (K=%d M=%d)", K, M);
  DALI_REQUIRE(!res || (norm_out_w && x2_out && h_out && counter), DALI_ETRACE,
               "norm_out needs weights, x2 / h outputs and a counter");
  const dali::gemv::NormArgs na{norm_in_w, res, norm_out_w, x2_out, h_out, counter, eps};
  const int rc = dali::launch_gemv_stream(x, w, Bt, M, K, y, dali::as_stream(stream), &na);
  DALI_REQUIRE(rc >= 0, DALI_ETRACE, "fused gemv: B=%d K=%d M=%d does not fit shared memory",
               Bt, K, M);
  return rc;
}
