// (5) GPU-resident expert execution: routing plan (stable counting sort),
// coalesced 128-bit permute, weight-streaming SwiGLU expert FFN for small
// per-expert token counts, and the Eq. (2) combine fused with the residual
// add.  The paper's combine: y = sum_j g_j * E_j(x).
//
// Expert weight block layout (bf16, one contiguous block per expert, the
// unit of HBM slots and of H2D transfers):
//   W13: (2f, d)  rows interleaved in 64-row groups:
//        rows [128b, 128b+64) = W1 (gate) rows [64b, 64b+64)
//        rows [128b+64, 128b+128) = W3 (up) rows [64b, 64b+64)
//   W2 : (d, f)
// so one 128-row M tile of W13 yields 64 finished SwiGLU columns.
#include <algorithm>

#include "common.cuh"

namespace dali {

// ---------------------------------------------------------------------------
// Plan: deterministic stable counting sort of the T*k (token, slot) pairs
// by expert.  One CTA of 32 warps; each warp owns a contiguous segment.
// ---------------------------------------------------------------------------
constexpr int kPlanWarps = 32;
constexpr int kPlanGatherMax = 64;    // fused plan+gather up to 64 (token, slot) rows

// GATHER: decode-sized batches also gather the permuted rows in the same CTA
// (saves the permute launch): xp[r,:] = x[perm_token[r],:].
template <bool GATHER>
__global__ void __launch_bounds__(kPlanWarps * 32)
plan_kernel(const int32_t* __restrict__ topk_idx, int64_t pairs, int k, int N,
            int32_t* __restrict__ offsets, int32_t* __restrict__ perm_token,
            int32_t* __restrict__ pos, const uint4* __restrict__ x, int d8,
            uint4* __restrict__ xp) {
  DALI_PDL_ENTRY();
  __shared__ int cnt[kPlanWarps][DALI_MAX_EXPERTS];
  __shared__ int tot[DALI_MAX_EXPERTS + 1];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < kPlanWarps * DALI_MAX_EXPERTS; i += blockDim.x)
    (&cnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t seg = (pairs + kPlanWarps - 1) / kPlanWarps;
  const int64_t a = warp * seg, b = min(pairs, a + seg);
  for (int64_t p = a + lane; p < b; p += 32) atomicAdd(&cnt[warp][topk_idx[p]], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int run = 0;
    for (int e = 0; e < N; ++e) {
      tot[e] = run;
      for (int w = 0; w < kPlanWarps; ++w) run += cnt[w][e];
    }
    tot[N] = run;
  }
  __syncthreads();
  // per-warp base = expert base + counts of earlier warps
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    int run = tot[e];
    for (int w = 0; w < kPlanWarps; ++w) {
      const int c = cnt[w][e];
      cnt[w][e] = run;
      run += c;
    }
  }
  for (int e = threadIdx.x; e <= N; e += blockDim.x) offsets[e] = tot[e];
  __syncthreads();
  for (int64_t p0 = a; p0 < b; p0 += 32) {
    const int64_t p = p0 + lane;
    const bool ok = p < b;
    const unsigned live = __ballot_sync(0xffffffffu, ok);
    if (ok) {
      const int e = topk_idx[p];
      const unsigned peers = __match_any_sync(live, e);
      const int rank = __popc(peers & ((1u << lane) - 1));
      const int dst = cnt[warp][e] + rank;
      perm_token[dst] = (int32_t)(p / k);
      pos[p] = dst;
      __syncwarp(live);
      if (rank == 0) cnt[warp][e] += __popc(peers);
    }
    __syncwarp();
  }
  if (GATHER) {
    __syncthreads();                       // perm_token written by this CTA
    for (int64_t r = warp; r < pairs; r += kPlanWarps) {
      const uint4* src = x + (int64_t)perm_token[r] * d8;
      uint4* dst = xp + r * d8;
      for (int c = lane; c < d8; c += 32) dst[c] = __ldg(src + c);
    }
  }
}

// ---------------------------------------------------------------------------
// Permute: out[r,:] = x[perm_token[r],:], one warp per row, uint4 (8 x bf16).
// ---------------------------------------------------------------------------
__global__ void permute_kernel(const uint4* __restrict__ x, const int32_t* __restrict__ perm,
                               int64_t rows, int d8, uint4* __restrict__ out) {
  DALI_PDL_ENTRY();
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < rows; r += nw) {
    const uint4* src = x + (int64_t)perm[r] * d8;
    uint4* dst = out + r * d8;
    for (int c = lane; c < d8; c += 32) dst[c] = __ldg(src + c);
  }
}

// ---------------------------------------------------------------------------
// Weight-streaming expert FFN (small token counts per expert).  One warp per
// weight row (pair); lanes stride K in 16-byte chunks; TT tokens per pass.
// ---------------------------------------------------------------------------
constexpr int kTT = 8;

__device__ __forceinline__ void fma8(float& acc, uint4 w, uint4 x) {
  const uint32_t* wp = reinterpret_cast<const uint32_t*>(&w);
  const uint32_t* xp = reinterpret_cast<const uint32_t*>(&x);
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float w0 = __uint_as_float(wp[q] << 16), w1 = __uint_as_float(wp[q] & 0xffff0000u);
    const float x0 = __uint_as_float(xp[q] << 16), x1 = __uint_as_float(xp[q] & 0xffff0000u);
    acc = fmaf(w0, x0, acc);
    acc = fmaf(w1, x1, acc);
  }
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float silu(float g) { return g / (1.0f + __expf(-g)); }

// Up projection + SwiGLU: h[r, j] = silu(x_r . W1_j) * (x_r . W3_j).
__global__ void __launch_bounds__(256)
ffn_up_simt(const uint16_t* __restrict__ xp, const int32_t* __restrict__ offsets,
            const uint64_t* __restrict__ expert_ptr, int d, int f, uint16_t* __restrict__ h) {
  const int e = blockIdx.y;
  const uint64_t base = expert_ptr[e];
  const int r0 = offsets[e], r1 = offsets[e + 1];
  if (base == 0 || r1 <= r0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = blockIdx.x * 8 + warp;                 // SwiGLU column
  if (j >= f) return;
  const int grp = j >> 6, off = j & 63;
  const uint16_t* W = reinterpret_cast<const uint16_t*>(base);
  const uint4* w1 = reinterpret_cast<const uint4*>(W + (int64_t)(grp * 128 + off) * d);
  const uint4* w3 = reinterpret_cast<const uint4*>(W + (int64_t)(grp * 128 + 64 + off) * d);
  const int d8 = d >> 3;
  for (int t0 = r0; t0 < r1; t0 += kTT) {
    const int nt = min(kTT, r1 - t0);
    float ag[kTT], au[kTT];
#pragma unroll
    for (int q = 0; q < kTT; ++q) { ag[q] = 0.f; au[q] = 0.f; }
    for (int c = lane; c < d8; c += 32) {
      const uint4 g4 = __ldg(w1 + c), u4 = __ldg(w3 + c);
#pragma unroll
      for (int q = 0; q < kTT; ++q) {
        if (q < nt) {
          const uint4 x4 = __ldg(reinterpret_cast<const uint4*>(xp + (int64_t)(t0 + q) * d) + c);
          fma8(ag[q], g4, x4);
          fma8(au[q], u4, x4);
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kTT; ++q) {
      if (q < nt) {
        const float g = warp_sum(ag[q]), u = warp_sum(au[q]);
        if (lane == 0) h[(int64_t)(t0 + q) * f + j] = f32_to_bf16_bits(silu(g) * u);
      }
    }
  }
}

// Down projection: y[r, m] = h_r . W2_m  (fp32 out).
__global__ void __launch_bounds__(256)
ffn_down_simt(const uint16_t* __restrict__ h, const int32_t* __restrict__ offsets,
              const uint64_t* __restrict__ expert_ptr, int d, int f, float* __restrict__ y) {
  const int e = blockIdx.y;
  const uint64_t base = expert_ptr[e];
  const int r0 = offsets[e], r1 = offsets[e + 1];
  if (base == 0 || r1 <= r0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * 8 + warp;
  if (m >= d) return;
  const uint16_t* W2 = reinterpret_cast<const uint16_t*>(base) + (int64_t)2 * f * d;
  const uint4* w = reinterpret_cast<const uint4*>(W2 + (int64_t)m * f);
  const int f8 = f >> 3;
  for (int t0 = r0; t0 < r1; t0 += kTT) {
    const int nt = min(kTT, r1 - t0);
    float acc[kTT];
#pragma unroll
    for (int q = 0; q < kTT; ++q) acc[q] = 0.f;
    for (int c = lane; c < f8; c += 32) {
      const uint4 w4 = __ldg(w + c);
#pragma unroll
      for (int q = 0; q < kTT; ++q)
        if (q < nt) fma8(acc[q], w4, __ldg(reinterpret_cast<const uint4*>(h + (int64_t)(t0 + q) * f) + c));
    }
#pragma unroll
    for (int q = 0; q < kTT; ++q) {
      if (q < nt) {
        const float v = warp_sum(acc[q]);
        if (lane == 0) y[(int64_t)(t0 + q) * d + m] = v;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Combine: out[t] = x[t] + sum_j w[t,j] * yp[pos[t,j]] (+ extra[t]); one warp
// per token, 8 columns (16 B of bf16) per lane step.
// ---------------------------------------------------------------------------
// PCIe quiet window.  The decode path's small host<->device transfers (CPU
// expert rows read by the combine, decision mirrors, pointer tables) queue
// behind whatever expert-block reads are in flight on the link.  The
// SM-driven expert copy (copy_h2d_sm_kernel) keeps that queue short and, in
// addition, pauses while this device clock deadline lies in the future: the
// control kernels extend it when they start, so the decode chain (combine ->
// attention -> routing -> policy -> mirrors) runs with an idle link and
// without the copy's loads competing on the SMs.
__device__ unsigned long long g_pcie_quiet_until = 0;
__device__ __forceinline__ unsigned long long gtimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pcie_quiet(unsigned long long ns) {
  atomicMax(&g_pcie_quiet_until, gtimer_ns() + ns);
}
constexpr unsigned long long kQuietChainNs = 120000;   // combine -> decision mirrors
constexpr unsigned long long kQuietCtlNs = 25000;      // one control transfer

// Host completion word.  The offloaded decode launches a layer's combine
// before the host worker has produced the CPU experts' rows: thread 0 of each
// CTA polls the mapped pinned word that the worker's last work unit stores
// (dali_cpu_submit_layer) until it reaches `want`, then the CTA reads the rows.
// One poller per CTA with a ~0.5 us back-off keeps the PCIe read traffic
// negligible (per-thread polling of the rows themselves was measured to slow
// the host worker down).  The poll uses ld.global.cv, which discards a
// System Memory line the GPU L2 holds and re-fetches it: repeated
// ld.volatile reads inside one kernel were measured to return a stale line
// for seconds now and then (tools/stress_launch_ahead.py).  The rows are then
// read once with plain loads (.cv there cost 5% at Qwen B=16).  Bounded:
// after kHostWaitNs the CTA gives up, counts a timeout
// (dali_host_wait_timeouts) and proceeds.
__device__ unsigned long long g_host_wait_timeouts = 0;
constexpr unsigned long long kHostWaitNs = 4000000000ull;
__device__ __forceinline__ void wait_host_word(const unsigned long long* w, unsigned long long want) {
  if (threadIdx.x == 0) {
    const unsigned long long t0 = gtimer_ns();
    while (__ldcv(w) < want) {
      if (gtimer_ns() - t0 > kHostWaitNs) {
        atomicAdd(&g_host_wait_timeouts, 1ull);
        break;
      }
      __nanosleep(500);
    }
    __threadfence_system();
  }
  __syncthreads();
}

__global__ void combine_kernel(const uint16_t* __restrict__ x, const float* __restrict__ yp,
                               const int32_t* __restrict__ idx, const int32_t* __restrict__ pos,
                               const float* __restrict__ wts, const int8_t* __restrict__ mask,
                               const float* __restrict__ cpu_rows,
                               const float* __restrict__ extra, int64_t T, int k, int d,
                               int splits, int64_t plane, uint16_t* __restrict__ out,
                               const unsigned long long* __restrict__ rows_ready,
                               unsigned long long rows_want) {
  // one thread per (token, 8-column chunk): all of a row's chunks load their
  // k x splits partial rows concurrently (decode: T=1 is latency-bound).
  // When the grid covers every item (decode), the routing inputs (top-k ids,
  // permuted positions, weights) and the residual row -- all written by
  // kernels that completed before the predecessor started -- are loaded
  // before the PDL wait.  The G mask is not: it lives in the layer's pointer
  // table, whose upload kernel is the direct predecessor when a layer has no
  // GPU expert.  The expert outputs (yp, the CPU rows, the shared-expert rows)
  // and the mask are read after the wait.
  const int d8 = d >> 3;
  const int64_t items = T * d8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t it0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int kPreK = 8;                 // top-k held in registers
  const bool single = items <= stride && k <= kPreK;
  if (single && it0 == 0) pcie_quiet(kQuietChainNs);      // decode: the chain starts here
  float g_[kPreK];
  int64_t r_[kPreK];
  int on_[kPreK];
  uint4 xv0 = make_uint4(0, 0, 0, 0);
  if (single && it0 < items) {
    const int64_t t = it0 / d8;
    const int c = (int)(it0 - t * d8);
#pragma unroll
    for (int j = 0; j < kPreK; ++j) {
      if (j < k) {
        g_[j] = wts[t * k + j];
        r_[j] = (int64_t)pos[t * k + j] * d;
        on_[j] = idx[t * k + j];              // expert id; the mask is applied after the wait
      }
    }
    xv0 = reinterpret_cast<const uint4*>(x + t * d)[c];
  }
  DALI_PDL_ENTRY();
  if (rows_ready) wait_host_word(rows_ready, rows_want);  // CPU experts' rows complete
  if (single && it0 < items) {
#pragma unroll
    for (int j = 0; j < kPreK; ++j)
      if (j < k) on_[j] = !mask || mask[on_[j]];
  }
  for (int64_t it = it0; it < items; it += stride) {
    const int64_t t = it / d8;
    const int c = (int)(it - t * d8);
    {
      float acc[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) acc[q] = 0.f;
      auto add_row = [&](bool on_gpu, float g, int64_t r) {
        if (on_gpu)
          combine_add_planes(acc, yp, splits, plane, r, c, g);
        else if (cpu_rows)                             // row computed by the CPU worker,
          combine_add_row(acc, cpu_rows + r, c, g);    // read once after the completion word
      };
      if (single) {
#pragma unroll
        for (int j = 0; j < kPreK; ++j)
          if (j < k) add_row(on_[j], g_[j], r_[j]);
      } else {
        for (int j = 0; j < k; ++j)
          add_row(!mask || mask[idx[t * k + j]], wts[t * k + j], (int64_t)pos[t * k + j] * d);
      }
      if (extra) combine_add_extra(acc, extra + t * d, c);
      const uint4 xv = single ? xv0 : reinterpret_cast<const uint4*>(x + t * d)[c];
      const uint4 ov = combine_finish(xv, acc);
      reinterpret_cast<uint4*>(out + t * d)[c] = ov;
    }
  }
}

// ---------------------------------------------------------------------------
// Counter-hash init: splitmix64(seed, index) -> 24-bit uniform.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void init_uniform_kernel(uint16_t* __restrict__ out, int64_t n, uint64_t seed,
                                    uint64_t offset, float scale) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t z = splitmix64(seed * 0xD1B54A32D192ED03ull + offset + (uint64_t)i);
    const float u = (float)(z >> 40) * (1.0f / 16777216.0f);      // [0, 1)
    out[i] = f32_to_bf16_bits(scale * (2.0f * u - 1.0f));
  }
}

static int sm_count() { return device_sm_count(); }

}  // namespace dali

using namespace dali;

extern "C" int dali_moe_plan(const int32_t* topk_idx, int64_t T, int32_t k, int32_t N,
                             int32_t* offsets, int32_t* perm_token, int32_t* pos, void* stream) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_ETRACE, "expert count %d", N);
  DALI_REQUIRE(T >= 0 && k >= 1 && T * k < (1ll << 31), DALI_ETRACE, "bad plan shape");
launch_pdl(plan_kernel<false>, dim3(1), dim3(kPlanWarps * 32), 0, as_stream(stream), topk_idx,
             T * k, k, N, offsets, perm_token, pos, (const uint4*)nullptr, 0, (uint4*)nullptr);
  DALI_LAUNCH_CHECK("plan_kernel");
  return DALI_OK;
}

extern "C" int dali_moe_plan_permute(const int32_t* topk_idx, int64_t T, int32_t k, int32_t N,
                                     const uint16_t* x, int32_t d, int32_t* offsets,
                                     int32_t* perm_token, int32_t* pos, uint16_t* xp,
                                     void* stream) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_ETRACE, "expert count %d", N);
  DALI_REQUIRE(T >= 0 && k >= 1 && T * k < (1ll << 31), DALI_ETRACE, "bad plan shape");
  DALI_REQUIRE(d % 8 == 0, DALI_ETRACE, "hidden dim %d must be a multiple of 8", d);
  if (T * k > kPlanGatherMax) {
    int rc = dali_moe_plan(topk_idx, T, k, N, offsets, perm_token, pos, stream);
    return rc ? rc : dali_permute(x, perm_token, T * k, d, xp, stream);
  }
  launch_pdl(plan_kernel<true>, dim3(1), dim3(kPlanWarps * 32), 0, as_stream(stream), topk_idx,
             T * k, k, N, offsets, perm_token, pos, reinterpret_cast<const uint4*>(x), d / 8,
             reinterpret_cast<uint4*>(xp));
  DALI_LAUNCH_CHECK("plan_kernel<gather>");
  return DALI_OK;
}

extern "C" int dali_permute(const uint16_t* x, const int32_t* perm_token, int64_t rows, int32_t d,
                            uint16_t* out, void* stream) {
  DALI_REQUIRE(d % 8 == 0, DALI_ETRACE, "hidden dim %d must be a multiple of 8", d);
  if (rows <= 0) return DALI_OK;
  const int64_t blocks = std::min<int64_t>((rows + 7) / 8, (int64_t)sm_count() * 8);
  launch_pdl(permute_kernel, dim3((unsigned)blocks), dim3(256), 0, as_stream(stream), 
      reinterpret_cast<const uint4*>(x), perm_token, rows, d / 8, reinterpret_cast<uint4*>(out));
  DALI_LAUNCH_CHECK("permute_kernel");
  return DALI_OK;
}

extern "C" int dali_expert_ffn_simt(const uint16_t* xp, const int32_t* offsets, int32_t N,
                                    const uint64_t* expert_ptr, int32_t d, int32_t f,
                                    uint16_t* hbuf, float* yp, void* stream) {
  DALI_REQUIRE(d % 8 == 0 && f % 64 == 0, DALI_ETRACE, "need d %% 8 == 0 and f %% 64 == 0");
  cudaStream_t st = as_stream(stream);
  ffn_up_simt<<<dim3((f + 7) / 8, N), 256, 0, st>>>(xp, offsets, expert_ptr, d, f, hbuf);
  DALI_LAUNCH_CHECK("ffn_up_simt");
  ffn_down_simt<<<dim3((d + 7) / 8, N), 256, 0, st>>>(hbuf, offsets, expert_ptr, d, f, yp);
  DALI_LAUNCH_CHECK("ffn_down_simt");
  return DALI_OK;
}

extern "C" int dali_unpermute_combine_wait(const uint16_t* x, const float* yp,
                                           const int32_t* topk_idx, const int32_t* pos,
                                           const float* topk_w, const int8_t* gpu_mask,
                                           const float* cpu_rows, const float* extra, int64_t T,
                                           int32_t k, int32_t d, int32_t splits, int64_t rows,
                                           uint16_t* out, const uint64_t* rows_ready,
                                           uint64_t rows_want, void* stream);

extern "C" int dali_unpermute_combine(const uint16_t* x, const float* yp, const int32_t* topk_idx,
                                      const int32_t* pos, const float* topk_w,
                                      const int8_t* gpu_mask, const float* cpu_rows,
                                      const float* extra, int64_t T, int32_t k, int32_t d,
                                      int32_t splits, int64_t rows, uint16_t* out,
                                      void* stream) {
  return dali_unpermute_combine_wait(x, yp, topk_idx, pos, topk_w, gpu_mask, cpu_rows, extra, T, k,
                                     d, splits, rows, out, nullptr, 0, stream);
}

extern "C" int dali_host_wait_timeouts(uint64_t* out, int32_t reset) {
  unsigned long long v = 0;
  DALI_REQUIRE(out && cudaMemcpyFromSymbol(&v, g_host_wait_timeouts, sizeof(v)) == cudaSuccess,
               DALI_ECUDA, "dali_host_wait_timeouts: read failed");
  if (reset) {
    const unsigned long long z = 0;
    cudaMemcpyToSymbol(g_host_wait_timeouts, &z, sizeof(z));
  }
  *out = v;
  return DALI_OK;
}

extern "C" int dali_unpermute_combine_wait(const uint16_t* x, const float* yp,
                                           const int32_t* topk_idx, const int32_t* pos,
                                           const float* topk_w, const int8_t* gpu_mask,
                                           const float* cpu_rows, const float* extra, int64_t T,
                                           int32_t k, int32_t d, int32_t splits, int64_t rows,
                                           uint16_t* out, const uint64_t* rows_ready,
                                           uint64_t rows_want, void* stream) {
  DALI_REQUIRE(d % 8 == 0, DALI_ETRACE, "hidden dim %d must be a multiple of 8", d);
  if (T <= 0) return DALI_OK;
  const int64_t blocks = std::min<int64_t>((T * (d / 8) + 255) / 256, (int64_t)sm_count() * 8);
  launch_pdl(combine_kernel, dim3((unsigned)blocks), dim3(256), 0, as_stream(stream), x, yp, topk_idx, pos, topk_w,
                                                                  gpu_mask, cpu_rows, extra, T, k,
                                                                  d,
                                                                  splits < 1 ? 1 : splits,
                                                                  rows * (int64_t)d, out,
                                                                  reinterpret_cast<const unsigned long long*>(rows_ready),
                                                                  (unsigned long long)rows_want);
  DALI_LAUNCH_CHECK("combine_kernel");
  return DALI_OK;
}

// ---------------------------------------------------------------------------
// Small host->device copies without a copy engine: every thread loads 16 B of
// mapped pinned host memory (UVA) and stores it to HBM.  Used for per-layer
// control data (pointer tables, CPU-expert result rows) so it never queues
// behind a multi-hundred-MB expert transfer on the H2D copy engine.
// ---------------------------------------------------------------------------
namespace dali {
__global__ void copy_mapped_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src,
                                   int64_t n16, uint8_t* __restrict__ dst_tail,
                                   const uint8_t* __restrict__ src_tail, int tail) {
  if (blockIdx.x == 0 && threadIdx.x == 0) pcie_quiet(kQuietCtlNs);
  DALI_PDL_ENTRY();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // plain loads: every source byte is read once per launch (the stale System
  // Memory lines seen with repeated in-kernel polls do not arise; see
  // wait_host_word)
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += stride)
    dst[i] = src[i];
  if (blockIdx.x == 0 && threadIdx.x < tail)
    dst_tail[threadIdx.x] = *reinterpret_cast<const volatile uint8_t*>(src_tail + threadIdx.x);
}
// Two independent ranges in one launch (the decode head's routing-block and
// permuted-row mirrors): same per-element copies as copy_mapped_kernel.
__global__ void copy_mapped2_kernel(uint4* __restrict__ d0, const uint4* __restrict__ s0,
                                    int64_t n0, uint4* __restrict__ d1,
                                    const uint4* __restrict__ s1, int64_t n1,
                                    uint8_t* __restrict__ dt0, const uint8_t* __restrict__ st0,
                                    int t0, uint8_t* __restrict__ dt1,
                                    const uint8_t* __restrict__ st1, int t1) {
  if (blockIdx.x == 0 && threadIdx.x == 0) pcie_quiet(kQuietCtlNs);
  DALI_PDL_ENTRY();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n0 + n1; i += stride) {
    if (i < n0) d0[i] = s0[i];
    else d1[i - n0] = s1[i - n0];
  }
  if (blockIdx.x == 0 && threadIdx.x < t0)
    dt0[threadIdx.x] = *reinterpret_cast<const volatile uint8_t*>(st0 + threadIdx.x);
  if (blockIdx.x == 0 && threadIdx.x >= 32 && threadIdx.x < 32 + t1)
    dt1[threadIdx.x - 32] = *reinterpret_cast<const volatile uint8_t*>(st1 + threadIdx.x - 32);
}
__global__ void copy_bytes_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                                  int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) dst[i] = src[i];
}
}  // namespace dali

// Bulk host->device copy driven by a few SMs instead of a copy engine: the
// number of CTAs bounds the bytes in flight on the PCIe link, so a small
// latency-critical read issued meanwhile (CPU-expert rows, pointer tables)
// waits behind at most that many bytes instead of a copy engine's deep queue.
namespace dali {
template <int U>
__global__ void __launch_bounds__(512) copy_h2d_sm_kernel(uint4* __restrict__ dst,
                                                           const uint4* __restrict__ src,
                                                           int64_t n16) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const volatile unsigned long long* quiet = &g_pcie_quiet_until;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcv(src + i + u * stride);
    unsigned long long q = *quiet;          // L2 read, overlapped with the PCIe loads
#pragma unroll
    for (int u = 0; u < U; ++u) __stcg(dst + i + u * stride, v[u]);
    while (gtimer_ns() < q) {               // a control transfer / decode chain is running
      __nanosleep(2000);
      q = *quiet;
    }
  }
  for (; i < n16; i += stride) __stcg(dst + i, __ldcv(src + i));
}
}  // namespace dali

// nctas = CTAs x 1 + 64 x (loads in flight per thread - 1), threads per CTA
// = 512 (the low 6 bits pick the CTA count, bits 6.. the unroll 1/2/4)
extern "C" int dali_copy_h2d_sm(void* dst, const void* src, int64_t nbytes, int32_t nctas,
                                void* stream) {
  if (nbytes <= 0) return DALI_OK;
  DALI_REQUIRE(dst && src && nctas >= 1 && ((((uintptr_t)dst | (uintptr_t)src | nbytes) & 15) == 0),
               DALI_ECUDA, "dali_copy_h2d_sm: needs 16-byte aligned pointers and size");
  const int ctas = nctas & 63, u = 1 + (nctas >> 6);
  auto* d4 = reinterpret_cast<uint4*>(dst);
  auto* s4 = reinterpret_cast<const uint4*>(src);
  cudaStream_t st = as_stream(stream);
  if (u >= 4) copy_h2d_sm_kernel<4><<<ctas, 512, 0, st>>>(d4, s4, nbytes >> 4);
  else if (u >= 2) copy_h2d_sm_kernel<2><<<ctas, 512, 0, st>>>(d4, s4, nbytes >> 4);
  else copy_h2d_sm_kernel<1><<<ctas, 512, 0, st>>>(d4, s4, nbytes >> 4);
  DALI_LAUNCH_CHECK("copy_h2d_sm_kernel");
  return DALI_OK;
}

extern "C" int dali_memcpy_async(void* dst, const void* src, size_t nbytes, void* stream) {
  if (nbytes == 0) return DALI_OK;
  DALI_REQUIRE(dst && src, DALI_ECUDA, "dali_memcpy_async: null pointer");
  const cudaError_t e = cudaMemcpyAsync(dst, src, nbytes, cudaMemcpyDefault, as_stream(stream));
  DALI_REQUIRE(e == cudaSuccess, DALI_ECUDA, "dali_memcpy_async: %s", cudaGetErrorString(e));
  return DALI_OK;
}

extern "C" int dali_copy_mapped(void* dst, const void* src, int64_t nbytes, void* stream) {
  if (nbytes <= 0) return DALI_OK;
  DALI_REQUIRE(dst && src, DALI_ECUDA, "dali_copy_mapped: null pointer");
  const bool aligned = (((uintptr_t)dst | (uintptr_t)src) & 15) == 0;
  if (!aligned) {             // small unaligned transfers (token ids): byte copies
    DALI_REQUIRE(nbytes <= (1 << 20), DALI_ECUDA,
                 "dali_copy_mapped: unaligned copies are limited to 1 MiB");
    copy_bytes_kernel<<<(unsigned)((nbytes + 255) / 256), 256, 0, as_stream(stream)>>>(
        reinterpret_cast<uint8_t*>(dst), reinterpret_cast<const uint8_t*>(src), nbytes);
    DALI_LAUNCH_CHECK("copy_bytes_kernel");
    return DALI_OK;
  }
  const int64_t n16 = nbytes >> 4;
  const int tail = (int)(nbytes & 15);
  const int64_t blocks =
      std::max<int64_t>(1, std::min<int64_t>((n16 + 255) / 256, (int64_t)sm_count() * 4));
  launch_pdl(copy_mapped_kernel, dim3((unsigned)blocks), dim3(256), 0, as_stream(stream), 
      reinterpret_cast<uint4*>(dst), reinterpret_cast<const uint4*>(src), n16,
      reinterpret_cast<uint8_t*>(dst) + n16 * 16, reinterpret_cast<const uint8_t*>(src) + n16 * 16,
      tail);
  DALI_LAUNCH_CHECK("copy_mapped_kernel");
  return DALI_OK;
}

extern "C" int dali_copy_mapped2(void* dst0, const void* src0, int64_t n0, void* dst1,
                                 const void* src1, int64_t n1, void* stream) {
  DALI_REQUIRE(n0 >= 0 && n1 >= 0, DALI_ECUDA, "dali_copy_mapped2: negative size");
  DALI_REQUIRE((n0 == 0 || (dst0 && src0)) && (n1 == 0 || (dst1 && src1)), DALI_ECUDA,
               "dali_copy_mapped2: null pointer");
  DALI_REQUIRE(((((uintptr_t)dst0 | (uintptr_t)src0) & 15) == 0 || n0 == 0) &&
               ((((uintptr_t)dst1 | (uintptr_t)src1) & 15) == 0 || n1 == 0),
               DALI_ECUDA, "dali_copy_mapped2: ranges must be 16-byte aligned");
  if (n0 + n1 == 0) return DALI_OK;
  const int64_t a16 = n0 >> 4, b16 = n1 >> 4;
  const int64_t blocks =
      std::max<int64_t>(1, std::min<int64_t>((a16 + b16 + 255) / 256, (int64_t)sm_count() * 4));
  launch_pdl(copy_mapped2_kernel, dim3((unsigned)blocks), dim3(256), 0, as_stream(stream),
             reinterpret_cast<uint4*>(dst0), reinterpret_cast<const uint4*>(src0), a16,
             reinterpret_cast<uint4*>(dst1), reinterpret_cast<const uint4*>(src1), b16,
             reinterpret_cast<uint8_t*>(dst0) + a16 * 16,
             reinterpret_cast<const uint8_t*>(src0) + a16 * 16, (int)(n0 & 15),
             reinterpret_cast<uint8_t*>(dst1) + b16 * 16,
             reinterpret_cast<const uint8_t*>(src1) + b16 * 16, (int)(n1 & 15));
  DALI_LAUNCH_CHECK("copy_mapped2_kernel");
  return DALI_OK;
}

// ---------------------------------------------------------------------------
// Shared-expert finish: out[t,:] = (sum_s ys[s,t,:]) * gate(t), gate(t) =
// sigmoid(h[t,:] . g) for Qwen's gated shared expert (1 when g == NULL).
// One CTA per token: replaces a plane sum + fp32 cast + GEMV + sigmoid + mul.
// ---------------------------------------------------------------------------
namespace dali {
__global__ void shared_finish_kernel(const float* __restrict__ ys, int splits, int64_t plane,
                                     const uint16_t* __restrict__ h,
                                     const uint16_t* __restrict__ g, int d,
                                     float* __restrict__ out) {
  DALI_PDL_ENTRY();
  const int64_t t = blockIdx.x;
  __shared__ float red[32];
  float gate = 1.0f;
  if (g) {
    float acc = 0.f;
    for (int i = threadIdx.x; i < d; i += blockDim.x)
      acc += bf16_bits_to_f32(h[t * d + i]) * bf16_bits_to_f32(g[i]);
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x < 32) {
      float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (threadIdx.x == 0) red[0] = 1.0f / (1.0f + __expf(-v));
    }
    __syncthreads();
    gate = red[0];
  }
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    float v = ys[t * d + i];
    for (int s = 1; s < splits; ++s) v += ys[s * plane + t * d + i];
    out[t * d + i] = v * gate;
  }
}
}  // namespace dali

extern "C" int dali_shared_finish(const float* ys, int32_t splits, int64_t T, int32_t d,
                                  const uint16_t* h, const uint16_t* gate_w, float* out,
                                  void* stream) {
  if (T <= 0) return DALI_OK;
  DALI_REQUIRE(splits >= 1, DALI_ETRACE, "splits must be >= 1");
  launch_pdl(shared_finish_kernel, dim3((unsigned)T), dim3(256), 0, as_stream(stream), ys,
             splits, T * (int64_t)d, h, gate_w, d, out);
  DALI_LAUNCH_CHECK("shared_finish_kernel");
  return DALI_OK;
}

// ---------------------------------------------------------------------------
// Decode GEMV: y (B, M) bf16 = x (B, K) bf16 . W (M, K)^T, B <= 8 tokens.
// Weight streaming: one warp per output row, 16-byte loads (8 bf16 per lane
// per step, 8 steps in flight), x staged in shared memory, fp32 accumulation.
// ---------------------------------------------------------------------------
namespace dali {
constexpr int kGemvWarps = 8;
constexpr int kGemvMaxB = 8;

template <int B>
__global__ void __launch_bounds__(kGemvWarps * 32)
gemv_bf16_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, int M, int K,
                 uint16_t* __restrict__ y) {
  DALI_PDL_ENTRY();
  extern __shared__ uint4 sx[];                       // B x K bf16
  const int k8 = K >> 3;
  for (int i = threadIdx.x; i < B * k8; i += blockDim.x) sx[i] = reinterpret_cast<const uint4*>(x)[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m = blockIdx.x * kGemvWarps + warp;
  if (m >= M) return;
  const uint4* wr = reinterpret_cast<const uint4*>(w + (int64_t)m * K);
  float acc[B];
#pragma unroll
  for (int b = 0; b < B; ++b) acc[b] = 0.f;
#pragma unroll 4
  for (int c = lane; c < k8; c += 32) {
    const uint4 wv = __ldg(wr + c);
    const uint32_t* ww = reinterpret_cast<const uint32_t*>(&wv);
#pragma unroll
    for (int b = 0; b < B; ++b) {
      const uint4 xv = sx[b * k8 + c];
      const uint32_t* xx = reinterpret_cast<const uint32_t*>(&xv);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc[b] = fmaf(__uint_as_float(ww[q] << 16), __uint_as_float(xx[q] << 16), acc[b]);
        acc[b] = fmaf(__uint_as_float(ww[q] & 0xffff0000u), __uint_as_float(xx[q] & 0xffff0000u),
                      acc[b]);
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
}  // namespace dali

namespace dali {
namespace gemv {
struct NormArgs;
}
int launch_gemv_stream(const uint16_t* x, const uint16_t* w, int Bt, int M, int K, uint16_t* y,
                       cudaStream_t st, const gemv::NormArgs* norm);
// A/B switch: DALI_GEMV_STREAM=0 keeps every GEMV on the row-per-warp kernel
static bool gemv_stream_enabled() {
  static const bool v = [] {
    const char* e = getenv("DALI_GEMV_STREAM");
    return !(e && e[0] == '0');
  }();
  return v;
}
}  // namespace dali

extern "C" int dali_gemv_bf16(const uint16_t* x, const uint16_t* w, int32_t Bt, int32_t M,
                              int32_t K, uint16_t* y, void* stream) {
  DALI_REQUIRE(Bt >= 1 && Bt <= dali::kGemvMaxB, DALI_ETRACE, "gemv batch %d outside [1, %d]",
               Bt, dali::kGemvMaxB);
  DALI_REQUIRE(K % 8 == 0 && M >= 1, DALI_ETRACE, "gemv needs K %% 8 == 0 (K=%d)", K);
  const size_t smem = (size_t)Bt * K * 2;
  DALI_REQUIRE(smem <= 200 * 1024, DALI_ETRACE, "gemv activations exceed shared memory");
  if (dali::gemv_stream_enabled()) {
    const int rc = dali::launch_gemv_stream(x, w, Bt, M, K, y, as_stream(stream), nullptr);
    if (rc >= 0) return rc;
  }
  const dim3 grid((unsigned)((M + dali::kGemvWarps - 1) / dali::kGemvWarps));
  const dim3 block(dali::kGemvWarps * 32);
  cudaStream_t st = as_stream(stream);
  cudaError_t e = cudaSuccess;
  switch (Bt) {
#define DALI_GEMV_CASE(BB)                                                                  \
  case BB: {                                                                                \
    DALI_ONCE_PER_DEVICE(cudaFuncSetAttribute(dali::gemv_bf16_kernel<BB>,                   \
                                              cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                              200 * 1024));                                \
    e = launch_pdl(dali::gemv_bf16_kernel<BB>, grid, block, smem, st, x, w, M, K, y);      \
    break;                                                                                 \
  }
    DALI_GEMV_CASE(1) DALI_GEMV_CASE(2) DALI_GEMV_CASE(3) DALI_GEMV_CASE(4)
    DALI_GEMV_CASE(5) DALI_GEMV_CASE(6) DALI_GEMV_CASE(7) DALI_GEMV_CASE(8)
#undef DALI_GEMV_CASE
  }
  (void)e;
  DALI_LAUNCH_CHECK("gemv_bf16_kernel");
  return DALI_OK;
}

extern "C" int dali_init_uniform_bf16(uint16_t* out, int64_t n, uint64_t seed, uint64_t offset,
                                      float stdev, void* stream) {
  if (n <= 0) return DALI_OK;
  const int64_t blocks = std::min<int64_t>((n + 255) / 256, (int64_t)sm_count() * 16);
  init_uniform_kernel<<<(unsigned)blocks, 256, 0, as_stream(stream)>>>(out, n, seed, offset,
                                                                       stdev * 1.7320508075688772f);
  DALI_LAUNCH_CHECK("init_uniform_kernel");
  return DALI_OK;
}

extern "C" int dali_expert_ffn(const uint16_t* xp, const int32_t* offsets, int32_t N,
                               const uint64_t* expert_ptr, int32_t d, int32_t f, int64_t rows,
                               int32_t max_rows_per_expert, uint16_t* hbuf, float* yp,
                               void* stream) {
  (void)rows;
  (void)max_rows_per_expert;
  return dali_expert_ffn_simt(xp, offsets, N, expert_ptr, d, f, hbuf, yp, stream);
}

// ---------------------------------------------------------------------------
// Fused residual add + RMSNorm (engine plumbing around the MoE layer):
//   x_out = x (+ a);  h = bf16(x_out * rsqrt(mean(x_out^2) + eps)) * w
// one CTA per row, 8 bf16 per thread step, fp32 statistics.
// ---------------------------------------------------------------------------
namespace dali {
__global__ void add_rmsnorm_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ a,
                                   const uint16_t* __restrict__ w, float eps, int d,
                                   uint16_t* __restrict__ x_out, uint16_t* __restrict__ h) {
  DALI_PDL_ENTRY();
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * d);
  const uint4* ar = a ? reinterpret_cast<const uint4*>(a + row * d) : nullptr;
  const int d8 = d >> 3;
  float ss = 0.f;
  for (int c = threadIdx.x; c < d8; c += blockDim.x) {
    uint4 xv = xr[c];
    uint32_t* xw = reinterpret_cast<uint32_t*>(&xv);
    if (ar) {
      const uint4 av = ar[c];
      const uint32_t* aw = reinterpret_cast<const uint32_t*>(&av);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float lo = __uint_as_float(xw[q] << 16) + __uint_as_float(aw[q] << 16);
        const float hi = __uint_as_float(xw[q] & 0xffff0000u) + __uint_as_float(aw[q] & 0xffff0000u);
        xw[q] = (uint32_t)f32_to_bf16_bits(lo) | ((uint32_t)f32_to_bf16_bits(hi) << 16);
      }
      if (x_out) reinterpret_cast<uint4*>(x_out + row * d)[c] = xv;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float lo = __uint_as_float(xw[q] << 16), hi = __uint_as_float(xw[q] & 0xffff0000u);
      ss += lo * lo + hi * hi;
    }
  }
  __shared__ float red[32];
  for (int o = 16; o; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  const float r = rsqrtf(red[0] / (float)d + eps);
  const uint4* src = (ar && x_out) ? reinterpret_cast<const uint4*>(x_out + row * d) : xr;
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  for (int c = threadIdx.x; c < d8; c += blockDim.x) {
    uint4 xv = src[c];
    if (ar && !x_out) {
      const uint4 av = ar[c];
      uint32_t* xw = reinterpret_cast<uint32_t*>(&xv);
      const uint32_t* aw = reinterpret_cast<const uint32_t*>(&av);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float lo = __uint_as_float(xw[q] << 16) + __uint_as_float(aw[q] << 16);
        const float hi = __uint_as_float(xw[q] & 0xffff0000u) + __uint_as_float(aw[q] & 0xffff0000u);
        xw[q] = (uint32_t)f32_to_bf16_bits(lo) | ((uint32_t)f32_to_bf16_bits(hi) << 16);
      }
    }
    const uint4 wv = wr[c];
    const uint32_t* xw = reinterpret_cast<const uint32_t*>(&xv);
    const uint32_t* ww = reinterpret_cast<const uint32_t*>(&wv);
    uint4 ov;
    uint32_t* ow = reinterpret_cast<uint32_t*>(&ov);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // torch order: bf16(x * r) then * w (bf16 product rounded)
      const float lo = __uint_as_float((uint32_t)f32_to_bf16_bits(__uint_as_float(xw[q] << 16) * r) << 16) *
                       __uint_as_float(ww[q] << 16);
      const float hi = __uint_as_float((uint32_t)f32_to_bf16_bits(__uint_as_float(xw[q] & 0xffff0000u) * r) << 16) *
                       __uint_as_float(ww[q] & 0xffff0000u);
      ow[q] = (uint32_t)f32_to_bf16_bits(lo) | ((uint32_t)f32_to_bf16_bits(hi) << 16);
    }
    reinterpret_cast<uint4*>(h + row * d)[c] = ov;
  }
}
}  // namespace dali

extern "C" int dali_add_rmsnorm(const uint16_t* x, const uint16_t* a, const uint16_t* w, float eps,
                                int64_t T, int32_t d, uint16_t* x_out, uint16_t* h,
                                void* stream) {
  DALI_REQUIRE(d % 8 == 0, DALI_ETRACE, "hidden dim %d must be a multiple of 8", d);
  if (T <= 0) return DALI_OK;
  launch_pdl(dali::add_rmsnorm_kernel, dim3((unsigned)T), dim3(256), 0, dali::as_stream(stream), x, a, w, eps, d, x_out,
                                                                             h);
  DALI_LAUNCH_CHECK("add_rmsnorm_kernel");
  return DALI_OK;
}
