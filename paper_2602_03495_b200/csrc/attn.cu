// Decode-step attention plumbing around the MoE layer (not one of the DALI
// subsystems, but on the per-token critical path): RoPE + KV-cache append
// and a split-K ("flash-decoding") GQA attention for one query token per
// sequence.  The position / valid length are read from DEVICE scalars so a
// whole decode step can be captured once in a CUDA graph and replayed.
#include "common.cuh"

namespace dali {

// qkv (B, (H+2KV)*hd) bf16 -> q (B, H, hd) bf16 rotated; k rotated and v
// written into the caches at position *pos: cache layout (B, KV, max_len, hd).
__global__ void rope_append_kernel(const uint16_t* __restrict__ qkv, const float* __restrict__ cos_t,
                                   const float* __restrict__ sin_t, const int32_t* __restrict__ pos_p,
                                   int H, int KV, int hd, int max_len, uint16_t* __restrict__ q_out,
                                   uint16_t* __restrict__ kc, uint16_t* __restrict__ vc) {
  DALI_PDL_ENTRY();
  const int b = blockIdx.y;
  const int head = blockIdx.x;                 // 0..H+2KV-1
  const int pos = *pos_p;
  const int half = hd >> 1;
  const uint16_t* src = qkv + ((int64_t)b * (H + 2 * KV) + head) * hd;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float x0 = bf16_bits_to_f32(src[i]), x1 = bf16_bits_to_f32(src[i + half]);
    if (head < H + KV) {
      const float c = cos_t[(int64_t)pos * half + i], s = sin_t[(int64_t)pos * half + i];
      const uint16_t o0 = f32_to_bf16_bits(x0 * c - x1 * s);
      const uint16_t o1 = f32_to_bf16_bits(x1 * c + x0 * s);
      if (head < H) {
        uint16_t* q = q_out + ((int64_t)b * H + head) * hd;
        q[i] = o0;
        q[i + half] = o1;
      } else {
        uint16_t* k = kc + (((int64_t)b * KV + (head - H)) * max_len + pos) * hd;
        k[i] = o0;
        k[i + half] = o1;
      }
    } else {
      uint16_t* v = vc + (((int64_t)b * KV + (head - H - KV)) * max_len + pos) * hd;
      v[i] = src[i];
      v[i + half] = src[i + half];
    }
  }
}

// Split-K decode attention.  grid (B*H, splits); 4 warps per CTA; each warp
// walks positions p = warp, warp+4, ... of its chunk with an online softmax;
// HD in {64, 128} (HD/32 elements per lane).  Partials -> ws, merged by attn_merge.
constexpr int kAttnWarps = 4;

template <int EL>
__device__ __forceinline__ void load_bf16_lane(const uint16_t* p, float* out) {
  if constexpr (EL == 4) {
    const uint2 raw = *reinterpret_cast<const uint2*>(p);
    out[0] = __uint_as_float(raw.x << 16);
    out[1] = __uint_as_float(raw.x & 0xffff0000u);
    out[2] = __uint_as_float(raw.y << 16);
    out[3] = __uint_as_float(raw.y & 0xffff0000u);
  } else {
    const uint32_t raw = *reinterpret_cast<const uint32_t*>(p);
    out[0] = __uint_as_float(raw << 16);
    out[1] = __uint_as_float(raw & 0xffff0000u);
  }
}

template <int HD>
__global__ void __launch_bounds__(kAttnWarps * 32)
decode_attn_kernel(const uint16_t* __restrict__ q, const uint16_t* __restrict__ kc,
                   const uint16_t* __restrict__ vc, const int32_t* __restrict__ len_p, int H,
                   int KV, int max_len, float scale, float* __restrict__ ws) {
  DALI_PDL_ENTRY();
  constexpr int EL = HD / 32;
  const int bh = blockIdx.x, b = bh / H, h = bh % H;
  const int kvh = h / (H / KV);
  const int split = blockIdx.y, nsplit = gridDim.y;
  const int len = *len_p;
  const int chunk = (len + nsplit - 1) / nsplit;
  const int p0 = split * chunk, p1 = min(len, p0 + chunk);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint16_t* qh = q + ((int64_t)b * H + h) * HD;
  float qv[EL];
#pragma unroll
  for (int i = 0; i < EL; ++i) qv[i] = bf16_bits_to_f32(qh[lane * EL + i]) * scale;
  const uint16_t* kb = kc + ((int64_t)b * KV + kvh) * max_len * HD;
  const uint16_t* vb = vc + ((int64_t)b * KV + kvh) * max_len * HD;
  float m = -INFINITY, l = 0.f, acc[EL];
#pragma unroll
  for (int i = 0; i < EL; ++i) acc[i] = 0.f;
  // one position of look-ahead: the next K/V rows are requested before this
  // position's dot product and shuffle reduction, so a warp has two rows of
  // loads in flight instead of one
  float kn[EL], vn[EL];
  if (p0 + warp < p1) {
    load_bf16_lane<EL>(kb + (int64_t)(p0 + warp) * HD + lane * EL, kn);
    load_bf16_lane<EL>(vb + (int64_t)(p0 + warp) * HD + lane * EL, vn);
  }
  for (int p = p0 + warp; p < p1; p += kAttnWarps) {
    float kv_[EL], vv[EL];
#pragma unroll
    for (int i = 0; i < EL; ++i) {
      kv_[i] = kn[i];
      vv[i] = vn[i];
    }
    if (p + kAttnWarps < p1) {
      load_bf16_lane<EL>(kb + (int64_t)(p + kAttnWarps) * HD + lane * EL, kn);
      load_bf16_lane<EL>(vb + (int64_t)(p + kAttnWarps) * HD + lane * EL, vn);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < EL; ++i) s += qv[i] * kv_[i];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mn = fmaxf(m, s);
    const float corr = __expf(m - mn), ps = __expf(s - mn);
    l = l * corr + ps;
#pragma unroll
    for (int i = 0; i < EL; ++i) acc[i] = acc[i] * corr + ps * vv[i];
    m = mn;
  }
  __shared__ float sm[kAttnWarps], sl[kAttnWarps], sacc[kAttnWarps][HD];
  if (lane == 0) { sm[warp] = m; sl[warp] = l; }
#pragma unroll
  for (int i = 0; i < EL; ++i) sacc[warp][lane * EL + i] = acc[i];
  __syncthreads();
  if (warp == 0) {
    float M = -INFINITY;
    for (int w = 0; w < kAttnWarps; ++w) M = fmaxf(M, sm[w]);
    float L = 0.f, A[EL];
#pragma unroll
    for (int i = 0; i < EL; ++i) A[i] = 0.f;
    for (int w = 0; w < kAttnWarps; ++w) {
      const float c = sm[w] == -INFINITY ? 0.f : __expf(sm[w] - M);
      L += sl[w] * c;
#pragma unroll
      for (int i = 0; i < EL; ++i) A[i] += sacc[w][lane * EL + i] * c;
    }
    float* out = ws + ((int64_t)bh * nsplit + split) * (HD + 2);
    if (lane == 0) { out[0] = M; out[1] = L; }
#pragma unroll
    for (int i = 0; i < EL; ++i) out[2 + lane * EL + i] = A[i];
  }
}

// Split merge.  Every partial of the row is loaded up front (the split count
// is bounded by kMergeMax) so the merge pays one memory latency instead of one
// per split; the arithmetic order is unchanged.
constexpr int kMergeMax = 16;

template <int HD>
__global__ void attn_merge_kernel(const float* __restrict__ ws, int nsplit,
                                  uint16_t* __restrict__ o) {
  DALI_PDL_ENTRY();
  const int bh = blockIdx.x;
  const float* in = ws + (int64_t)bh * nsplit * (HD + 2);
  float ms[kMergeMax], ls[kMergeMax];
#pragma unroll
  for (int s = 0; s < kMergeMax; ++s) {
    ms[s] = s < nsplit ? in[s * (HD + 2)] : -INFINITY;
    ls[s] = s < nsplit ? in[s * (HD + 2) + 1] : 0.f;
  }
  float M = -INFINITY;
#pragma unroll
  for (int s = 0; s < kMergeMax; ++s)
    if (s < nsplit) M = fmaxf(M, ms[s]);
  for (int i = threadIdx.x; i < HD; i += blockDim.x) {
    float as[kMergeMax];
#pragma unroll
    for (int s = 0; s < kMergeMax; ++s) as[s] = s < nsplit ? in[s * (HD + 2) + 2 + i] : 0.f;
    float L = 0.f, A = 0.f;
#pragma unroll
    for (int s = 0; s < kMergeMax; ++s) {
      if (s >= nsplit) break;
      const float c = ms[s] == -INFINITY ? 0.f : __expf(ms[s] - M);
      L += ls[s] * c;
      A += as[s] * c;
    }
    o[(int64_t)bh * HD + i] = f32_to_bf16_bits(A / L);
  }
}

}  // namespace dali

extern "C" int dali_rope_append(const uint16_t* qkv, const float* cos_t, const float* sin_t,
                                const int32_t* pos, int32_t B, int32_t H, int32_t KV, int32_t hd,
                                int32_t max_len, uint16_t* q_out, uint16_t* k_cache,
                                uint16_t* v_cache, void* stream) {
  DALI_REQUIRE(hd % 2 == 0 && H % KV == 0, DALI_ETRACE, "bad attention geometry");
  dali::launch_pdl(dali::rope_append_kernel, dim3(dim3(H + 2 * KV, B)), dim3(64), 0, dali::as_stream(stream), 
      qkv, cos_t, sin_t, pos, H, KV, hd, max_len, q_out, k_cache, v_cache);
  DALI_LAUNCH_CHECK("rope_append_kernel");
  return DALI_OK;
}

extern "C" int dali_decode_attention(const uint16_t* q, const uint16_t* k_cache,
                                     const uint16_t* v_cache, const int32_t* len, int32_t B,
                                     int32_t H, int32_t KV, int32_t hd, int32_t max_len,
                                     int32_t splits, float scale, float* workspace, uint16_t* out,
                                     void* stream) {
  DALI_REQUIRE(hd == 128 || hd == 64, DALI_ETRACE,
               "decode attention kernel supports head_dim 64 or 128, got %d", hd);
  DALI_REQUIRE(H % KV == 0 && splits >= 1 && splits <= dali::kMergeMax, DALI_ETRACE,
               "bad attention geometry (splits %d, at most %d)", splits, dali::kMergeMax);
  cudaStream_t st = dali::as_stream(stream);
  if (hd == 128) {
    dali::launch_pdl(dali::decode_attn_kernel<128>, dim3(dim3(B * H, splits)), dim3(dali::kAttnWarps * 32), 0, st, 
        q, k_cache, v_cache, len, H, KV, max_len, scale, workspace);
    DALI_LAUNCH_CHECK("decode_attn_kernel");
    dali::launch_pdl(dali::attn_merge_kernel<128>, dim3(B * H), dim3(128), 0, st, workspace, splits, out);
  } else {
    dali::launch_pdl(dali::decode_attn_kernel<64>, dim3(dim3(B * H, splits)), dim3(dali::kAttnWarps * 32), 0, st, 
        q, k_cache, v_cache, len, H, KV, max_len, scale, workspace);
    DALI_LAUNCH_CHECK("decode_attn_kernel");
    dali::launch_pdl(dali::attn_merge_kernel<64>, dim3(B * H), dim3(64), 0, st, workspace, splits, out);
  }
  DALI_LAUNCH_CHECK("attn_merge_kernel");
  return DALI_OK;
}
