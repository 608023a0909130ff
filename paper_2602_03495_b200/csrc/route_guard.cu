// (1) Gating, engine path: bf16 hidden x bf16 router, fp32 FFMA logits with a
// certified rank margin and an fp64 recompute of the rows it cannot certify.
// Restates derive_workloads / topk_indices (reference trace.py:236-265) and
// the residual shift of predict_next_layer (prefetch.py:127-136).
//
// Why fp32 is allowed to decide the reference's fp64 ranks.  Every logit is
// a dot product z_j = sum_i x_i W_ij.  bf16 x bf16 products are exact in fp32
// and every FFMA rounds once, so for any summation tree of height H
//     |fl32(z_j) - z_j| <= gamma_H * sum_i |x_i W_ij| <= gamma_H ||x|| ||W_:j||
// (gamma_H = H u / (1 - H u), u = 2^-24; Cauchy-Schwarz for the last step).
// The reference ranks fp64 dgemm logits, whose own error (gamma_d in fp64) is
// ~1e-13 relative, far below any margin this kernel certifies.  A row whose
// k+1 leading fp32 logits are separated pairwise by more than the sum of the
// two bounds therefore has exactly the reference's top-k indices, in the
// reference's order.  Every other row (near-ties, non-finite values, softmax
// underflow territory) is recomputed in fp64 by the same CTA and ranked like
// the reference (softmax, ties to the lower index); each such row bumps a
// device fire counter (dali_route_fire_count).
//
// Summation height.  Each thread accumulates its d-slice in blocks of 32
// FFMAs that are flushed into an outer accumulator (height 32 + #blocks), the
// S slices are summed by a pairwise tree (log2 S) and, for the cluster
// variant, the C CTAs' partials are summed in rank order (C - 1).  The host
// computes H from the launch geometry; a 1% factor covers the fp32 error of
// the norms themselves.
//
// Two launch shapes:
//  * T <= 16 (decode): one thread-block cluster of C CTAs splits d; partial
//    logits and norms go to the leader CTA through distributed shared memory
//    and the leader ranks, writes the histogram directly (no zeroing launch).
//    The router slices (which do not depend on the previous kernel) are
//    requested before the PDL wait, so they stream while the predecessor
//    drains; only the hidden rows wait.
//  * T > 16 (prefill): one CTA per TB tokens over the whole of d.
// Operands stream through a 3-stage cp.async ring (raw bf16); each stage is
// converted once to fp32 in shared memory (residual added in fp64 there, as
// numpy's `hidden + res`), then every thread accumulates a 4-token x
// 8-expert register tile.
// Ranking (rank_tail): at decode sizes (tokens x experts <= 2 x threads)
// every (token, expert) pair is ranked at once by one thread counting the
// experts that beat it (logit, then lower index); larger tiles pick the k+1
// leaders by warp-wide argmax rounds, a warp per token.  Then a warp per
// token certifies the k+1 leading gaps, finishes the softmax and writes.
#include <algorithm>
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace dali {

__device__ unsigned long long g_route_fires = 0;     // rows recomputed in fp64
__device__ unsigned long long g_route_rows = 0;      // rows routed by this kernel
#ifdef DALI_RG_PROF
__device__ unsigned long long g_rg_prof[8][12];
#define RG_MARK(i)                                                                \
  do {                                                                            \
    if (threadIdx.x == 0 && blockIdx.x < 8) {                                     \
      unsigned long long _t;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t));                      \
      g_rg_prof[blockIdx.x][i] = _t;                                              \
    }                                                                             \
  } while (0)
#else
#define RG_MARK(i) do {} while (0)
#endif

namespace rg {

constexpr int kThreads = 256;
constexpr int kStages = 3;
constexpr int kStageBytes = 24 * 1024;

struct Geo {            // launch geometry shared by host and device
  int TB, NP, EG, TG, S, logS, DC, C, ds, warp_mode;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

__device__ __forceinline__ void bf16x2_to_f32(uint32_t v, float& lo, float& hi) {
  lo = __uint_as_float(v << 16);
  hi = __uint_as_float(v & 0xffff0000u);
}

// fp64 recompute of one uncertified row by the whole CTA (rare path).  Only
// the candidate experts U -- every j whose fp32 upper bound z_j + B_j reaches
// L = min over the k fp32-leading experts of z - B -- are recomputed: the k
// leaders certainly beat every expert outside U (their exact logits are >= L
// > the outsider's), so the exact top-k lies in U and its order is the fp64
// order within U.  fp64 products and sums, max-shifted fp64 softmax (logits
// outside U enter the denominator from fp32), rank by (-p, index): the
// reference's gate_scores + topk_indices (trace.py:229-250).  B200's fp64
// pipe is narrow, so recomputing 2-4 candidates instead of all N experts is
// what keeps a fire cheap.
__device__ __forceinline__ double bf16_to_f64_fast(uint32_t b) {
  const uint32_t e = (b >> 7) & 0xffu;
  if (e - 1u < 254u) {                          // normal: rebias exponent, shift mantissa
    const uint32_t hi = ((b & 0x8000u) << 16) | ((e + 896u) << 20) | ((b & 0x7fu) << 13);
    return __hiloint2double((int)hi, 0);
  }
  return (double)__uint_as_float(b << 16);      // zero / subnormal / inf / nan
}

__device__ void fp64_row_cand(const uint16_t* __restrict__ hrow,
                              const double* __restrict__ residual,
                              const uint16_t* __restrict__ gate, int d, int N, int k, int renorm,
                              const uint32_t* cmask, const float* z32, double* xs64,
                              double* sh_part, double* sh_row, int* sh_cl, int* sh_nc,
                              int32_t* idx_out, float* w_out, int* sh_hist) {
  const int tid = threadIdx.x;
  if (tid < 32) {                                // candidate list, ascending index
    int base = 0;
    for (int q = 0; q < 8; ++q) {
      const uint32_t m = cmask[q];
      if ((m >> tid) & 1u) sh_cl[base + __popc(m & ((1u << tid) - 1u))] = 32 * q + tid;
      base += __popc(m);
    }
    if (tid == 0) *sh_nc = base;
  }
  __syncthreads();
  RG_MARK(9);
  const int nc = *sh_nc;
  if (nc <= 16) {
    // Few candidates (the normal fire): a warp step covers R = 32 / nc
    // router rows, lane = (row r, candidate c), so one load instruction
    // touches R rows' lines (not 32) and the row element is a broadcast.
    // Each thread loads its rows and router elements straight from global
    // (16 in flight, no staging pass); partials meet in a fixed order.
    const int R = 32 / nc;
    const int lane = tid & 31, warp = tid >> 5;
    const int r = lane / nc, c = lane - r * nc;
    double acc0 = 0.0, acc1 = 0.0;
    if (r < R) {
      const uint16_t* gcol = gate + sh_cl[c];
      constexpr int kB = 16;
      const int stride = (kThreads / 32) * R;    // rows per CTA step
      int i0 = warp * R + r;
#pragma unroll 2
      for (; i0 + (kB - 1) * stride < d; i0 += kB * stride) {
        uint16_t w[kB], xb[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          w[b] = __ldg(gcol + (int64_t)(i0 + b * stride) * N);
          xb[b] = hrow[i0 + b * stride];
        }
#pragma unroll
        for (int b = 0; b < kB; b += 2) {
          double x0 = bf16_to_f64_fast(xb[b]), x1 = bf16_to_f64_fast(xb[b + 1]);
          if (residual) {
            x0 = __dadd_rn(x0, residual[i0 + b * stride]);
            x1 = __dadd_rn(x1, residual[i0 + (b + 1) * stride]);
          }
          acc0 = fma(x0, bf16_to_f64_fast(w[b]), acc0);
          acc1 = fma(x1, bf16_to_f64_fast(w[b + 1]), acc1);
        }
      }
      for (int i = i0; i < d; i += stride) {
        double x = bf16_to_f64_fast(hrow[i]);
        if (residual) x = __dadd_rn(x, residual[i]);
        acc0 = fma(x, bf16_to_f64_fast(__ldg(gcol + (int64_t)i * N)), acc0);
      }
    }
    double* part = sh_part + 64;                  // [kThreads]
    part[tid] = acc0 + acc1;
    __syncthreads();
    if (tid < nc) {
      double t = 0.0;
      for (int q = 0; q < kThreads / 32; ++q)
        for (int rr = 0; rr < R; ++rr) t += part[q * 32 + rr * nc + tid];
      sh_part[tid] = t;                           // candidate logits, list order
    }
    __syncthreads();
  } else {
    for (int i = tid; i < d; i += kThreads) {      // the row in fp64 (+ residual), once
      double x = bf16_to_f64_fast(hrow[i]);
      if (residual) x = __dadd_rn(x, residual[i]);
      xs64[i] = x;
    }
    __syncthreads();
    int S = 1;
    while (2 * S * nc <= kThreads) S *= 2;         // power-of-two slices per candidate
    const int c = tid % nc, sl = tid / nc;
    if (sl < S) {
      const int e = sh_cl[c];
      double acc0 = 0.0, acc1 = 0.0;
      constexpr int kB = 16;                      // router loads in flight per thread
      for (int i0 = sl; i0 < d; i0 += kB * S) {
        uint16_t w[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int i = i0 + b * S;
          w[b] = i < d ? __ldg(gate + (int64_t)i * N + e) : (uint16_t)0;
        }
#pragma unroll
        for (int b = 0; b < kB; b += 2) {
          const int i = i0 + b * S;
          if (i < d) acc0 = fma(xs64[i], bf16_to_f64_fast(w[b]), acc0);
          if (i + S < d) acc1 = fma(xs64[i + S], bf16_to_f64_fast(w[b + 1]), acc1);
        }
      }
      sh_part[sl * nc + c] = acc0 + acc1;
    }
    __syncthreads();
    for (int half = S >> 1; half >= 1; half >>= 1) {
      for (int i = tid; i < half * nc; i += kThreads) sh_part[i] += sh_part[i + half * nc];
      __syncthreads();
    }
  }
  RG_MARK(10);
  if (tid < 32) {
    const int lane = tid;
    // logits: fp64 for candidates, fp32 for the rest (denominator only)
    for (int j = lane; j < N; j += 32) sh_row[j] = (double)z32[j];
    __syncwarp();
    for (int q = lane; q < nc; q += 32) sh_row[sh_cl[q]] = sh_part[q];
    __syncwarp();
    double mx = -INFINITY;
    for (int j = lane; j < N; j += 32) mx = fmax(mx, sh_row[j]);
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double sum = 0.0;
    for (int j = lane; j < N; j += 32) {
      const double ex = exp(sh_row[j] - mx);
      sh_row[j] = ex;
      sum += ex;
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    __syncwarp();
    for (int j = lane; j < N; j += 32) sh_row[j] = sh_row[j] / sum;
    __syncwarp();
    int sel[DALI_MAX_TOPK];                    // lane 0 only (k <= 16)
    for (int q = lane; q < nc; q += 32) {
      const int j = sh_cl[q];
      const double pj = sh_row[j];
      int rank = 0;
      for (int u = 0; u < nc; ++u) {
        const int ju = sh_cl[u];
        const double pu = sh_row[ju];
        rank += (pu > pj) || (pu == pj && ju < j);
      }
      if (rank < k) {
        sh_part[1024 + rank] = (double)j;       // selected ids, rank order
        if (idx_out) idx_out[rank] = j;
        atomicAdd(&sh_hist[j], 1);
      }
    }
    __syncwarp();
    if (w_out && lane == 0) {
      double tot = 0.0;
      for (int r = 0; r < k; ++r) {
        sel[r] = (int)sh_part[1024 + r];
        tot += sh_row[sel[r]];
      }
      for (int r = 0; r < k; ++r) {
        const double p = sh_row[sel[r]];
        w_out[r] = (float)(renorm ? p / tot : p);
      }
    }
  }
  __syncthreads();
}

// Shared tail of both launch shapes.  zl: [TB][NP] fp32 logits of this
// CTA's tokens, xn: [TB] squared token norms, wn: [N] router column norms.
// Counting ranks, then a warp per token certifies / softmaxes / writes; rows
// that cannot be certified are recomputed in fp64 (fp64_row_cand).  ring64
// is scratch for the recompute: >= (d + 1040) doubles, not aliasing zl.
struct TailSmem {
  int* hist;                          // [256] per-CTA expert histogram
  int (*sel)[DALI_MAX_TOPK + 1];      // [TB] leading experts in rank order
  int* flag;                          // [TB] rows sent to fp64
  int* nflag;
  uint32_t (*cmask)[8];               // [TB] candidate masks of those rows
  int* bad;                           // [TB] non-finite logit seen
  double* row64;                      // [256]
  int* cl;                            // [256]
  int* nc;
};

template <int TB>
__device__ void rank_tail(const float* zl, int NP, const float* xn, const float* wn, int tb_n,
                          int64_t t0, int N, int k, int renorm, float gamma, int force_fp64,
                          const uint16_t* __restrict__ hidden, const double* __restrict__ residual,
                          const uint16_t* __restrict__ gate, int d, int32_t* __restrict__ topk_idx,
                          float* __restrict__ topk_w, double* ring64, const TailSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = (k < N) ? k : N - 1;          // last rank whose order must be certain
  const bool counting = tb_n * N <= 2 * kThreads;
  // (1) decode sizes: counting ranks, rank(j) = #{i : z_i > z_j or
  //     (z_i == z_j and i < j)}; only ranks <= kk are kept
  for (int p = tid; counting && p < tb_n * N; p += kThreads) {
    const int t = p / N, j = p - t * N;
    const float* z = zl + t * NP;
    const float zj = z[j];
    if (!(fabsf(zj) < 3.0e38f)) {
      sm.bad[t] = 1;
      continue;
    }
    // NP % 8 == 0, padded logits are never read past N: count in float4s
    const float4* z4 = reinterpret_cast<const float4*>(z);
    int r = 0;
#pragma unroll 4
    for (int i4 = 0; i4 < N / 4; ++i4) {
      const float4 v = z4[i4];
      const int i = 4 * i4;
      r += (v.x > zj) || (v.x == zj && i < j);
      r += (v.y > zj) || (v.y == zj && i + 1 < j);
      r += (v.z > zj) || (v.z == zj && i + 2 < j);
      r += (v.w > zj) || (v.w == zj && i + 3 < j);
    }
    if (r <= kk) sm.sel[t][r] = j;
  }
  // (1') larger tiles: k+1 warp-wide argmax rounds over (logit, -index)
  for (int t = warp; !counting && t < tb_n; t += kThreads / 32) {
    const float* z = zl + t * NP;
    float zq[8];
    unsigned taken = 0;
    bool nonfin = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int j = lane + 32 * q;
      zq[q] = (j < N) ? z[j] : -INFINITY;
      if (j >= N) taken |= 1u << q;
      else if (!(fabsf(zq[q]) < 3.0e38f)) nonfin = true;
    }
    if (__any_sync(0xffffffffu, nonfin)) {
      if (lane == 0) sm.bad[t] = 1;
      continue;
    }
    for (int r = 0; r <= kk; ++r) {
      float bv = -INFINITY;
      int bj = 0x7fffffff;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = lane + 32 * q;
        if (!(taken & (1u << q)) && (zq[q] > bv || (zq[q] == bv && j < bj))) {
          bv = zq[q];
          bj = j;
        }
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ov > bv || (ov == bv && oj < bj)) {
          bv = ov;
          bj = oj;
        }
      }
      if (lane == 0) sm.sel[t][r] = bj;
      if ((bj & 31) == lane) taken |= 1u << (bj >> 5);
    }
  }
  __syncthreads();
  // (2) certificate, softmax, outputs: one warp per token
  for (int t = warp; t < tb_n; t += kThreads / 32) {
    const float* z = zl + t * NP;
    const int* sel = sm.sel[t];
    if (sm.bad[t] || force_fp64) {
      if (lane == 0) {
        const int f = atomicAdd(sm.nflag, 1);
        sm.flag[f] = t;
        for (int q = 0; q < 8; ++q)
          sm.cmask[f][q] = (32 * q >= N) ? 0u : (N - 32 * q >= 32 ? 0xffffffffu
                                                                  : ((1u << (N - 32 * q)) - 1u));
      }
      __syncwarp();
      continue;
    }
    const float zr = (lane <= kk) ? z[sel[lane]] : 0.f;   // my rank's logit (lane r <= kk)
    const float z0 = __shfl_sync(0xffffffffu, zr, 0);
    const float zn = __shfl_down_sync(0xffffffffu, zr, 1);
    // certificate: every rank r <= kk clear of the fp64 softmax underflow
    // zone; gaps (r, r+1) for r < kk wider than both bounds
    int ok = 1;
    if (lane <= kk) {
      const int a = sel[lane];
      ok = (zr - z0 > -600.f);
      if (lane < kk) {
        const int b = sel[lane + 1];
        const float bnd = gamma * sqrtf(xn[t]) * (wn[a] + wn[b]) + 1e-30f;
        ok = ok && (zr - zn > bnd);
      }
    }
    const bool spread = __any_sync(0xffffffffu, lane <= kk && !(zr - z0 > -600.f));
    ok = __all_sync(0xffffffffu, ok);
    if (!ok) {
      // candidates: j with z_j + B_j >= L = min_{r<k} (z_r - B_r); every
      // expert when the row reaches the fp64 softmax underflow zone
      const float xnr = gamma * sqrtf(xn[t]);
      float lo = INFINITY;
      if (lane < k) lo = zr - (xnr * wn[sel[lane]] + 1e-30f);
#pragma unroll
      for (int o = 16; o; o >>= 1) lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      uint32_t words[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int j = lane + 32 * q;
        const bool in = j < N && (spread || z[j] + (xnr * wn[j] + 1e-30f) >= lo);
        words[q] = __ballot_sync(0xffffffffu, in);
      }
      if (lane == 0) {
        const int f = atomicAdd(sm.nflag, 1);
        sm.flag[f] = t;
        for (int q = 0; q < 8; ++q) sm.cmask[f][q] = words[q];
      }
      __syncwarp();
      continue;
    }
    float sum = 0.f;
    for (int j = lane; j < N; j += 32) sum += expf(z[j] - z0);
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    const int64_t tt = t0 + t;
    const float p = (lane < k) ? expf(zr - z0) / sum : 0.f;
    float tot = p;
#pragma unroll
    for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
    if (lane < k) {
      const int j = sel[lane];
      if (topk_idx) topk_idx[tt * k + lane] = j;
      if (topk_w) topk_w[tt * k + lane] = renorm ? p / tot : p;
      atomicAdd(&sm.hist[j], 1);
    }
    __syncwarp();
  }
  __syncthreads();
  RG_MARK(7);
  // (3) fp64 recompute of the uncertified rows (rare)
  const int nflag = *sm.nflag;
  for (int f = 0; f < nflag; ++f) {
    const int t = sm.flag[f];
    const int64_t tt = t0 + t;
    fp64_row_cand(hidden + tt * (int64_t)d, residual, gate, d, N, k, renorm, sm.cmask[f],
                  zl + t * NP, ring64, ring64 + d, sm.row64, sm.cl, sm.nc,
                  topk_idx ? topk_idx + tt * k : nullptr, topk_w ? topk_w + tt * k : nullptr,
                  sm.hist);
  }
  RG_MARK(8);
  if (tid == 0) {
    if (nflag) atomicAdd(&g_route_fires, (unsigned long long)nflag);
    atomicAdd(&g_route_rows, (unsigned long long)tb_n);
  }
  __syncthreads();
}

// Decode-sized batches: the routing plan and the permute of dali_moe_plan_permute
// (moe.cu plan_kernel: a stable counting sort of the T*k (token, slot) pairs
// by expert, then the 128-bit gather of the permuted rows) done by the CTA
// that owns the whole batch, right after its top-k -- one launch fewer on the
// decode critical path.  Same outputs: offsets (N+1), perm_token (T*k), pos
// (T, k), xp (T*k, d).
struct PlanOut {
  int32_t* offsets;
  int32_t* perm;
  int32_t* pos;
  uint16_t* xp;
};

__device__ void plan_gather(const PlanOut& plan, const int32_t* topk_idx,
                            const uint16_t* __restrict__ hidden, int T, int k, int N, int d,
                            const int* hist, int* scratch /* >= N + 1 + 256 ints */) {
  const int tid = threadIdx.x;
  const int R = T * k;
  int* offs = scratch;                     // N + 1
  int* perm = scratch + N + 1;             // R <= 256 - N - 1 by the host's guard
  if (tid == 0) {
    int run = 0;
    for (int e = 0; e < N; ++e) {
      offs[e] = run;
      run += hist[e];
    }
    offs[N] = run;
  }
  __syncthreads();                          // topk_idx rows written by this CTA are visible
  for (int e = tid; e <= N; e += kThreads) plan.offsets[e] = offs[e];
  for (int p = tid; p < R; p += kThreads) {
    const int e = topk_idx[p];
    int before = 0;                          // earlier pairs routed to the same expert
    for (int q = 0; q < p; ++q) before += topk_idx[q] == e;
    const int row = offs[e] + before;
    plan.pos[p] = row;
    plan.perm[row] = p / k;
    perm[row] = p / k;
  }
  __syncthreads();
  const int d8 = d >> 3;
  const uint4* src = reinterpret_cast<const uint4*>(hidden);
  uint4* dst = reinterpret_cast<uint4*>(plan.xp);
  for (int u = tid; u < R * d8; u += kThreads) {
    const int row = u / d8, c = u - row * d8;
    dst[u] = src[(int64_t)perm[row] * d8 + c];
  }
}

template <int TB, int C>
__global__ void __launch_bounds__(kThreads)
route_guard_kernel(const uint16_t* __restrict__ hidden, const double* __restrict__ residual,
                   const uint16_t* __restrict__ gate, int64_t T, int d, int N, int k,
                   int renorm, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                   unsigned long long* __restrict__ workloads,
                   const float* __restrict__ wnorm2, Geo g, float gamma, int force_fp64,
                   PlanOut plan) {
  RG_MARK(0);
  constexpr int TG = TB / 4;
  extern __shared__ __align__(16) unsigned char smem[];
  // [ring: kStages x kStageBytes (aliased by red after the main loop)]
  // [xs: TB x (DC + 4) f32] [gather: C x (TB*NP + TB + NP) f32 (C > 1)]
  unsigned char* ring = smem;
  float* xs = reinterpret_cast<float*>(smem + kStages * kStageBytes);
  const int xld = g.DC + 4;
  float* gath = xs + TB * xld;
  const int gsz = TB * g.NP + TB;

  __shared__ float sh_logit[TB * 64 > 4096 ? TB * 64 : 4096];   // TB x NP final logits
  __shared__ float sh_xn[TB], sh_wn[256];
  __shared__ float sh_red_xn[(kThreads / 32) * TB];
  __shared__ int sh_hist[256];
  __shared__ int sh_sel[TB][DALI_MAX_TOPK + 1];
  __shared__ int sh_bad[TB];
  __shared__ int sh_flag[TB];
  __shared__ int sh_nflag;
  __shared__ double sh_row64[256];
  __shared__ int sh_cl[256];
  __shared__ int sh_nc;
  __shared__ uint32_t sh_cmask[TB][8];

  const int tid = threadIdx.x;
  int crank = 0;
  if constexpr (C > 1) crank = (int)cg::this_cluster().block_rank();
  const int64_t t0 = (C > 1) ? 0 : (int64_t)blockIdx.x * TB;
  const int tb_n = (int)((T - t0 < TB) ? (T - t0) : TB);
  const int d0 = crank * g.ds, d1 = d0 + g.ds;
  const int nchunks = (g.ds + g.DC - 1) / g.DC;
  const int xraw_bytes = TB * g.DC * 2;

  for (int i = tid; i < N; i += kThreads) sh_hist[i] = 0;
  for (int i = tid; i < TB; i += kThreads) sh_bad[i] = 0;
  if (tid == 0) sh_nflag = 0;

  // stage issue: raw bf16 x rows [TB][DC] and the contiguous W rows [DC][N]
  auto issue_x = [&](int c, int slot) {
    unsigned char* st = ring + slot * kStageBytes;
    const int c0 = d0 + c * g.DC;
    const int upr = g.DC / 8;                        // 16-byte units per x row
    for (int u = tid; u < TB * upr; u += kThreads) {
      const int t = u / upr, q = u % upr;
      const int col = c0 + q * 8;
      const bool ok = (t < tb_n) && (col < d1);
      const uint16_t* src = ok ? hidden + (t0 + t) * (int64_t)d + col : hidden;
      cp_async16(st + u * 16, src, ok);
    }
  };
  auto issue_w = [&](int c, int slot) {
    unsigned char* st = ring + slot * kStageBytes;
    const int c0 = d0 + c * g.DC;
    const int wunits = g.DC * N / 8;
    const int64_t wbase = (int64_t)c0 * N;          // element offset, multiple of 8
    const int64_t wend = (int64_t)d1 * N;
    for (int u = tid; u < wunits; u += kThreads) {
      const int64_t el = wbase + (int64_t)u * 8;
      const bool ok = el < wend;
      cp_async16(st + xraw_bytes + u * 16, ok ? gate + el : gate, ok);
    }
  };
  auto issue = [&](int c, int slot) {
    issue_x(c, slot);
    issue_w(c, slot);
  };

  // register tile: tokens tg + TG*j (j < 4), experts eg*8 .. eg*8+7, d-slice s.
  // Warp mode (g.warp_mode: EG*TG divides 8): every warp owns one tile and
  // its 32 lanes are 32 consecutive slices, reduced by a shuffle transpose;
  // otherwise the tile index runs fastest and slices meet in shared memory.
  const int tile_threads = g.EG * TG;
  const int lane = tid & 31, wid = tid >> 5;
  int eg, tg, s;
  if (g.warp_mode) {
    const int tile_id = wid % tile_threads;
    eg = tile_id % g.EG;
    tg = tile_id / g.EG;
    s = (wid / tile_threads) * 32 + lane;
  } else {
    eg = tid % g.EG;
    tg = (tid / g.EG) % TG;
    s = tid / tile_threads;
  }
  const bool active = s < g.S;
  float acc[4][8], blk[4][8];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[j][e] = blk[j][e] = 0.f;

  // token-norm partials: token xt over columns xsub, xsub + 256/TB, ...
  const int x_per_tok = kThreads / TB;
  const int xt = tid % TB, xsub = tid / TB;
  float xn_p = 0.f;

  // the router (and its column norms, for the bound) never depends on the
  // previous kernel: request the first stages' router rows before the PDL
  // wait so they stream while the predecessor drains
  for (int c = 0; c < kStages - 1; ++c)
    if (c < nchunks) issue_w(c, c);
  const float wn2v = tid < N ? __ldg(wnorm2 + tid) : 0.f;
  DALI_PDL_ENTRY();
  for (int c = 0; c < kStages - 1; ++c) {
    if (c < nchunks) issue_x(c, c);
    cp_commit();
  }
  RG_MARK(1);
  for (int c = 0; c < nchunks; ++c) {
    cp_wait<kStages - 2>();
    __syncthreads();                                  // stage c landed; xs free
    if (c == 0) RG_MARK(2);
    const unsigned char* st = ring + (c % kStages) * kStageBytes;
    const uint16_t* xr = reinterpret_cast<const uint16_t*>(st);
    const uint16_t* wr = reinterpret_cast<const uint16_t*>(st + xraw_bytes);
    const int c0 = d0 + c * g.DC;
    // x: bf16 -> f32 (+ residual in fp64), token norms; 8 columns per unit
    for (int q8 = xsub; q8 < g.DC / 8; q8 += x_per_tok) {
      const uint4 raw = *reinterpret_cast<const uint4*>(xr + xt * g.DC + q8 * 8);
      float v[8];
      bf16x2_to_f32(raw.x, v[0], v[1]);
      bf16x2_to_f32(raw.y, v[2], v[3]);
      bf16x2_to_f32(raw.z, v[4], v[5]);
      bf16x2_to_f32(raw.w, v[6], v[7]);
      if (residual) {
        const int col = c0 + q8 * 8;
        if (col < d1) {
#pragma unroll
          for (int q = 0; q < 8; ++q) v[q] = (float)__dadd_rn((double)v[q], residual[col + q]);
        }
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) xn_p = fmaf(v[q], v[q], xn_p);
      float4* dst = reinterpret_cast<float4*>(xs + xt * xld + q8 * 8);
      dst[0] = make_float4(v[0], v[1], v[2], v[3]);
      dst[1] = make_float4(v[4], v[5], v[6], v[7]);
    }
    __syncthreads();
    // the next stage's loads go out before this stage's FFMAs
    if (c + kStages - 1 < nchunks) issue(c + kStages - 1, (c + kStages - 1) % kStages);
    cp_commit();
    if (active) {
      // one 32-term block per chunk at most (g.DC <= 32 * g.S), flushed below
      const int nq = g.DC / g.S;
#pragma unroll 4
      for (int q = 0; q < nq; ++q) {
        const int i = s + q * g.S;
        float w[8];
        const uint16_t* wp = wr + i * N + eg * 8;
        if ((N & 7) == 0) {
          const uint4 v = *reinterpret_cast<const uint4*>(wp);
          bf16x2_to_f32(v.x, w[0], w[1]);
          bf16x2_to_f32(v.y, w[2], w[3]);
          bf16x2_to_f32(v.z, w[4], w[5]);
          bf16x2_to_f32(v.w, w[6], w[7]);
        } else {
          const uint2 a = *reinterpret_cast<const uint2*>(wp);
          const uint2 b = *reinterpret_cast<const uint2*>(wp + 4);
          bf16x2_to_f32(a.x, w[0], w[1]);
          bf16x2_to_f32(a.y, w[2], w[3]);
          bf16x2_to_f32(b.x, w[4], w[5]);
          bf16x2_to_f32(b.y, w[6], w[7]);
        }
        float x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = xs[(tg + TG * j) * xld + i];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
          for (int e = 0; e < 8; ++e) blk[j][e] = fmaf(x[j], w[e], blk[j][e]);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 8; ++e) { acc[j][e] += blk[j][e]; blk[j][e] = 0.f; }
    }
  }
  cp_wait<0>();
  RG_MARK(3);
  __syncthreads();                         // ring free: reuse as the slice reduction buffer
  float* red = reinterpret_cast<float*>(ring);
  const int tile = TB * g.NP;
  // token norms: lanes sharing xt (xor offsets >= TB), then 8 warps in order
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1)
    if (m >= TB) xn_p += __shfl_xor_sync(0xffffffffu, xn_p, m);
  if (lane < TB) sh_red_xn[wid * TB + lane] = xn_p;
  if (g.warp_mode) {
    // 32 values (4 tokens x 8 experts) over 32 lanes: 5 butterfly rounds,
    // lane v ends with the warp's sum of value v; then the warps of a tile
    // (slice groups) meet in shared memory: red[sgroup][tile]
    float v[32];
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) v[j * 8 + e] = acc[j][e];
#pragma unroll
    for (int m = 16, n = 32; m >= 1; m >>= 1, n >>= 1) {
      const bool up = (lane & m) != 0;
#pragma unroll
      for (int q = 0; q < n / 2; ++q) {
        const float send = up ? v[q] : v[q + n / 2];
        const float keep = up ? v[q + n / 2] : v[q];
        v[q] = keep + __shfl_xor_sync(0xffffffffu, send, m);
      }
    }
    const int j = lane >> 3, e = lane & 7;
    red[(wid / tile_threads) * tile + (tg + TG * j) * g.NP + eg * 8 + e] = v[0];
  } else if (active) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e)
        red[s * tile + (tg + TG * j) * g.NP + eg * 8 + e] = acc[j][e];
  }
  __syncthreads();
  const int nred = g.warp_mode ? g.S / 32 : g.S;          // partial tiles left
  for (int half = nred >> 1; half >= 1; half >>= 1) {      // pairwise tree
    for (int i = tid; i < half * tile; i += kThreads) red[i] += red[i + half * tile];
    __syncthreads();
  }
  RG_MARK(4);
  float* part_logit = red;                 // [TB][NP]
  float part_xn = 0.f;
  if (tid < TB) {
    for (int q = 0; q < kThreads / 32; ++q) part_xn += sh_red_xn[q * TB + tid];
  }

  if constexpr (C > 1) {
    cg::cluster_group cl = cg::this_cluster();
    float* dst = cl.map_shared_rank(gath, 0) + crank * gsz;
    for (int i = tid; i < tile; i += kThreads) dst[i] = part_logit[i];
    if (tid < TB) dst[tile + tid] = part_xn;
    RG_MARK(5);
    cl.sync();
    RG_MARK(6);
    if (crank != 0) return;
    for (int i = tid; i < tile; i += kThreads) {
      float v = gath[i];
      for (int q = 1; q < C; ++q) v += gath[q * gsz + i];
      sh_logit[i] = v;
    }
    if (tid < TB) {
      float v = 0.f;
      for (int q = 0; q < C; ++q) v += gath[q * gsz + tile + tid];
      sh_xn[tid] = v;
    }
  } else {
    for (int i = tid; i < tile; i += kThreads) sh_logit[i] = part_logit[i];
    if (tid < TB) sh_xn[tid] = part_xn;
  }
  __syncthreads();

  if (tid < N) sh_wn[tid] = sqrtf(wn2v);
  __syncthreads();
  TailSmem tsm{sh_hist, sh_sel, sh_flag, &sh_nflag, sh_cmask, sh_bad, sh_row64, sh_cl, &sh_nc};
  rank_tail<TB>(sh_logit, g.NP, sh_xn, sh_wn, tb_n, t0, N, k, renorm, gamma, force_fp64, hidden,
                residual, gate, d, topk_idx, topk_w, reinterpret_cast<double*>(ring), tsm);
  if (workloads) {
    const bool single = (C > 1) || gridDim.x == 1;
    for (int i = tid; i < N; i += kThreads) {
      if (single) workloads[i] = (unsigned long long)sh_hist[i];
      else if (sh_hist[i]) atomicAdd(workloads + i, (unsigned long long)sh_hist[i]);
    }
  }
  if (plan.offsets) plan_gather(plan, topk_idx, hidden, tb_n, k, N, d, sh_hist, sh_cl);
}

// ---------------------------------------------------------------------------
// Prefill shape (T > 16, N <= 64): compile-time geometry.  CTA = TB tokens x
// NP (8 or 64, padded) experts over the whole of d; thread tile 4 tokens x
// 8 experts, S = 256 / (NP/8 * TB/4) d-slices.  Per chunk of DC router rows
// (2-stage cp.async ring of raw bf16) the CTA converts the router rows once
// to fp32 in a [half][row][expert-group][4] layout and the token rows to a
// transposed fp32 [row][token] tile, so the inner step is three 16-byte
// shared loads and 32 FFMAs with no per-step conversion or runtime index
// math.  Summation: KQ-term blocks per chunk flushed into an outer
// accumulator, pairwise slice tree -- the same certified-height argument
// and rank_tail as the decode shape.
template <int TB, int NP>
struct PCfg {
  static constexpr int EG = NP / 8, TG = TB / 4, TT = EG * TG, S = kThreads / TT;
  static constexpr int row_bytes = (NP + TB) * 2;
  static constexpr int KQ = (S * 16 * row_bytes <= 24576) ? 16
                            : (S * 8 * row_bytes <= 24576) ? 8 : 4;
  static constexpr int DC = S * KQ;
  static constexpr int STG = DC * row_bytes;            // raw: W [DC][N] then x [DC/8][TB][8]
  static constexpr int WF = DC * NP * 4, XF = DC * TB * 4;
  static constexpr int UNITS = TB * DC / 8;             // x 16-byte units per chunk
  static constexpr int XR = (UNITS + kThreads - 1) / kThreads;
  static constexpr int TILE = TB * NP;
  static constexpr int RED = S * TILE * 4;
  static constexpr int MAIN = (2 * STG + WF + XF) > RED ? (2 * STG + WF + XF) : RED;
  static constexpr int SMEM = MAIN + TILE * 4 + kThreads * 4;
  static_assert(TT <= kThreads && S * TT == kThreads, "tile threads");
  static_assert(KQ <= 32, "block height");
};

template <int TB, int NP>
__global__ void __launch_bounds__(kThreads, 2)
route_prefill_kernel(const uint16_t* __restrict__ hidden, const double* __restrict__ residual,
                     const uint16_t* __restrict__ gate, int64_t T, int d, int N, int k,
                     int renorm, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
                     unsigned long long* __restrict__ workloads,
                     const float* __restrict__ wnorm2, float gamma, int force_fp64) {
  using P = PCfg<TB, NP>;
  constexpr int DC = P::DC, S = P::S, EG = P::EG, TG = P::TG, KQ = P::KQ;
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* ring = smem;                                   // 2 x STG raw stages
  float* wF = reinterpret_cast<float*>(smem + 2 * P::STG);     // [2][DC][EG][4]
  float* xT = wF + DC * NP;                                     // [DC][TB]
  float* logit = reinterpret_cast<float*>(smem + P::MAIN);      // [TB][NP]
  float* xnu = logit + P::TILE;                                 // [kThreads] norm partials

  __shared__ float sh_xn[TB], sh_wn[256];
  __shared__ int sh_hist[256];
  __shared__ int sh_sel[TB][DALI_MAX_TOPK + 1];
  __shared__ int sh_bad[TB];
  __shared__ int sh_flag[TB];
  __shared__ int sh_nflag;
  __shared__ double sh_row64[256];
  __shared__ int sh_cl[256];
  __shared__ int sh_nc;
  __shared__ uint32_t sh_cmask[TB][8];

  const int tid = threadIdx.x;
  const int64_t t0 = (int64_t)blockIdx.x * TB;
  const int tb_n = (int)((T - t0 < TB) ? (T - t0) : TB);
  const int nchunks = (d + DC - 1) / DC;
  for (int i = tid; i < N; i += kThreads) sh_hist[i] = 0;
  for (int i = tid; i < TB; i += kThreads) sh_bad[i] = 0;
  if (tid == 0) sh_nflag = 0;

  auto issue_w = [&](int c) {
    unsigned char* st = ring + (c & 1) * P::STG;
    const int64_t wbase = (int64_t)c * DC * N, wend = (int64_t)d * N;
    for (int u = tid; u < DC * N / 8; u += kThreads) {
      const int64_t el = wbase + (int64_t)u * 8;
      cp_async16(st + u * 16, el < wend ? gate + el : gate, el < wend);
    }
  };
  auto issue_x = [&](int c) {
    unsigned char* st = ring + (c & 1) * P::STG + DC * N * 2;
    for (int u = tid; u < P::UNITS; u += kThreads) {
      const int t = u % TB, q8 = u / TB;                    // unit-major: [q8][t]
      const int col = c * DC + q8 * 8;
      const bool ok = t < tb_n && col < d;
      cp_async16(st + u * 16, ok ? hidden + (t0 + t) * (int64_t)d + col : hidden, ok);
    }
  };

  const int eg = tid % EG, tg = (tid / EG) % TG, s = tid / P::TT;
  float acc[4][8], blk[4][8];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[j][e] = 0.f;
  float xn_p = 0.f;                                 // token tid % TB (units u = tid + 256 r)

  issue_w(0);                                       // the router does not depend on the predecessor
  const float wn2v = tid < N ? __ldg(wnorm2 + tid) : 0.f;
  DALI_PDL_ENTRY();
  issue_x(0);
  cp_commit();
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      issue_w(c + 1);
      issue_x(c + 1);
    }
    cp_commit();
    cp_wait<1>();
    __syncthreads();                                // chunk c landed everywhere; fp32 tiles free
    const unsigned char* st = ring + (c & 1) * P::STG;
    {   // router rows -> fp32 [half][row][eg][4], padded experts zero
      const uint16_t* wr = reinterpret_cast<const uint16_t*>(st);
      if ((N & 7) == 0) {
        for (int u = tid; u < DC * N / 8; u += kThreads) {
          const int i = u / (N / 8), g8 = u - i * (N / 8);
          const uint4 raw = *reinterpret_cast<const uint4*>(wr + u * 8);
          float v[8];
          bf16x2_to_f32(raw.x, v[0], v[1]);
          bf16x2_to_f32(raw.y, v[2], v[3]);
          bf16x2_to_f32(raw.z, v[4], v[5]);
          bf16x2_to_f32(raw.w, v[6], v[7]);
          *reinterpret_cast<float4*>(wF + (i * EG + g8) * 4) = make_float4(v[0], v[1], v[2], v[3]);
          *reinterpret_cast<float4*>(wF + ((DC + i) * EG + g8) * 4) =
              make_float4(v[4], v[5], v[6], v[7]);
        }
        if (N < NP) {
          for (int u = tid; u < DC * (NP - N) / 8; u += kThreads) {
            const int i = u / ((NP - N) / 8), g8 = N / 8 + u % ((NP - N) / 8);
            *reinterpret_cast<float4*>(wF + (i * EG + g8) * 4) = make_float4(0.f, 0.f, 0.f, 0.f);
            *reinterpret_cast<float4*>(wF + ((DC + i) * EG + g8) * 4) =
                make_float4(0.f, 0.f, 0.f, 0.f);
          }
        }
      } else if ((N & 3) == 0) {                    // 4-element units never straddle rows
        for (int u = tid; u < DC * N / 4; u += kThreads) {
          const int i = u / (N / 4), j = (u - i * (N / 4)) * 4;
          const uint2 raw = *reinterpret_cast<const uint2*>(wr + u * 4);
          float v[4];
          bf16x2_to_f32(raw.x, v[0], v[1]);
          bf16x2_to_f32(raw.y, v[2], v[3]);
          *reinterpret_cast<float4*>(wF + (((j >> 2) & 1) * DC + i) * (NP / 2) + (j >> 3) * 4) =
              make_float4(v[0], v[1], v[2], v[3]);
        }
        for (int u = tid; u < DC * (NP - N) / 4; u += kThreads) {
          const int i = u / ((NP - N) / 4), j = N + (u % ((NP - N) / 4)) * 4;
          *reinterpret_cast<float4*>(wF + (((j >> 2) & 1) * DC + i) * (NP / 2) + (j >> 3) * 4) =
              make_float4(0.f, 0.f, 0.f, 0.f);
        }
      } else {
        for (int u = tid; u < DC * NP; u += kThreads) {
          const int i = u / NP, j = u - i * NP;
          const float v = j < N ? __uint_as_float((uint32_t)wr[i * N + j] << 16) : 0.f;
          wF[(((j >> 2) & 1) * DC + i) * NP / 2 + (j >> 3) * 4 + (j & 3)] = v;
        }
      }
    }
    {   // token rows -> fp32 transposed [row][token] (+ residual in fp64), norms
      const uint16_t* xr = reinterpret_cast<const uint16_t*>(st + DC * N * 2);
#pragma unroll
      for (int r = 0; r < P::XR; ++r) {
        const int u = tid + r * kThreads;
        if (u < P::UNITS) {
          const int t = u % TB, q8 = u / TB;
          const uint4 raw = *reinterpret_cast<const uint4*>(xr + u * 8);
          float v[8];
          bf16x2_to_f32(raw.x, v[0], v[1]);
          bf16x2_to_f32(raw.y, v[2], v[3]);
          bf16x2_to_f32(raw.z, v[4], v[5]);
          bf16x2_to_f32(raw.w, v[6], v[7]);
          const int col = c * DC + q8 * 8;
          if (residual && col < d) {
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = (float)__dadd_rn((double)v[q], residual[col + q]);
          }
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            xn_p = fmaf(v[q], v[q], xn_p);
            xT[(q8 * 8 + q) * TB + t] = v[q];
          }
        }
      }
    }
    __syncthreads();
    // KQ-term block: rows i = s + q*S of this chunk
    const float* wa = wF + eg * 4;
    const float* wb = wF + DC * NP / 2 + eg * 4;
    const float* xa = xT + tg * 4;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) blk[j][e] = 0.f;
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      const int i = s + q * S;
      const float4 w0 = *reinterpret_cast<const float4*>(wa + i * (NP / 2));
      const float4 w1 = *reinterpret_cast<const float4*>(wb + i * (NP / 2));
      const float4 xv = *reinterpret_cast<const float4*>(xa + i * TB);
      const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
      const float x[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int e = 0; e < 8; ++e) blk[j][e] = fmaf(x[j], w[e], blk[j][e]);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[j][e] += blk[j][e];
  }
  cp_wait<0>();
  __syncthreads();                                  // ring + fp32 tiles free: slice partials
  float* red = reinterpret_cast<float*>(smem);      // [S][TB][NP]
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float* dst = red + s * P::TILE + (tg * 4 + j) * NP + eg * 8;
    *reinterpret_cast<float4*>(dst) = make_float4(acc[j][0], acc[j][1], acc[j][2], acc[j][3]);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(acc[j][4], acc[j][5], acc[j][6], acc[j][7]);
  }
  xnu[tid] = xn_p;
  __syncthreads();
  for (int half = S >> 1; half >= 1; half >>= 1) {  // pairwise slice tree
    for (int i = tid; i < half * P::TILE; i += kThreads) red[i] += red[i + half * P::TILE];
    __syncthreads();
  }
  for (int i = tid; i < P::TILE; i += kThreads) logit[i] = red[i];
  if (tid < TB) {
    float v = 0.f;
    for (int q = tid; q < kThreads; q += TB) v += xnu[q];
    sh_xn[tid] = v;
  }
  if (tid < N) sh_wn[tid] = sqrtf(wn2v);
  __syncthreads();
  TailSmem tsm{sh_hist, sh_sel, sh_flag, &sh_nflag, sh_cmask, sh_bad, sh_row64, sh_cl, &sh_nc};
  rank_tail<TB>(logit, NP, sh_xn, sh_wn, tb_n, t0, N, k, renorm, gamma, force_fp64, hidden,
                residual, gate, d, topk_idx, topk_w, reinterpret_cast<double*>(smem), tsm);
  if (workloads) {
    for (int i = tid; i < N; i += kThreads) {
      if (gridDim.x == 1) workloads[i] = (unsigned long long)sh_hist[i];
      else if (sh_hist[i]) atomicAdd(workloads + i, (unsigned long long)sh_hist[i]);
    }
  }
}

static int ilog2(int x) { int r = 0; while ((1 << (r + 1)) <= x) ++r; return r; }

static Geo make_geo(int TB, int N, int C, int d) {
  Geo g{};
  g.TB = TB;
  g.NP = (N + 7) / 8 * 8;
  g.EG = g.NP / 8;
  g.TG = TB / 4;
  int s = kThreads / (g.EG * g.TG);
  g.S = s >= 1 ? (1 << ilog2(s)) : 0;
  g.warp_mode = (8 % (g.EG * g.TG)) == 0;                  // one tile per warp
  if (g.warp_mode) g.S = (8 / (g.EG * g.TG)) * 32;
  g.logS = g.S ? ilog2(g.S) : 0;
  g.C = C;
  g.ds = d / C;
  // chunk: as many d-rows as fit one stage, a multiple of max(S, 8)
  const int per_row = TB * 2 + N * 2;
  int dc = kStageBytes / per_row;
  const int m = g.S > 8 ? g.S : 8;
  dc = dc / m * m;
  const int cap = (g.ds + m - 1) / m * m;
  if (dc > cap) dc = cap;
  if (dc > 32 * g.S) dc = 32 * g.S / m * m;          // <= 32 terms per thread per chunk
  g.DC = dc;
  return g;
}

static size_t smem_bytes(const Geo& g) {
  size_t b = (size_t)kStages * kStageBytes + (size_t)g.TB * (g.DC + 4) * 4;
  if (g.C > 1) b += (size_t)g.C * (g.TB * g.NP + g.TB) * 4;
  return b;
}

static double s_guard_scale = 1.0;          // test hook: < 0 forces every row to fp64
static int s_prefill_variant = 0;           // A/B hook: 0 auto, 1 chunked, 2 fixed-geometry

template <int TB, int C>
static int launch_tb(const uint16_t* hidden, const double* residual, const uint16_t* gate,
                     int64_t T, int d, int N, int k, int renorm, int32_t* idx, float* w,
                     unsigned long long* wl, const float* wn2, cudaStream_t st, const Geo& g,
                     PlanOut plan = PlanOut{nullptr, nullptr, nullptr, nullptr}) {
  const size_t sm = smem_bytes(g);
  DALI_ONCE_PER_DEVICE(cudaFuncSetAttribute(route_guard_kernel<TB, C>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            180 * 1024));
  // summation height: one block of DC/S terms per chunk, one flush per chunk,
  // slice tree, cluster sum, and one for a rounded (residual-shifted) input
  const int nch = (g.ds + g.DC - 1) / g.DC;
  const int H = g.DC / g.S + nch + g.logS + (C - 1) + 1;
  const double u = 1.0 / (1 << 24);
  double gam = H * u / (1.0 - H * u) + (residual ? 2 * u : 0.0) + 1e-12;
  gam *= 1.01 * (s_guard_scale > 0 ? s_guard_scale : 1.0);
  const int force = s_guard_scale < 0;
  const unsigned grid = C > 1 ? (unsigned)C : (unsigned)((T + TB - 1) / TB);
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attrs[0].val.programmaticStreamSerializationAllowed = 1;
  int na = 1;
  if (C > 1) {
    attrs[1].id = cudaLaunchAttributeClusterDimension;
    attrs[1].val.clusterDim.x = C;
    attrs[1].val.clusterDim.y = 1;
    attrs[1].val.clusterDim.z = 1;
    na = 2;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sm;
  cfg.stream = st;
  cfg.attrs = attrs;
  cfg.numAttrs = na;
  cudaLaunchKernelEx(&cfg, route_guard_kernel<TB, C>, hidden, residual, gate, T, d, N, k, renorm,
                     idx, w, wl, wn2, g, (float)gam, force, plan);
  DALI_LAUNCH_CHECK("route_guard_kernel");
  return DALI_OK;
}

template <int TB, int NP>
static int launch_prefill(const uint16_t* hidden, const double* residual, const uint16_t* gate,
                          int64_t T, int d, int N, int k, int renorm, int32_t* idx, float* w,
                          unsigned long long* wl, const float* wn2, cudaStream_t st) {
  using P = PCfg<TB, NP>;
  if ((size_t)(d + 1040) * 8 > (size_t)P::MAIN) return 1;     // fp64 scratch: chunked kernel
  DALI_ONCE_PER_DEVICE(cudaFuncSetAttribute(route_prefill_kernel<TB, NP>,
                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                            P::SMEM));
  // summation height: a KQ-term block per chunk, one flush per chunk, the
  // slice tree, and one for a rounded (residual-shifted) input
  const int nch = (d + P::DC - 1) / P::DC;
  const int H = P::KQ + nch + ilog2(P::S) + 1;
  const double u = 1.0 / (1 << 24);
  double gam = H * u / (1.0 - H * u) + (residual ? 2 * u : 0.0) + 1e-12;
  gam *= 1.01 * (s_guard_scale > 0 ? s_guard_scale : 1.0);
  const int force = s_guard_scale < 0;
  const unsigned grid = (unsigned)((T + TB - 1) / TB);
  if (wl && grid > 1) cudaMemsetAsync(wl, 0, sizeof(int64_t) * N, st);
  launch_pdl(route_prefill_kernel<TB, NP>, dim3(grid), dim3(kThreads), (size_t)P::SMEM, st,
             hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, (float)gam, force);
  DALI_LAUNCH_CHECK("route_prefill_kernel");
  return DALI_OK;
}

}  // namespace rg

// Returns 1 if launched (or T == 0 handled), 0 if the shape is not eligible
// (caller falls back to the fp64 kernel), < 0 / error code on failure.
int launch_route_guarded(const uint16_t* hidden, const double* residual, const uint16_t* gate,
                         const float* wn2, int64_t T, int d, int N, int k, int renorm,
                         int32_t* idx, float* w, int64_t* workloads, void* stream,
                         int* launched, const int32_t* const* plan_ptrs, uint16_t* plan_xp) {
  using namespace rg;
  PlanOut plan{nullptr, nullptr, nullptr, nullptr};
  if (plan_ptrs) {
    // only the single-CTA-owner shape (T <= 16) plans in-kernel, and only
    // when the pairs fit the scratch; the caller plans separately otherwise
    if (T > 16 || idx == nullptr || T * k + N + 1 > 256 || (d & 7)) return DALI_OK;
    plan = PlanOut{const_cast<int32_t*>(plan_ptrs[0]), const_cast<int32_t*>(plan_ptrs[1]),
                   const_cast<int32_t*>(plan_ptrs[2]), plan_xp};
  }
  *launched = 0;
  // d <= 8000: the fp64 recompute stages one row (d doubles) in the 72 KB ring
  if (wn2 == nullptr || d > 8000 || N < 4 || N > 256 || (N & 3) || (d & 7) || k > DALI_MAX_TOPK || k > N || T <= 0)
    return DALI_OK;
  cudaStream_t st = as_stream(stream);
  auto* wl = reinterpret_cast<unsigned long long*>(workloads);
  int rc = 1;                                   // 1: not launched yet
  if (T <= 16) {
    int C = 8;
    while (C > 1 && (d % (C * 8) || d / C < 256)) C >>= 1;
    const int TB = T <= 4 ? 4 : T <= 8 ? 8 : 16;
    const Geo g = make_geo(TB, N, C, d);
    if (g.S < 1 || smem_bytes(g) > 180 * 1024 || (size_t)TB * g.NP > 4096) return DALI_OK;
#define DALI_RG_SMALL(TBv)                                                              \
  (C == 8 ? launch_tb<TBv, 8>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g, plan) \
   : C == 4 ? launch_tb<TBv, 4>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g, plan) \
   : C == 2 ? launch_tb<TBv, 2>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g, plan) \
            : launch_tb<TBv, 1>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g, plan))
    rc = TB == 4 ? DALI_RG_SMALL(4) : TB == 8 ? DALI_RG_SMALL(8) : DALI_RG_SMALL(16);
#undef DALI_RG_SMALL
  } else if (N <= 64 && s_prefill_variant != 1 &&
             (s_prefill_variant == 2 || T >= ((N <= 8 || (N & 7)) ? 2048 : 1024))) {
    // measured (tools/prof_route.py, profiles/r02_route_prefill.txt): 10-25%
    // faster from ~1k tokens (2k at N <= 8, where each token element feeds
    // only 8 FMAs and the fp32 staging costs about what it saves, and at
    // N % 8 != 0, whose router rows convert in 4-element units); below that
    // the chunked kernel's shorter chunk chain per CTA wins
    int TB = 4;
    while (TB < 32 && (T + TB - 1) / TB > 2 * 148) TB <<= 1;   // up to 2 CTAs per SM
#define DALI_RG_PRE(TBv) (N <= 8 ? launch_prefill<TBv, 8>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st) \
                         : launch_prefill<TBv, 64>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st))
    rc = TB == 4 ? DALI_RG_PRE(4) : TB == 8 ? DALI_RG_PRE(8) : TB == 16 ? DALI_RG_PRE(16)
                                                               : DALI_RG_PRE(32);
#undef DALI_RG_PRE
  }
  if (T > 16 && rc == 1) {
    int TB = 4;
    while (TB < 32 && (T + TB - 1) / TB > 2 * 148) TB <<= 1;   // up to 2 CTAs per SM
    const Geo g = make_geo(TB, N, 1, d);
    if (g.S < 1 || smem_bytes(g) > 180 * 1024 || (size_t)TB * g.NP > 4096) return DALI_OK;
    if (workloads && (T + TB - 1) / TB > 1) {
      cudaMemsetAsync(workloads, 0, sizeof(int64_t) * N, st);
    }
    rc = TB == 4    ? launch_tb<4, 1>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g)
         : TB == 8  ? launch_tb<8, 1>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g)
         : TB == 16 ? launch_tb<16, 1>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g)
                    : launch_tb<32, 1>(hidden, residual, gate, T, d, N, k, renorm, idx, w, wl, wn2, st, g);
  }
  if (rc == DALI_OK) *launched = 1;
  return rc;
}

}  // namespace dali

extern "C" int dali_route_guard_scale(double scale) {
  dali::rg::s_guard_scale = scale;
  return DALI_OK;
}

extern "C" int dali_route_prefill_variant(int32_t variant) {
  dali::rg::s_prefill_variant = variant;
  return DALI_OK;
}

extern "C" int dali_route_fire_count(uint64_t* fires, uint64_t* rows, int32_t reset) {
  unsigned long long f = 0, r = 0;
  cudaError_t e = cudaMemcpyFromSymbol(&f, dali::g_route_fires, sizeof(f));
  if (e == cudaSuccess) e = cudaMemcpyFromSymbol(&r, dali::g_route_rows, sizeof(r));
  if (e == cudaSuccess && reset) {
    const unsigned long long z = 0;
    e = cudaMemcpyToSymbol(dali::g_route_fires, &z, sizeof(z));
    if (e == cudaSuccess) e = cudaMemcpyToSymbol(dali::g_route_rows, &z, sizeof(z));
  }
  if (e != cudaSuccess) {
    dali::set_error("dali_route_fire_count: %s", cudaGetErrorString(e));
    return DALI_ECUDA;
  }
  if (fires) *fires = f;
  if (rows) *rows = r;
  return DALI_OK;
}

#ifdef DALI_RG_PROF
extern "C" int dali_rg_prof(uint64_t* out) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, dali::g_rg_prof, sizeof(unsigned long long) * 8 * 12);
  return DALI_OK;
}
#endif
