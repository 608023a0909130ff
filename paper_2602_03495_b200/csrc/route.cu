// (1) Gating: fused gate projection + fp64 softmax + stable top-k + workload
// histogram.  Restates derive_workloads (reference trace.py:229-265) and the
// residual shift of predict_next_layer (prefetch.py:127-136).
//
// Layout: one CTA handles TB consecutive tokens.  The (TB x CH) hidden chunk
// is staged into shared memory in fp64 (with the residual added once, the
// same rounding as numpy's `hidden + res`), then thread (e, s) accumulates
// logits of expert e over the d-slice s, s+S, ... (S = blockDim / N).
// Partial sums are reduced in a fixed order (deterministic), one warp per
// token computes the softmax and the stable rank of every expert, and the
// histogram is built with shared-memory atomics, then one global atomic per
// (CTA, expert).
#include "common.cuh"

namespace dali {

// threads per CTA are a template parameter: 256 for token batches, up to
// 1024 when one CTA carries a single decode token (more d-slices in flight)
// tokens per CTA (TB <= warps per CTA) is a template parameter: 8 for long
// prompts, fewer when T is small so the grid still covers the SMs.
// hidden chunk staged per iteration: as much of the CTA's rows as fits the
// 64 KB staging budget (decode: the whole row in one pass, so the loop is not
// a chain of global-load latencies).  Always a multiple of S = 256 / N's
// largest value (256), so every thread visits its d-slice in the same order
// whatever the chunking (bit-identical sums).
constexpr int kRouteStageBytes = 64 * 1024;
template <int TB> constexpr int route_ch() { return kRouteStageBytes / (8 * TB); }

template <typename TH, typename TW, int kRouteTB, int kRouteThreads>
__global__ void __launch_bounds__(kRouteThreads)
route_kernel(const TH* __restrict__ hidden, const double* __restrict__ residual,
             const TW* __restrict__ gate, int64_t T, int d, int N, int k,
             int renorm, int32_t* __restrict__ topk_idx, float* __restrict__ topk_w,
             unsigned long long* __restrict__ workloads, double* __restrict__ probs) {
  DALI_PDL_ENTRY();
  constexpr int kRouteCH = route_ch<kRouteTB>();
  __shared__ double sh_red[kRouteTB * DALI_MAX_EXPERTS];   // logits, then probs
  __shared__ int sh_hist[DALI_MAX_EXPERTS];
  __shared__ int sh_sel[kRouteTB][DALI_MAX_TOPK];
  extern __shared__ double sh_dyn[];
  double (*sh_h)[kRouteCH] = reinterpret_cast<double (*)[kRouteCH]>(sh_dyn);   // [TB][CH]
  double* sh_part = sh_dyn + kRouteTB * kRouteCH;                              // [TB][N][S]

  const int tid = threadIdx.x;
  const int S = kRouteThreads / N;                          // >= 1 (N <= 256)
  const int e = tid % N;
  const int s = tid / N;
  const bool active = s < S;
  const int64_t t0 = (int64_t)blockIdx.x * kRouteTB;
  const int tb_n = (T - t0 < kRouteTB) ? (int)(T - t0) : kRouteTB;

  for (int i = tid; i < N; i += kRouteThreads) sh_hist[i] = 0;

  double acc[kRouteTB];
#pragma unroll
  for (int j = 0; j < kRouteTB; ++j) acc[j] = 0.0;

  for (int c0 = 0; c0 < d; c0 += kRouteCH) {
    const int cn = min(kRouteCH, d - c0);
    __syncthreads();
    // stage the chunk: batches of 8 independent loads per thread so the
    // global-load latency is paid once per batch, not once per element
    constexpr int kBatch = 8;
    const int n_el = kRouteTB * kRouteCH;
    for (int base = tid; base < n_el; base += kRouteThreads * kBatch) {
      double v[kBatch];
#pragma unroll
      for (int q = 0; q < kBatch; ++q) {
        const int idx = base + q * kRouteThreads;
        const int tb = idx / kRouteCH, i = idx % kRouteCH;
        v[q] = 0.0;
        if (idx < n_el && tb < tb_n && i < cn) {
          v[q] = to_f64(hidden[(t0 + tb) * (int64_t)d + c0 + i]);
          if (residual) v[q] = __dadd_rn(v[q], residual[c0 + i]);
        }
      }
#pragma unroll
      for (int q = 0; q < kBatch; ++q) {
        const int idx = base + q * kRouteThreads;
        if (idx < n_el) sh_h[idx / kRouteCH][idx % kRouteCH] = v[q];
      }
    }
    __syncthreads();
    if (active) {
#pragma unroll 8
      for (int i = s; i < cn; i += S) {
        const double w = to_f64(gate[(int64_t)(c0 + i) * N + e]);
#pragma unroll
        for (int j = 0; j < kRouteTB; ++j) acc[j] = fma(sh_h[j][i], w, acc[j]);
      }
    }
  }
  if (active) {
#pragma unroll
    for (int j = 0; j < kRouteTB; ++j) sh_part[(j * N + e) * S + s] = acc[j];
  }
  __syncthreads();
  for (int idx = tid; idx < kRouteTB * N; idx += kRouteThreads) {
    double v = 0.0;
    const double* p = sh_part + idx * S;
    for (int q = 0; q < S; ++q) v += p[q];
    sh_red[idx] = v;
  }
  __syncthreads();

  // One warp per token: softmax (max-shifted, fp64) and stable ranks.
  const int warp = tid >> 5, lane = tid & 31;
  if (warp < tb_n) {
    double* row = sh_red + warp * N;
    double mx = -INFINITY;
    for (int j = lane; j < N; j += 32) mx = fmax(mx, row[j]);
    for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    double sum = 0.0;
    for (int j = lane; j < N; j += 32) {
      const double ex = exp(row[j] - mx);
      row[j] = ex;
      sum += ex;
    }
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    __syncwarp();
    for (int j = lane; j < N; j += 32) row[j] = row[j] / sum;
    __syncwarp();
    const int64_t t = t0 + warp;
    if (probs)
      for (int j = lane; j < N; j += 32) probs[t * N + j] = row[j];
    for (int j = lane; j < N; j += 32) {
      const double pj = row[j];
      int rank = 0;
      for (int q = 0; q < N; ++q) {
        const double pq = row[q];
        rank += (pq > pj) || (pq == pj && q < j);
      }
      if (rank < k) {
        sh_sel[warp][rank] = j;
        if (topk_idx) topk_idx[t * k + rank] = j;
        atomicAdd(&sh_hist[j], 1);
      }
    }
    __syncwarp();
    if (topk_w && lane == 0) {
      // Selected probabilities in rank order; optional renormalisation
      // (sequential sum over the k selected, rank order).
      double tot = 0.0;
      for (int r = 0; r < k; ++r) tot += row[sh_sel[warp][r]];
      for (int r = 0; r < k; ++r) {
        const double p = row[sh_sel[warp][r]];
        topk_w[t * k + r] = (float)(renorm ? p / tot : p);
      }
    }
  }
  __syncthreads();
  if (workloads) {
    if (gridDim.x == 1) {          // single CTA: the histogram is the result (no zeroing pass)
      for (int i = tid; i < N; i += kRouteThreads)
        workloads[i] = (unsigned long long)sh_hist[i];
    } else {
      for (int i = tid; i < N; i += kRouteThreads)
        if (sh_hist[i]) atomicAdd(workloads + i, (unsigned long long)sh_hist[i]);
    }
  }
}

__global__ void zero_i64(int64_t* p, int n) {
  DALI_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = 0;
}

template <typename TH, typename TW>
static int launch_route(const TH* hidden, const double* residual, const TW* gate,
                        int64_t T, int32_t d, int32_t N, int32_t k, int32_t renorm,
                        int32_t* topk_idx, float* topk_w, int64_t* workloads,
                        void* stream, double* probs = nullptr) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_ETRACE,
               "num experts %d outside [1, %d]", N, DALI_MAX_EXPERTS);
  DALI_REQUIRE(k >= 1 && k <= N, DALI_ETRACE, "top_k %d out of range for %d experts", k, N);
  DALI_REQUIRE(k <= DALI_MAX_TOPK, DALI_ETRACE, "top_k %d exceeds %d", k, DALI_MAX_TOPK);
  DALI_REQUIRE(d >= 1 && T >= 0, DALI_ETRACE, "bad shape T=%lld d=%d", (long long)T, d);
  DALI_REQUIRE(workloads != nullptr || probs != nullptr, DALI_ETRACE,
               "workloads output required");
  cudaStream_t st = as_stream(stream);
  if (workloads && (T > 2 || T == 0)) {   // 1 <= T <= 2: one CTA writes the histogram
    launch_pdl(zero_i64, dim3((N + 255) / 256), dim3(256), 0, st, workloads, N);
    DALI_LAUNCH_CHECK("zero_i64");
  }
  if (T == 0) return DALI_OK;
  DALI_REQUIRE((T + 1) / 2 < (1ll << 31), DALI_ETRACE, "too many tokens");
  // dynamic smem = staged hidden rows (64 KB) + partial logits (TB*N*S doubles)
  DALI_ONCE_PER_DEVICE({
    cudaFuncSetAttribute(route_kernel<TH, TW, 8, 256>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRouteStageBytes + 8 * 8 * 256);
    cudaFuncSetAttribute(route_kernel<TH, TW, 4, 256>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRouteStageBytes + 8 * 4 * 256);
    cudaFuncSetAttribute(route_kernel<TH, TW, 2, 512>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRouteStageBytes + 8 * 2 * 512);
    cudaFuncSetAttribute(route_kernel<TH, TW, 1, 1024>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kRouteStageBytes + 8 * 1 * 1024);
  });
  auto* ul = reinterpret_cast<unsigned long long*>(workloads);
  if (T >= 8 * 148) {
    launch_pdl(route_kernel<TH, TW, 8, 256>, dim3((unsigned)((T + 7) / 8)), dim3(256), kRouteStageBytes + sizeof(double) * 8 * N * (256 / N), st, 
        hidden, residual, gate, T, d, N, k, renorm, topk_idx, topk_w, ul, probs);
  } else if (T >= 4 * 148) {
    launch_pdl(route_kernel<TH, TW, 4, 256>, dim3((unsigned)((T + 3) / 4)), dim3(256), kRouteStageBytes + sizeof(double) * 4 * N * (256 / N), st, 
        hidden, residual, gate, T, d, N, k, renorm, topk_idx, topk_w, ul, probs);
  } else if (T > 1) {
    launch_pdl(route_kernel<TH, TW, 2, 512>, dim3((unsigned)((T + 1) / 2)), dim3(512), kRouteStageBytes + sizeof(double) * 2 * N * (512 / N), st, 
        hidden, residual, gate, T, d, N, k, renorm, topk_idx, topk_w, ul, probs);
  } else {
    launch_pdl(route_kernel<TH, TW, 1, 1024>, dim3(1u), dim3(1024), kRouteStageBytes + sizeof(double) * N * (1024 / N), st, 
        hidden, residual, gate, T, d, N, k, renorm, topk_idx, topk_w, ul, probs);
  }
  DALI_LAUNCH_CHECK("route_kernel");
  return DALI_OK;
}

// Stable top-P of predicted workloads (prefetch.py:153-156): rank by
// (-value, index).
__global__ void prefetch_select_kernel(const int64_t* __restrict__ pred, int N, int P,
                                       int32_t* __restrict__ set) {
  for (int j = threadIdx.x; j < N; j += blockDim.x) {
    const int64_t v = pred[j];
    int rank = 0;
    for (int q = 0; q < N; ++q) rank += (pred[q] > v) || (pred[q] == v && q < j);
    if (rank < P) set[rank] = j;
  }
}

}  // namespace dali

extern "C" int dali_route_f64(const double* hidden, const double* residual,
                              const double* gate, int64_t T, int32_t d, int32_t N,
                              int32_t k, int32_t renorm, int32_t* topk_idx,
                              float* topk_w, int64_t* workloads, void* stream) {
  return dali::launch_route<double, double>(hidden, residual, gate, T, d, N, k, renorm,
                                            topk_idx, topk_w, workloads, stream);
}

namespace dali {
int launch_route_guarded(const uint16_t* hidden, const double* residual, const uint16_t* gate,
                         const float* wn2, int64_t T, int d, int N, int k, int renorm,
                         int32_t* idx, float* w, int64_t* workloads, void* stream,
                         int* launched, const int32_t* const* plan_ptrs = nullptr,
                         uint16_t* plan_xp = nullptr);
}

// bf16 engine path: the fp32 certified-margin kernel (route_guard.cu) for
// every eligible shape; the fp64 kernel below for the rest.
extern "C" int dali_route_bf16(const uint16_t* hidden, const double* residual,
                               const uint16_t* gate, const float* gate_norm2, int64_t T,
                               int32_t d, int32_t N,
                               int32_t k, int32_t renorm, int32_t* topk_idx,
                               float* topk_w, int64_t* workloads, void* stream) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_ETRACE,
               "num experts %d outside [1, %d]", N, DALI_MAX_EXPERTS);
  DALI_REQUIRE(k >= 1 && k <= N, DALI_ETRACE, "top_k %d out of range for %d experts", k, N);
  DALI_REQUIRE(workloads != nullptr, DALI_ETRACE, "workloads output required");
  int launched = 0;
  const int rc = dali::launch_route_guarded(hidden, residual, gate, gate_norm2, T, d, N, k,
                                            renorm, topk_idx, topk_w, workloads, stream,
                                            &launched);
  if (rc != DALI_OK || launched) return rc;
  return dali::launch_route<uint16_t, uint16_t>(hidden, residual, gate, T, d, N, k, renorm,
                                                topk_idx, topk_w, workloads, stream);
}

// Routing + plan + permute in one launch for decode-sized batches (T <= 16,
// T*k + N < 256): the certified routing kernel's batch-owning CTA also does
// dali_moe_plan_permute's work; otherwise the two run as separate launches.
extern "C" int dali_route_plan_bf16(const uint16_t* hidden, const uint16_t* gate,
                                    const float* gate_norm2, int64_t T, int32_t d, int32_t N,
                                    int32_t k, int32_t renorm, int32_t* topk_idx, float* topk_w,
                                    int64_t* workloads, int32_t* offsets, int32_t* perm_token,
                                    int32_t* pos, uint16_t* xp, void* stream) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_ETRACE,
               "num experts %d outside [1, %d]", N, DALI_MAX_EXPERTS);
  DALI_REQUIRE(k >= 1 && k <= N, DALI_ETRACE, "top_k %d out of range for %d experts", k, N);
  DALI_REQUIRE(workloads && topk_idx && offsets && perm_token && pos && xp, DALI_ETRACE,
               "route+plan needs every output");
  const int32_t* plan[3] = {offsets, perm_token, pos};
  int launched = 0;
  int rc = dali::launch_route_guarded(hidden, nullptr, gate, gate_norm2, T, d, N, k, renorm,
                                      topk_idx, topk_w, workloads, stream, &launched, plan, xp);
  if (rc != DALI_OK) return rc;
  if (!launched) {
    rc = dali_route_bf16(hidden, nullptr, gate, gate_norm2, T, d, N, k, renorm, topk_idx, topk_w,
                         workloads, stream);
    if (rc != DALI_OK) return rc;
    return dali_moe_plan_permute(topk_idx, T, k, N, hidden, d, offsets, perm_token, pos, xp,
                                 stream);
  }
  return DALI_OK;
}

extern "C" int dali_prefetch_select(const int64_t* predicted, int32_t N, int32_t P,
                                    int32_t* set, void* stream) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_EPREFETCH, "bad expert count %d", N);
  DALI_REQUIRE(P >= 0, DALI_EPREFETCH, "prefetch_size must be >= 0");
  if (P > N) P = N;
  if (P == 0) return DALI_OK;
  dali::prefetch_select_kernel<<<1, 256, 0, dali::as_stream(stream)>>>(predicted, N, P, set);
  DALI_LAUNCH_CHECK("prefetch_select_kernel");
  return DALI_OK;
}

extern "C" int dali_gate_probs_f64(const double* hidden, const double* gate, int64_t T, int32_t d,
                                   int32_t N, double* probs, void* stream) {
  DALI_REQUIRE(probs != nullptr, DALI_ETRACE, "probs output required");
  return dali::launch_route<double, double>(hidden, nullptr, gate, T, d, N, 1, 0, nullptr,
                                            nullptr, nullptr, stream, probs);
}

extern "C" int dali_gate_probs_bf16(const uint16_t* hidden, const uint16_t* gate, int64_t T,
                                    int32_t d, int32_t N, double* probs, void* stream) {
  DALI_REQUIRE(probs != nullptr, DALI_ETRACE, "probs output required");
  return dali::launch_route<uint16_t, uint16_t>(hidden, nullptr, gate, T, d, N, 1, 0, nullptr,
                                                nullptr, nullptr, stream, probs);
}
