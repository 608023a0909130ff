// (2) Greedy assignment, (3) prefetch arrival rule, (4) workload-aware cache,
// fused into single-CTA policy kernels.  Compiled with -fmad=false: every
// fp64 expression is evaluated exactly as the reference's Python/numpy
// expression (no contraction), so decisions are bit-identical.
//
// Reference: cost_model.py:19-27,70-103 (cost evaluation), assignment.py:
// 119-123,172-199 (order + greedy), simulator.py:151-197 (GPU-lane
// timeline), simulator.py:354-444 (driver order: residency, lookups,
// prefetch window, cache update), cache.py:146-214 (window update).
//
// Parallel structure: the per-expert cost evaluation, the stable ranking
// of activated experts (one thread per expert counting its predecessors),
// the cache candidate/victim ranks and all vector bookkeeping run one
// thread per expert; the greedy completion-time scan and the virtual-clock
// timeline are inherently sequential (each decision depends on the running
// lane totals) and run on lane 0 over <= n_act experts.
#include <climits>

#include "common.cuh"

namespace dali {

constexpr int kPolThreads = 256;   // == DALI_MAX_EXPERTS

__device__ double interp_ms(double w, const double* xs, const double* ys, int n) {
  // np.interp inside the table, last-segment extrapolation beyond it.
  const double xl = xs[n - 1];
  if (w > xl) {
    const double slope = n >= 2 ? (ys[n - 1] - ys[n - 2]) / (xl - xs[n - 2]) : 0.0;
    return ys[n - 1] + slope * (w - xl);
  }
  if (w >= xl) return ys[n - 1];
  if (w <= xs[0]) return ys[0];
  int lo = 0, hi = n - 1;                // xs[lo] <= w < xs[hi]
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (xs[mid] <= w) lo = mid; else hi = mid;
  }
  if (w == xs[lo]) return ys[lo];
  const double slope = (ys[lo + 1] - ys[lo]) / (xs[lo + 1] - xs[lo]);
  return slope * (w - xs[lo]) + ys[lo];
}

__device__ __forceinline__ double t_cpu(const dali_cost_model& cm, double w) {
  return w == 0.0 ? 0.0 : interp_ms(w, cm.cpu_xs, cm.cpu_ys, cm.n_cpu);
}
__device__ __forceinline__ double t_gpu_compute(const dali_cost_model& cm, double w) {
  return w == 0.0 ? 0.0 : interp_ms(w, cm.gpu_xs, cm.gpu_ys, cm.n_gpu);
}
__device__ __forceinline__ double py_max(double a, double b) { return b > a ? b : a; }
__device__ __forceinline__ double py_min(double a, double b) { return b < a ? b : a; }

// CPython float_floor_div (Objects/floatobject.c) for the prefetch window.
__device__ double py_floordiv(double vx, double wx) {
  double mod = fmod(vx, wx);
  double div = (vx - mod) / wx;
  if (mod != 0.0) {
    if ((wx < 0) != (mod < 0)) { mod += wx; div -= 1.0; }
  }
  double fl;
  if (div != 0.0) {
    fl = floor(div);
    if (div - fl > 0.5) fl += 1.0;
  } else {
    fl = copysign(0.0, vx / wx);
  }
  return fl;
}

struct PolShared {
  double ct[DALI_MAX_EXPERTS];
  double gt[DALI_MAX_EXPERTS];
  double wl[DALI_MAX_EXPERTS];
  int order[DALI_MAX_EXPERTS];
  uint8_t res[DALI_MAX_EXPERTS];
  int8_t C[DALI_MAX_EXPERTS];
  int8_t G[DALI_MAX_EXPERTS];
  int cand[DALI_MAX_EXPERTS];
  int vict[DALI_MAX_EXPERTS];
  int n_act;
};

// Stable descending rank of |gpu - cpu| over activated experts
// (sorted_order, assignment.py:119-123).  All threads participate.
__device__ void rank_activated(PolShared& s, int N) {
  const int e = threadIdx.x;
  int act = 0;
  if (e < N) {
    act = s.wl[e] > 0.0;
    s.order[e] = -1;
  }
  const int n_act = __syncthreads_count(act);
  if (e < N && act) {
    const double g = fabs(s.gt[e] - s.ct[e]);
    int r = 0;
    for (int j = 0; j < N; ++j) {
      if (!(s.wl[j] > 0.0)) continue;
      const double gj = fabs(s.gt[j] - s.ct[j]);
      r += (gj > g) || (gj == g && j < e);
    }
    s.order[r] = e;
  }
  if (threadIdx.x == 0) s.n_act = n_act;
  __syncthreads();
}

// Algorithm 1 with the capacity guard (greedy_assign, assignment.py:172-199).
// Lane 0 only.
__device__ void greedy_scan(PolShared& s, int cap) {
  double lane_cpu = 0.0, lane_gpu = 0.0;
  int slots = cap;
  for (int r = 0; r < s.n_act; ++r) {
    const int e = s.order[r];
    const double g = s.gt[e], c = s.ct[e];
    const bool may = cap < 0 || slots > 0 || s.res[e];
    if (may && lane_gpu + g <= lane_cpu + c) {
      s.G[e] = 1;
      lane_gpu = lane_gpu + g;
      if (cap >= 0 && !s.res[e]) --slots;
    } else {
      s.C[e] = 1;
      lane_cpu = lane_cpu + c;
    }
  }
}

__global__ void __launch_bounds__(kPolThreads)
greedy_kernel(const int64_t* __restrict__ workloads, const uint8_t* __restrict__ resident,
              int N, int cap, dali_cost_model cm, int use_cm,
              const double* __restrict__ cpu_times, const double* __restrict__ gpu_times,
              int8_t* __restrict__ C, int8_t* __restrict__ G, int32_t* __restrict__ order,
              double* __restrict__ times_out) {
  __shared__ PolShared s;
  const int e = threadIdx.x;
  if (e < N) {
    const double w = (double)workloads[e];
    s.wl[e] = w;
    s.res[e] = resident[e] ? 1 : 0;
    if (use_cm) {
      s.ct[e] = t_cpu(cm, w);
      s.gt[e] = w == 0.0 ? 0.0 : py_max(s.res[e] ? 0.0 : cm.trans_time, t_gpu_compute(cm, w));
    } else {
      s.ct[e] = cpu_times[e];
      s.gt[e] = gpu_times[e];
    }
    s.C[e] = 0;
    s.G[e] = 0;
  }
  __syncthreads();
  rank_activated(s, N);
  if (threadIdx.x == 0) greedy_scan(s, cap);
  __syncthreads();
  if (e < N) {
    C[e] = s.C[e];
    G[e] = s.G[e];
    order[e] = s.order[e];
    if (times_out) {
      times_out[e] = s.ct[e];
      times_out[N + e] = s.gt[e];
    }
  }
}

__global__ void cost_eval_kernel(dali_cost_model cm, const double* __restrict__ w, int64_t n,
                                 double* __restrict__ co, double* __restrict__ go) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    if (co) co[i] = t_cpu(cm, w[i]);
    if (go) go[i] = t_gpu_compute(cm, w[i]);
  }
}

// Workload-policy window update (record_and_maybe_replace, cache.py:146-214)
// on one layer's state.  vec(e) supplies the f64 increment.  All threads.
// Returns via shared: ev_valid, n_swap, s.cand / s.vict hold admitted/evicted.
struct CacheOut { int valid, n_swap; };

template <typename VecF>
__device__ CacheOut cache_window_update(PolShared& s, uint8_t* on_gpu, double* scores,
                                        int32_t* counters, int N, int w_size, int u_size,
                                        bool is_eos, VecF vec) {
  __shared__ int sh_flag[2];
  CacheOut out{0, 0};
  const int e = threadIdx.x;
  const int stopped = counters[1];
  if (stopped) return out;                 // uniform across the CTA
  if (e < N) scores[e] = scores[e] + vec(e);
  __syncthreads();
  const int window = counters[0] + 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    counters[0] = window;
    if (is_eos) counters[1] = 1;
  }
  if (is_eos || window < w_size) { __syncthreads(); return out; }
  // Candidates: off-GPU by (-score, idx); victims: on-GPU by (score, idx).
  if (e < N) { s.cand[e] = -1; s.vict[e] = -1; }
  __syncthreads();
  if (e < N) {
    const double se = scores[e];
    const bool on = on_gpu[e] != 0;
    int r = 0;
    for (int j = 0; j < N; ++j) {
      if ((on_gpu[j] != 0) != on) continue;
      const double sj = scores[j];
      r += on ? ((sj < se) || (sj == se && j < e)) : ((sj > se) || (sj == se && j < e));
    }
    if (r < u_size) { if (on) s.vict[r] = e; else s.cand[r] = e; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int m = 0;
    while (m < u_size && s.cand[m] >= 0 && s.vict[m] >= 0 &&
           scores[s.cand[m]] >= scores[s.vict[m]])
      ++m;
    sh_flag[0] = m;
  }
  __syncthreads();
  const int m = sh_flag[0];
  if (e < m) {
    on_gpu[s.vict[e]] = 0;
    on_gpu[s.cand[e]] = 1;
  }
  __syncthreads();
  if (e < N) scores[e] = 0.0;
  if (threadIdx.x == 0) counters[0] = 0;
  __syncthreads();
  out.valid = 1;
  out.n_swap = m;
  return out;
}

__global__ void __launch_bounds__(kPolThreads)
cache_record_kernel(uint8_t* on_gpu, double* scores, int32_t* counters, int N, int w_size,
                    int u_size, const double* __restrict__ workload, int is_eos, int32_t* ev) {
  __shared__ PolShared s;
  CacheOut o = cache_window_update(s, on_gpu, scores, counters, N, w_size, u_size, is_eos != 0,
                                   [&](int e) { return workload[e]; });
  if (threadIdx.x == 0) { ev[0] = o.valid; ev[1] = o.n_swap; }
  if ((int)threadIdx.x < o.n_swap) {
    ev[2 + threadIdx.x] = s.vict[threadIdx.x];
    ev[2 + DALI_MAX_EXPERTS + threadIdx.x] = s.cand[threadIdx.x];
  }
}

// Fused per-layer policy step; see dali.h for the contract.
__global__ void __launch_bounds__(kPolThreads)
policy_layer_kernel(dali_policy_config cfg, dali_cost_model cm, int step, int layer,
                    int token_index, int is_eos, const int64_t* __restrict__ workloads,
                    const int64_t* __restrict__ predicted, uint8_t* on_gpu_all,
                    double* scores_all, int32_t* counters_all, uint8_t* arrived_all,
                    int32_t* slot_of_all, dali_layer_record* rec,
                    const int32_t* __restrict__ desc) {
  __shared__ PolShared s;
  if (desc) {                     // graph replay: per-step scalars live on device
    step = desc[0];
    token_index = desc[1];
    is_eos = step == desc[2];
    rec += desc[3] + layer;
  }
  __shared__ double sh_d[8];
  const int N = cfg.N, L = cfg.L;
  const int e = threadIdx.x;
  uint8_t* on_gpu = on_gpu_all + (size_t)layer * N;
  uint8_t* arrived = arrived_all + (size_t)layer * N;
  const bool prefetch_on = cfg.prefetch_size > 0;
  const bool has_next = layer < L - 1;

  // 1. residency = cache | arrived prefetches; per-expert costs.
  if (e < N) {
    const double w = (double)workloads[e];
    uint8_t r = 0;
    if (cfg.cache_enabled && on_gpu[e]) r = 1;
    if (arrived[e] || cfg.all_resident) r = 1;
    arrived[e] = 0;                       // consumed for this step
    s.wl[e] = w;
    s.res[e] = r;
    s.ct[e] = t_cpu(cm, w);
    s.gt[e] = w == 0.0 ? 0.0 : py_max(r ? 0.0 : cm.trans_time, t_gpu_compute(cm, w));
    s.C[e] = 0;
    s.G[e] = 0;
  }
  __syncthreads();
  rank_activated(s, N);

  // 2. assignment + GPU-lane timeline (simulate_layer, simulator.py:151-193).
  if (threadIdx.x == 0) {
    int nodes;
    if (cfg.assignment == 0) {
      greedy_scan(s, cfg.gpu_capacity);
      nodes = s.n_act;
    } else if (cfg.assignment == 2) {
      // all_gpu_assign (assignment.py:387-402): activated experts in index
      // order; capacity overflow of non-resident experts falls back to CPU
      int slots = cfg.gpu_capacity;
      for (int j = 0; j < N; ++j) {
        if (!(s.wl[j] > 0.0)) continue;
        if (slots < 0 || slots > 0 || s.res[j]) {
          s.G[j] = 1;
          if (slots >= 0 && !s.res[j]) --slots;
        } else {
          s.C[j] = 1;
        }
      }
      nodes = 0;
    } else {
      for (int r = 0; r < s.n_act; ++r) s.C[s.order[r]] = 1;
      nodes = 0;
    }
    double cpu_busy = 0.0;
    for (int j = 0; j < N; ++j)
      if (s.C[j]) cpu_busy = cpu_busy + s.ct[j];
    double pcie_t = 0.0, engine_t = 0.0, demand_ms = 0.0;
    int n_demand = 0;
    for (int r = 0; r < s.n_act; ++r) {
      const int x = s.order[r];
      if (!s.G[x]) continue;
      const double comp = t_gpu_compute(cm, s.wl[x]);
      double start;
      if (s.res[x]) {
        start = engine_t;
      } else {
        const double end = pcie_t + cm.trans_time;
        demand_ms = demand_ms + (end - pcie_t);
        pcie_t = end;
        ++n_demand;
        start = py_max(engine_t, end);
      }
      engine_t = start + comp;
    }
    const double shared_ms = cfg.has_shared ? cm.shared_expert_gpu_time : 0.0;
    const double extra = (prefetch_on && has_next) ? cfg.prefetch_compute_ms : 0.0;
    const double latency = py_max(cpu_busy, engine_t) + shared_ms + cfg.scheduling_overhead_ms +
                           cfg.solver_node_cost_ms * (double)nodes + extra;
    sh_d[0] = cpu_busy;
    sh_d[1] = engine_t;
    sh_d[2] = latency;
    sh_d[3] = n_demand ? pcie_t : 0.0;     // demand_end
    sh_d[4] = demand_ms;
    rec->step = step;
    rec->layer = layer;
    rec->token_index = token_index;
    rec->n_act = s.n_act;
    rec->nodes = nodes;
    rec->n_demand = n_demand;
    rec->cpu_busy = cpu_busy;
    rec->gpu_makespan = engine_t;
    rec->latency = latency;
    rec->demand_end = sh_d[3];
    rec->demand_ms = demand_ms;
  }
  __syncthreads();

  // 3. lookups of GPU-assigned experts (hit iff cached; workload policy
  // does not mutate on lookup, cache.py:104-117).
  int ng = 0, nc = 0;
  if (e < N) {
    rec->C[e] = s.C[e];
    rec->G[e] = s.G[e];
    rec->workload[e] = (int32_t)workloads[e];
    rec->resident[e] = s.res[e];
    rec->hit[e] = (cfg.cache_enabled && s.G[e] && on_gpu[e]) ? 1 : 0;
    rec->order[e] = (int16_t)s.order[e];
    ng = s.G[e];
    nc = s.C[e];
  }
  ng = __syncthreads_count(ng);
  nc = __syncthreads_count(nc);
  if (threadIdx.x == 0) { rec->n_gpu = ng; rec->n_cpu = nc; }

  // 4. prefetch for layer+1 with the virtual-clock arrival rule
  // (simulator.py:382-423).
  if (has_next) {
    uint8_t* arr_next = arrived_all + (size_t)(layer + 1) * N;
    if (e < N) arr_next[e] = 0;
    if (e < N) rec->pset[e] = -1;
    __syncthreads();
    if (prefetch_on && predicted != nullptr) {
      const int P = cfg.prefetch_size < N ? cfg.prefetch_size : N;
      if (e < N) {
        const int64_t v = predicted[e];
        int r = 0;
        for (int q = 0; q < N; ++q) r += (predicted[q] > v) || (predicted[q] == v && q < e);
        if (r < P) s.cand[r] = e;         // pset in rank order
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        const uint8_t* next_cache = on_gpu_all + (size_t)(layer + 1) * N;
        int nc2 = 0;
        for (int r = 0; r < P; ++r) {
          const int x = s.cand[r];
          rec->pset[r] = (int16_t)x;
          if (!(cfg.cache_enabled && next_cache[x])) rec->cand[nc2++] = (int16_t)x;
        }
        const double idle = py_max(0.0, sh_d[2] + cfg.non_moe - sh_d[3]);
        int n_done;
        double consumed;
        if (cm.trans_time > 0) {
          const double nf = py_floordiv(idle, cm.trans_time);
          long long nfit = (long long)nf;
          n_done = nfit < nc2 ? (int)(nfit < 0 ? 0 : nfit) : nc2;
          consumed = py_min((double)nc2 * cm.trans_time, idle);
        } else {
          n_done = nc2;
          consumed = 0.0;
        }
        for (int r = 0; r < n_done; ++r) arr_next[rec->cand[r]] = 1;
        rec->n_pset = P;
        rec->n_cand = nc2;
        rec->n_done = n_done;
        rec->consumed = consumed;
      }
    } else if (threadIdx.x == 0) {
      rec->n_pset = 0; rec->n_cand = 0; rec->n_done = 0; rec->consumed = 0.0;
    }
  } else if (threadIdx.x == 0) {
    rec->n_pset = 0; rec->n_cand = 0; rec->n_done = 0; rec->consumed = 0.0;
  }
  __syncthreads();

  // 5. cache window update on this layer's true workloads.
  CacheOut o{0, 0};
  if (cfg.cache_enabled) {
    o = cache_window_update(s, on_gpu, scores_all + (size_t)layer * N,
                            counters_all + 2 * layer, N, cfg.w_size, cfg.u_size,
                            is_eos != 0, [&](int x) { return s.wl[x]; });
    if ((int)threadIdx.x < o.n_swap) {
      const int v = s.vict[threadIdx.x], c = s.cand[threadIdx.x];
      rec->evicted[threadIdx.x] = (int16_t)v;
      rec->admitted[threadIdx.x] = (int16_t)c;
      if (slot_of_all) {
        int32_t* slot_of = slot_of_all + (size_t)layer * N;
        slot_of[c] = slot_of[v];
        slot_of[v] = -1;
      }
    }
  }
  if (threadIdx.x == 0) {
    rec->ev_valid = o.valid;
    rec->ev_n = o.n_swap;
    rec->boundary = o.valid ? (double)o.n_swap * cm.trans_time : 0.0;
    rec->stopped = cfg.cache_enabled ? counters_all[2 * layer + 1] : 0;
  }
}

static bool valid_cm(const dali_cost_model* cm) {
  return cm && cm->n_cpu >= 2 && cm->n_cpu <= DALI_MAX_SAMPLES && cm->n_gpu >= 2 &&
         cm->n_gpu <= DALI_MAX_SAMPLES;
}

}  // namespace dali

extern "C" int dali_greedy(const int64_t* workloads, const uint8_t* resident, int32_t N,
                           int32_t gpu_capacity, const dali_cost_model* cm,
                           const double* cpu_times, const double* gpu_times, int8_t* C,
                           int8_t* G, int32_t* order, double* times_out, void* stream) {
  DALI_REQUIRE(N >= 0 && N <= DALI_MAX_EXPERTS, DALI_EASSIGN, "expert count %d outside [0, %d]",
               N, DALI_MAX_EXPERTS);
  const bool use_cm = cpu_times == nullptr || gpu_times == nullptr;
  DALI_REQUIRE(!use_cm || dali::valid_cm(cm), DALI_EASSIGN,
               "either a cost model or explicit times required");
  if (N == 0) return DALI_OK;
  dali_cost_model local{};
  if (use_cm) local = *cm;
  dali::greedy_kernel<<<1, dali::kPolThreads, 0, dali::as_stream(stream)>>>(
      workloads, resident, N, gpu_capacity, local, use_cm ? 1 : 0, cpu_times, gpu_times, C, G,
      order, times_out);
  DALI_LAUNCH_CHECK("greedy_kernel");
  return DALI_OK;
}

extern "C" int dali_cost_eval(const dali_cost_model* cm, const double* w, int64_t n,
                              double* cpu_out, double* gpu_out, void* stream) {
  DALI_REQUIRE(dali::valid_cm(cm), DALI_ECOSTMODEL, "invalid cost model tables");
  if (n <= 0) return DALI_OK;
  dali::cost_eval_kernel<<<(unsigned)((n + 255) / 256), 256, 0, dali::as_stream(stream)>>>(
      *cm, w, n, cpu_out, gpu_out);
  DALI_LAUNCH_CHECK("cost_eval_kernel");
  return DALI_OK;
}

extern "C" int dali_cache_record(uint8_t* on_gpu, double* scores, int32_t* counters, int32_t N,
                                 int32_t w_size, int32_t u_size, const double* workload,
                                 int32_t is_eos, int32_t* ev, void* stream) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_ECACHE, "expert count %d outside [1, %d]",
               N, DALI_MAX_EXPERTS);
  DALI_REQUIRE(w_size >= 1, DALI_ECACHE, "w_size must be >= 1, got %d", w_size);
  DALI_REQUIRE(u_size >= 0, DALI_ECACHE, "u_size must be >= 0, got %d", u_size);
  dali::cache_record_kernel<<<1, dali::kPolThreads, 0, dali::as_stream(stream)>>>(
      on_gpu, scores, counters, N, w_size, u_size, workload, is_eos, ev);
  DALI_LAUNCH_CHECK("cache_record_kernel");
  return DALI_OK;
}

extern "C" int dali_policy_layer(const dali_policy_config* cfg, const dali_cost_model* cm,
                                 int32_t step, int32_t layer, int32_t token_index,
                                 int32_t is_eos, const int64_t* workloads,
                                 const int64_t* predicted, uint8_t* on_gpu, double* scores,
                                 int32_t* counters, uint8_t* arrived, int32_t* slot_of,
                                 dali_layer_record* rec, void* stream) {
  DALI_REQUIRE(cfg != nullptr && dali::valid_cm(cm), DALI_ESIM, "invalid config / cost model");
  DALI_REQUIRE(cfg->N >= 1 && cfg->N <= DALI_MAX_EXPERTS, DALI_ESIM, "expert count %d", cfg->N);
  DALI_REQUIRE(layer >= 0 && layer < cfg->L, DALI_ESIM, "layer %d out of range", layer);
  DALI_REQUIRE(!cfg->cache_enabled || cfg->u_size <= DALI_MAX_EXPERTS, DALI_ESIM, "u_size");
  dali::policy_layer_kernel<<<1, dali::kPolThreads, 0, dali::as_stream(stream)>>>(
      *cfg, *cm, step, layer, token_index, is_eos, workloads, predicted, on_gpu, scores,
      counters, arrived, slot_of, rec, nullptr);
  DALI_LAUNCH_CHECK("policy_layer_kernel");
  return DALI_OK;
}

extern "C" int dali_policy_layer_desc(const dali_policy_config* cfg, const dali_cost_model* cm,
                                      int32_t layer, const int32_t* desc,
                                      const int64_t* workloads, const int64_t* predicted,
                                      uint8_t* on_gpu, double* scores, int32_t* counters,
                                      uint8_t* arrived, int32_t* slot_of,
                                      dali_layer_record* rec_base, void* stream) {
  DALI_REQUIRE(cfg != nullptr && dali::valid_cm(cm) && desc != nullptr, DALI_ESIM,
               "invalid config / cost model / descriptor");
  DALI_REQUIRE(layer >= 0 && layer < cfg->L, DALI_ESIM, "layer %d out of range", layer);
  dali::policy_layer_kernel<<<1, dali::kPolThreads, 0, dali::as_stream(stream)>>>(
      *cfg, *cm, 0, layer, 0, 0, workloads, predicted, on_gpu, scores, counters, arrived,
      slot_of, rec_base, desc);
  DALI_LAUNCH_CHECK("policy_layer_kernel(desc)");
  return DALI_OK;
}

namespace dali {
__global__ void step_advance_kernel(int32_t* desc) {
  desc[0] += 1;            // step
  desc[1] += 1;            // token_index
  desc[3] += desc[6];      // record_index += L
  desc[4] += 1;            // pos
  desc[5] += 1;            // len
}
}  // namespace dali

extern "C" int dali_step_advance(int32_t* desc, void* stream) {
  dali::step_advance_kernel<<<1, 1, 0, dali::as_stream(stream)>>>(desc);
  DALI_LAUNCH_CHECK("step_advance_kernel");
  return DALI_OK;
}
