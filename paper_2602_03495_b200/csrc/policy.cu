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

// ---------------------------------------------------------------------------
// Baseline solvers (assignment.py:154-402).  Lane 0 only,
// sequential exactly like the reference loops; scratch in shared memory.
// ---------------------------------------------------------------------------
struct BeamScratch {
  double tc[2 * DALI_MAX_BEAM], tg[2 * DALI_MAX_BEAM];
  int used[2 * DALI_MAX_BEAM], parent[2 * DALI_MAX_BEAM], dev[2 * DALI_MAX_BEAM];
  double stc[DALI_MAX_BEAM], stg[DALI_MAX_BEAM];
  int sused[DALI_MAX_BEAM];
  uint8_t back[DALI_MAX_EXPERTS][DALI_MAX_BEAM];   // (parent << 1) | device
};
struct BBScratch {
  double tc[DALI_MAX_EXPERTS + 1], tg[DALI_MAX_EXPERTS + 1], rem[DALI_MAX_EXPERTS + 1];
  int used[DALI_MAX_EXPERTS + 1], ng[DALI_MAX_EXPERTS + 1];
  int8_t stage[DALI_MAX_EXPERTS + 1], first_gpu[DALI_MAX_EXPERTS + 1], ok[DALI_MAX_EXPERTS + 1];
  int8_t choice[DALI_MAX_EXPERTS];
  uint8_t best_set[DALI_MAX_EXPERTS], cur_set[DALI_MAX_EXPERTS];
};
union SolverScratch {
  BeamScratch beam;
  BBScratch bb;
  double wsort[DALI_MAX_EXPERTS];
};

// float(cpu_times @ C), float(gpu_times @ G) in index order (assignment.py:166-168)
__device__ double lane_dot(const double* t, const int8_t* x, int N) {
  double acc = 0.0;
  for (int j = 0; j < N; ++j)
    if (x[j]) acc = acc + t[j];
  return acc;
}

// beam_assign (assignment.py:202-247).  Expects s.C/s.G zeroed.
__device__ void beam_scan(PolShared& s, BeamScratch& b, int N, int cap, int bw) {
  greedy_scan(s, cap);
  const double gmk = py_max(lane_dot(s.ct, s.C, N), lane_dot(s.gt, s.G, N));
  int n_st = 1;
  b.stc[0] = 0.0;
  b.stg[0] = 0.0;
  b.sused[0] = 0;
  for (int r = 0; r < s.n_act; ++r) {
    const int e = s.order[r];
    const double g = s.gt[e], c = s.ct[e];
    const int needs = s.res[e] ? 0 : 1;
    int nk = 0;
    for (int i = 0; i < n_st; ++i) {
      const double tc = b.stc[i], tg = b.stg[i];
      const int used = b.sused[i];
      const bool gok = cap < 0 || !needs || used < cap;
      auto push = [&](int dev) {
        b.tc[nk] = dev ? tc : tc + c;
        b.tg[nk] = dev ? tg + g : tg;
        b.used[nk] = dev ? used + needs : used;
        b.parent[nk] = i;
        b.dev[nk] = dev;
        ++nk;
      };
      if (gok && tg + g <= tc + c) { push(1); push(0); }
      else if (gok) { push(0); push(1); }
      else push(0);
    }
    // stable insertion sort by max(t_cpu, t_gpu)
    for (int i = 1; i < nk; ++i) {
      const double ktc = b.tc[i], ktg = b.tg[i], key = py_max(ktc, ktg);
      const int ku = b.used[i], kp = b.parent[i], kd = b.dev[i];
      int j = i - 1;
      while (j >= 0 && py_max(b.tc[j], b.tg[j]) > key) {
        b.tc[j + 1] = b.tc[j]; b.tg[j + 1] = b.tg[j]; b.used[j + 1] = b.used[j];
        b.parent[j + 1] = b.parent[j]; b.dev[j + 1] = b.dev[j];
        --j;
      }
      b.tc[j + 1] = ktc; b.tg[j + 1] = ktg; b.used[j + 1] = ku;
      b.parent[j + 1] = kp; b.dev[j + 1] = kd;
    }
    n_st = nk < bw ? nk : bw;
    for (int i = 0; i < n_st; ++i) {
      b.stc[i] = b.tc[i];
      b.stg[i] = b.tg[i];
      b.sused[i] = b.used[i];
      b.back[r][i] = (uint8_t)((b.parent[i] << 1) | b.dev[i]);
    }
  }
  if (gmk < py_max(b.stc[0], b.stg[0])) return;   // greedy strictly better: keep it
  for (int j = 0; j < N; ++j) { s.C[j] = 0; s.G[j] = 0; }
  int i = 0;
  for (int r = s.n_act - 1; r >= 0; --r) {
    const int v = b.back[r][i];
    if (v & 1) s.G[s.order[r]] = 1; else s.C[s.order[r]] = 1;
    i = v >> 1;
  }
}

// optimal_assign_with_stats (assignment.py:268-346): iterative branch and
// bound.  Returns the explored node count, or -1 when n_act > limit.
__device__ long long optimal_bb(PolShared& s, BBScratch& b, int N, int cap, int limit) {
  const int n = s.n_act;
  if (n > limit) return -1;
  double acc = 0.0;
  b.rem[n] = 0.0;
  for (int i = n - 1; i >= 0; --i) {
    const int e = s.order[i];
    const double m = s.gt[e] < s.ct[e] ? s.gt[e] : s.ct[e];
    acc = acc + m;
    b.rem[i] = acc;
  }
  greedy_scan(s, cap);
  double best_mk = py_max(lane_dot(s.ct, s.C, N), lane_dot(s.gt, s.G, N));
  int best_n = 0;
  for (int j = 0; j < N; ++j) { b.best_set[j] = s.G[j]; best_n += s.G[j]; }
  bool found = false;
  long long nodes = 0;
  int depth = 0;
  b.tc[0] = 0.0; b.tg[0] = 0.0; b.used[0] = 0; b.ng[0] = 0; b.stage[0] = 0;
  while (depth >= 0) {
    const double tc = b.tc[depth], tg = b.tg[depth];
    if (b.stage[depth] == 0) {
      ++nodes;
      const double lb = py_max(py_max(tc, tg), (tc + tg + b.rem[depth]) / 2.0);
      if (lb > best_mk || (lb == best_mk && b.ng[depth] > best_n)) { --depth; continue; }
      if (depth == n) {
        const double mk = py_max(tc, tg);
        for (int j = 0; j < N; ++j) b.cur_set[j] = 0;
        for (int i = 0; i < n; ++i) if (b.choice[i]) b.cur_set[s.order[i]] = 1;
        const int ng = b.ng[depth];
        bool better = mk < best_mk || (mk == best_mk && ng < best_n);
        if (!better && mk == best_mk && ng == best_n) {
          for (int j = 0; j < N; ++j)
            if (b.cur_set[j] != b.best_set[j]) { better = b.cur_set[j] != 0; break; }
        }
        if (better) {
          best_mk = mk;
          best_n = ng;
          for (int j = 0; j < N; ++j) b.best_set[j] = b.cur_set[j];
          found = true;
        }
        --depth;
        continue;
      }
      const int e = s.order[depth];
      const int needs = s.res[e] ? 0 : 1;
      b.ok[depth] = (cap < 0 || b.used[depth] + needs <= cap) ? 1 : 0;
      b.first_gpu[depth] = (tg + s.gt[e] <= tc + s.ct[e]) ? 1 : 0;
      b.stage[depth] = 1;
    }
    if (b.stage[depth] == 3) {
      b.choice[depth] = 0;
      --depth;
      continue;
    }
    // stage 1: first branch, stage 2: second branch
    const int dev = (b.stage[depth] == 1) == (b.first_gpu[depth] != 0) ? 1 : 0;
    b.stage[depth] += 1;
    if (dev == 1 && !b.ok[depth]) continue;
    const int e = s.order[depth];
    const int needs = s.res[e] ? 0 : 1;
    b.choice[depth] = (int8_t)dev;
    b.tc[depth + 1] = dev ? tc : tc + s.ct[e];
    b.tg[depth + 1] = dev ? tg + s.gt[e] : tg;
    b.used[depth + 1] = b.used[depth] + (dev ? needs : 0);
    b.ng[depth + 1] = b.ng[depth] + dev;
    b.stage[depth + 1] = 0;
    ++depth;
  }
  if (found) {
    for (int j = 0; j < N; ++j) {
      const bool act = s.wl[j] > 0.0;
      s.G[j] = act && b.best_set[j] ? 1 : 0;
      s.C[j] = act && !b.best_set[j] ? 1 : 0;
    }
  }
  return nodes;
}

// static_threshold_assign (assignment.py:349-377).  Expects s.C/s.G zeroed.
__device__ void static_scan(PolShared& s, double* wsort, int N, int cap, int has_thr,
                            double thr) {
  int n = 0;
  for (int j = 0; j < N; ++j)
    if (s.wl[j] > 0.0) wsort[n++] = s.wl[j];
  if (n == 0) return;
  if (!has_thr) {
    for (int i = 1; i < n; ++i) {          // insertion sort (values only)
      const double v = wsort[i];
      int j = i - 1;
      while (j >= 0 && wsort[j] > v) { wsort[j + 1] = wsort[j]; --j; }
      wsort[j + 1] = v;
    }
    thr = (n & 1) ? wsort[n / 2] : (wsort[n / 2 - 1] + wsort[n / 2]) / 2.0;
  }
  int slots = cap;
  // descending workload, ties to the lower index
  for (int done = 0; done < n; ++done) {
    int best = -1;
    for (int j = 0; j < N; ++j) {
      if (!(s.wl[j] > 0.0) || s.C[j] || s.G[j]) continue;
      if (best < 0 || s.wl[j] > s.wl[best]) best = j;
    }
    const bool allowed = slots < 0 || slots > 0 || s.res[best];
    if (s.wl[best] >= thr && allowed) {
      s.G[best] = 1;
      if (slots >= 0 && !s.res[best]) --slots;
    } else {
      s.C[best] = 1;
    }
  }
}

// force_insert victim (cache.py:128-143): lowest score (LRU: oldest clock),
// first in index order.
__device__ int insert_victim(const uint8_t* on_gpu, const double* scores, const int64_t* lru,
                             int N, bool use_lru) {
  int v = -1;
  for (int j = 0; j < N; ++j) {
    if (!on_gpu[j]) continue;
    if (v < 0 || (use_lru ? lru[j] < lru[v] : scores[j] < scores[v])) v = j;
  }
  return v;
}

// One assignment instance with any reference solver (assignment.py:172-402).
__global__ void __launch_bounds__(kPolThreads)
assign_kernel(const int64_t* __restrict__ workloads, const uint8_t* __restrict__ resident, int N,
              int cap, dali_cost_model cm, int use_cm, const double* __restrict__ cpu_times,
              const double* __restrict__ gpu_times, int policy, int beam_width, int limit,
              int has_thr, double thr, int8_t* __restrict__ C, int8_t* __restrict__ G,
              int64_t* __restrict__ nodes_out) {
  __shared__ PolShared s;
  __shared__ SolverScratch scratch;
  __shared__ long long sh_nodes;
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
  if (threadIdx.x == 0) {
    long long nodes = 0;
    switch (policy) {
      case 0: greedy_scan(s, cap); nodes = s.n_act; break;
      case 1: for (int r = 0; r < s.n_act; ++r) s.C[s.order[r]] = 1; break;
      case 2: {
        int slots = cap;
        for (int j = 0; j < N; ++j) {
          if (!(s.wl[j] > 0.0)) continue;
          if (slots < 0 || slots > 0 || s.res[j]) {
            s.G[j] = 1;
            if (slots >= 0 && !s.res[j]) --slots;
          } else {
            s.C[j] = 1;
          }
        }
        break;
      }
      case 3: beam_scan(s, scratch.beam, N, cap, beam_width); nodes = (long long)s.n_act * beam_width;
        break;
      case 4: nodes = optimal_bb(s, scratch.bb, N, cap, limit); break;
      default: static_scan(s, scratch.wsort, N, cap, has_thr, thr); break;
    }
    sh_nodes = nodes;
  }
  __syncthreads();
  if (e < N) {
    C[e] = s.C[e];
    G[e] = s.G[e];
  }
  if (threadIdx.x == 0 && nodes_out) nodes_out[0] = sh_nodes;
}

// Single cache operation on one layer's state (drop-in lookup / force_insert,
// cache.py:104-143).  lru: (N+1) int64 clocks with the clock last.
// out[0] = hit (lookup) or 1 if inserted (force_insert), out[1] = victim or -1.
__global__ void cache_op_kernel(uint8_t* on_gpu, const double* scores, int64_t* lru, int N,
                                int use_lru, int expert, int op, int32_t* out) {
  int victim = -1, flag = 0;
  if (op == 0) {                                   // lookup
    flag = on_gpu[expert] != 0;
    if (use_lru) {
      const int64_t clock = lru[N] + 1;
      lru[N] = clock;
      if (!flag) {
        victim = insert_victim(on_gpu, scores, lru, N, true);
        on_gpu[victim] = 0;
        on_gpu[expert] = 1;
      }
      lru[expert] = clock;
    }
  } else if (!on_gpu[expert]) {                    // force_insert
    victim = insert_victim(on_gpu, scores, lru, N, use_lru != 0);
    on_gpu[victim] = 0;
    on_gpu[expert] = 1;
    flag = 1;
  }
  out[0] = flag;
  out[1] = victim;
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
                    int32_t* slot_of_all, int64_t* lru_all,
                    const double* __restrict__ gate_probs, int n_tokens,
                    dali_layer_record* rec, const int32_t* __restrict__ desc) {
  DALI_PDL_ENTRY();
  __shared__ PolShared s;
  __shared__ SolverScratch scratch;
  __shared__ int sh_nins;
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
    } else if (cfg.assignment == 3) {
      beam_scan(s, scratch.beam, N, cfg.gpu_capacity, cfg.beam_width);
      nodes = s.n_act * cfg.beam_width;
    } else if (cfg.assignment == 4) {
      const long long nn = optimal_bb(s, scratch.bb, N, cfg.gpu_capacity,
                                      cfg.exact_solver_limit);
      if (nn < 0) {                 // refused: the host raises AssignmentError
        rec->err = 1;
        greedy_scan(s, cfg.gpu_capacity);
        nodes = 0;
      } else {
        nodes = (int)(nn > INT_MAX ? INT_MAX : nn);
        rec->err = 0;
      }
    } else if (cfg.assignment == 5) {
      static_scan(s, scratch.wsort, N, cfg.gpu_capacity, cfg.has_threshold, cfg.threshold);
      nodes = 0;
    } else {
      for (int r = 0; r < s.n_act; ++r) s.C[s.order[r]] = 1;
      nodes = 0;
    }
    if (cfg.assignment != 4) rec->err = 0;
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
  // does not mutate on lookup, cache.py:104-117).  LRU lookups and the
  // demand-insert toggle mutate the cache: sequential on lane 0 in index
  // order (simulator.py:372-379, cache.py:104-143).
  int ng = 0, nc = 0;
  const bool seq_lookup = cfg.cache_enabled && (cfg.cache_policy == 1 || cfg.insert_demand);
  if (threadIdx.x == 0) sh_nins = 0;
  if (e < N) {
    rec->C[e] = s.C[e];
    rec->G[e] = s.G[e];
    rec->workload[e] = (int32_t)workloads[e];
    rec->resident[e] = s.res[e];
    rec->hit[e] = (!seq_lookup && cfg.cache_enabled && s.G[e] && on_gpu[e]) ? 1 : 0;
    rec->order[e] = (int16_t)s.order[e];
    ng = s.G[e];
    nc = s.C[e];
  }
  __syncthreads();
  if (seq_lookup && threadIdx.x == 0) {
    const bool lru = cfg.cache_policy == 1;
    int64_t* lc = lru_all ? lru_all + (size_t)layer * (N + 1) : nullptr;
    const double* sc = scores_all + (size_t)layer * N;
    int32_t* slot_of = slot_of_all ? slot_of_all + (size_t)layer * N : nullptr;
    int nins = 0;
    for (int x = 0; x < N; ++x) {
      if (!s.G[x]) continue;
      const bool hit = on_gpu[x] != 0;
      rec->hit[x] = hit ? 1 : 0;
      int victim = -1;
      if (lru) {
        const int64_t clock = lc[N] + 1;
        lc[N] = clock;
        if (hit) {
          lc[x] = clock;
        } else {
          victim = insert_victim(on_gpu, sc, lc, N, true);
          lc[x] = clock;
          rec->ins_kind[nins] = 0;
        }
      } else if (!hit && cfg.insert_demand && !s.res[x]) {
        victim = insert_victim(on_gpu, sc, lc, N, false);
        rec->ins_kind[nins] = 1;
      }
      if (victim >= 0) {
        on_gpu[victim] = 0;
        on_gpu[x] = 1;
        if (slot_of) { slot_of[x] = slot_of[victim]; slot_of[victim] = -1; }
        rec->ins_victim[nins] = (int16_t)victim;
        rec->ins_expert[nins] = (int16_t)x;
        ++nins;
      }
    }
    sh_nins = nins;
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
        if (cfg.cache_enabled && cfg.insert_prefetched) {
          // force-insert the arrivals into layer+1's cache (simulator.py:421-423)
          uint8_t* nc_on = on_gpu_all + (size_t)(layer + 1) * N;
          const double* nsc = scores_all + (size_t)(layer + 1) * N;
          const int64_t* nlc = lru_all ? lru_all + (size_t)(layer + 1) * (N + 1) : nullptr;
          int32_t* nslot = slot_of_all ? slot_of_all + (size_t)(layer + 1) * N : nullptr;
          int nins = sh_nins;
          for (int r = 0; r < n_done; ++r) {
            const int x = rec->cand[r];
            if (nc_on[x]) continue;
            const int v = insert_victim(nc_on, nsc, nlc, N, cfg.cache_policy == 1);
            nc_on[v] = 0;
            nc_on[x] = 1;
            if (nslot) { nslot[x] = nslot[v]; nslot[v] = -1; }
            rec->ins_victim[nins] = (int16_t)v;
            rec->ins_expert[nins] = (int16_t)x;
            rec->ins_kind[nins] = 2;
            ++nins;
          }
          sh_nins = nins;
        }
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

  // 5. cache window update on this layer's true workloads (score policy:
  // summed gate scores of the layer's tokens; LRU: only EOS stops it).
  CacheOut o{0, 0};
  if (cfg.cache_enabled && cfg.cache_policy == 1) {
    if (threadIdx.x == 0 && is_eos) counters_all[2 * layer + 1] = 1;
    __syncthreads();
  } else if (cfg.cache_enabled && cfg.cache_policy == 2) {
    if (e < N) {               // gate_scores(...).sum(axis=0): rows in token order
      double acc = 0.0;
      for (int t = 0; t < n_tokens; ++t) acc = acc + gate_probs[(size_t)t * N + e];
      s.ct[e] = acc;           // cost scratch is free again here
    }
    __syncthreads();
    o = cache_window_update(s, on_gpu, scores_all + (size_t)layer * N,
                            counters_all + 2 * layer, N, cfg.w_size, cfg.u_size,
                            is_eos != 0, [&](int x) { return s.ct[x]; });
  } else if (cfg.cache_enabled) {
    o = cache_window_update(s, on_gpu, scores_all + (size_t)layer * N,
                            counters_all + 2 * layer, N, cfg.w_size, cfg.u_size,
                            is_eos != 0, [&](int x) { return s.wl[x]; });
  }
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
  if (threadIdx.x == 0) {
    rec->ev_valid = o.valid;
    rec->ev_n = o.n_swap;
    rec->boundary = o.valid ? (double)o.n_swap * cm.trans_time : 0.0;
    rec->stopped = cfg.cache_enabled ? counters_all[2 * layer + 1] : 0;
    rec->n_ins = sh_nins;
  }
}

static bool valid_baselines(const dali_policy_config* c, const int64_t* lru, const double* gp) {
  if (c->assignment == 3 && (c->beam_width < 1 || c->beam_width > DALI_MAX_BEAM)) return false;
  if (c->cache_enabled && c->cache_policy == 1 && !lru) return false;
  if (c->cache_enabled && c->cache_policy == 2 && !gp) return false;
  return true;
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
                                 int64_t* lru_state, const double* gate_probs,
                                 int32_t n_tokens, dali_layer_record* rec, void* stream) {
  DALI_REQUIRE(cfg != nullptr && dali::valid_cm(cm), DALI_ESIM, "invalid config / cost model");
  DALI_REQUIRE(dali::valid_baselines(cfg, lru_state, gate_probs), DALI_ESIM,
               "baseline policy configuration needs its state (beam width in [1, %d], "
               "LRU clocks, gate scores)", DALI_MAX_BEAM);
  DALI_REQUIRE(cfg->N >= 1 && cfg->N <= DALI_MAX_EXPERTS, DALI_ESIM, "expert count %d", cfg->N);
  DALI_REQUIRE(layer >= 0 && layer < cfg->L, DALI_ESIM, "layer %d out of range", layer);
  DALI_REQUIRE(!cfg->cache_enabled || cfg->u_size <= DALI_MAX_EXPERTS, DALI_ESIM, "u_size");
  dali::launch_pdl(dali::policy_layer_kernel, dim3(1), dim3(dali::kPolThreads), 0, dali::as_stream(stream), 
      *cfg, *cm, step, layer, token_index, is_eos, workloads, predicted, on_gpu, scores,
      counters, arrived, slot_of, lru_state, gate_probs, n_tokens, rec, nullptr);
  DALI_LAUNCH_CHECK("policy_layer_kernel");
  return DALI_OK;
}

extern "C" int dali_policy_layer_desc(const dali_policy_config* cfg, const dali_cost_model* cm,
                                      int32_t layer, const int32_t* desc,
                                      const int64_t* workloads, const int64_t* predicted,
                                      uint8_t* on_gpu, double* scores, int32_t* counters,
                                      uint8_t* arrived, int32_t* slot_of, int64_t* lru_state,
                                      const double* gate_probs, int32_t n_tokens,
                                      dali_layer_record* rec_base, void* stream) {
  DALI_REQUIRE(cfg != nullptr && dali::valid_cm(cm) && desc != nullptr, DALI_ESIM,
               "invalid config / cost model / descriptor");
  DALI_REQUIRE(dali::valid_baselines(cfg, lru_state, gate_probs), DALI_ESIM,
               "baseline policy configuration needs its state");
  DALI_REQUIRE(layer >= 0 && layer < cfg->L, DALI_ESIM, "layer %d out of range", layer);
  dali::launch_pdl(dali::policy_layer_kernel, dim3(1), dim3(dali::kPolThreads), 0, dali::as_stream(stream), 
      *cfg, *cm, 0, layer, 0, 0, workloads, predicted, on_gpu, scores, counters, arrived,
      slot_of, lru_state, gate_probs, n_tokens, rec_base, desc);
  DALI_LAUNCH_CHECK("policy_layer_kernel(desc)");
  return DALI_OK;
}

namespace dali {
__global__ void step_advance_kernel(int32_t* desc) {
  DALI_PDL_ENTRY();
  desc[0] += 1;            // step
  desc[1] += 1;            // token_index
  desc[3] += desc[6];      // record_index += L
  desc[4] += 1;            // pos
  desc[5] += 1;            // len
}
}  // namespace dali

extern "C" int dali_step_advance(int32_t* desc, void* stream) {
  dali::launch_pdl(dali::step_advance_kernel, dim3(1), dim3(1), 0, dali::as_stream(stream), desc);
  DALI_LAUNCH_CHECK("step_advance_kernel");
  return DALI_OK;
}

extern "C" int dali_assign(int32_t policy, const int64_t* workloads, const uint8_t* resident,
                           int32_t N, int32_t gpu_capacity, const dali_cost_model* cm,
                           const double* cpu_times, const double* gpu_times, int32_t beam_width,
                           int32_t exact_solver_limit, int32_t has_threshold, double threshold,
                           int8_t* C, int8_t* G, int64_t* nodes, void* stream) {
  DALI_REQUIRE(N >= 0 && N <= DALI_MAX_EXPERTS, DALI_EASSIGN, "expert count %d outside [0, %d]",
               N, DALI_MAX_EXPERTS);
  DALI_REQUIRE(policy >= 0 && policy <= 5, DALI_EASSIGN, "unknown assignment policy %d", policy);
  DALI_REQUIRE(policy != 3 || (beam_width >= 1 && beam_width <= DALI_MAX_BEAM), DALI_EASSIGN,
               "beam_width must be in [1, %d], got %d", DALI_MAX_BEAM, beam_width);
  const bool use_cm = cpu_times == nullptr || gpu_times == nullptr;
  DALI_REQUIRE(!use_cm || dali::valid_cm(cm), DALI_EASSIGN,
               "either a cost model or explicit times required");
  if (N == 0) return DALI_OK;
  dali_cost_model local{};
  if (use_cm) local = *cm;
  dali::assign_kernel<<<1, dali::kPolThreads, 0, dali::as_stream(stream)>>>(
      workloads, resident, N, gpu_capacity, local, use_cm ? 1 : 0, cpu_times, gpu_times, policy,
      beam_width, exact_solver_limit, has_threshold, threshold, C, G, nodes);
  DALI_LAUNCH_CHECK("assign_kernel");
  return DALI_OK;
}

extern "C" int dali_cache_op(uint8_t* on_gpu, const double* scores, int64_t* lru_state,
                             int32_t N, int32_t use_lru, int32_t expert, int32_t op, int32_t* out,
                             void* stream) {
  DALI_REQUIRE(N >= 1 && N <= DALI_MAX_EXPERTS, DALI_ECACHE, "expert count %d outside [1, %d]",
               N, DALI_MAX_EXPERTS);
  DALI_REQUIRE(expert >= 0 && expert < N, DALI_ECACHE, "expert %d out of range [0, %d)", expert,
               N);
  DALI_REQUIRE(!use_lru || lru_state, DALI_ECACHE, "LRU clocks required");
  dali::cache_op_kernel<<<1, 1, 0, dali::as_stream(stream)>>>(on_gpu, scores, lru_state, N,
                                                              use_lru, expert, op, out);
  DALI_LAUNCH_CHECK("cache_op_kernel");
  return DALI_OK;
}
