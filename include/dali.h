/*
 * dali.h -- C-ABI of the B200-native DALI hot path (libdali.so, sm_100a).
 *
 * Plain pointers and sizes only; no torch types.  Every entry point is
 * asynchronous on the caller's CUDA stream (passed as `void*`, NULL = legacy
 * default stream) unless stated otherwise, and returns 0 on success or one
 * of the DALI_E* codes below.  The message of the last failure on the
 * calling thread is available from dali_last_error().
 *
 * Device-pointer arguments are marked [dev]; host pointers [host].
 *
 * The reference (``moesim``, pure Python/numpy) has no FFI; each function
 * below names the reference Python function it replaces (file:line relative
 * to /root/reference/pkg/src/moesim).  INTEGRATION.md shows the ctypes
 * binding a maintainer would add on the reference side.
 */
#ifndef DALI_H_
#define DALI_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes; the Python shim maps them onto moesim.errors classes
 * (errors.py:4-50). */
#define DALI_OK 0
#define DALI_ETRACE 1       /* TraceError: shape / top_k / gating input   */
#define DALI_ECOSTMODEL 2   /* CostModelError                             */
#define DALI_EASSIGN 3      /* AssignmentError                            */
#define DALI_EPREFETCH 4    /* PrefetchError                              */
#define DALI_ECACHE 5       /* CacheError                                 */
#define DALI_ESIM 6         /* SimulationError                            */
#define DALI_ECUDA 100      /* CUDA runtime failure                       */

#define DALI_MAX_SAMPLES 32    /* cost-model table length incl. (0,0)     */
#define DALI_MAX_EXPERTS 256   /* routed experts per layer                */
#define DALI_MAX_TOPK 16

/* Piecewise-linear cost model, passed BY VALUE into kernels.
 * Mirrors CostModel (cost_model.py:54-68): xs/ys include the (0,0) anchor. */
typedef struct dali_cost_model {
  int32_t n_cpu, n_gpu;
  double cpu_xs[DALI_MAX_SAMPLES], cpu_ys[DALI_MAX_SAMPLES];
  double gpu_xs[DALI_MAX_SAMPLES], gpu_ys[DALI_MAX_SAMPLES];
  double trans_time;
  double shared_expert_gpu_time;
  double non_moe_layer_time;
} dali_cost_model;

/* Per-layer decision record written by dali_policy_layer (one per
 * step x layer).  Fields follow the reference driver loop
 * (simulator.py:354-475).  Expert lists are -1 terminated / counted. */
typedef struct dali_layer_record {
  int32_t step, layer, token_index, n_act;
  int32_t n_gpu, n_cpu, n_demand, n_pset;
  int32_t n_cand, n_done, ev_valid, ev_n;
  int32_t nodes, stopped, n_ins, err; /* err 1: exact solver refused   */
  double cpu_busy;      /* cpu_times @ C                                  */
  double gpu_makespan;  /* engine_t of the GPU-lane pipeline              */
  double latency;       /* layer_latency                                  */
  double demand_end;    /* end of the last demand transfer                */
  double demand_ms;     /* sum of demand interval lengths                 */
  double consumed;      /* prefetch channel time charged                  */
  double boundary;      /* replacement transfer charge                    */
  double pad2;
  int8_t C[DALI_MAX_EXPERTS];
  int8_t G[DALI_MAX_EXPERTS];
  uint8_t resident[DALI_MAX_EXPERTS];
  uint8_t hit[DALI_MAX_EXPERTS];      /* lookup result for G experts      */
  int16_t order[DALI_MAX_EXPERTS];    /* sorted_order (activated)         */
  int16_t pset[DALI_MAX_EXPERTS];     /* prefetch set for layer+1         */
  int16_t cand[DALI_MAX_EXPERTS];     /* pset minus cache[layer+1]        */
  int16_t evicted[DALI_MAX_EXPERTS];
  int16_t admitted[DALI_MAX_EXPERTS];
  int32_t workload[DALI_MAX_EXPERTS]; /* realised workloads of this layer  */
  /* cache insertions outside the window (baseline policies): LRU miss
   * inserts and demand toggles act on this layer, prefetch toggles on
   * layer+1; ins_kind 0 = lru, 1 = demand, 2 = prefetch */
  int16_t ins_victim[DALI_MAX_EXPERTS];
  int16_t ins_expert[DALI_MAX_EXPERTS];
  int8_t ins_kind[DALI_MAX_EXPERTS];
} dali_layer_record;

/* Scalar knobs of the fused per-layer policy step (SimConfig,
 * simulator.py:45-74). */
typedef struct dali_policy_config {
  int32_t L, N, k;
  int32_t assignment;        /* 0 = greedy, 1 = all-cpu, 2 = all-gpu,
                              * 3 = beam, 4 = optimal (branch and bound),
                              * 5 = static-threshold (assignment.py:202-402) */
  int32_t gpu_capacity;      /* < 0 = unlimited                             */
  int32_t prefetch_size;     /* 0 = prefetch off                            */
  int32_t cache_enabled;
  int32_t w_size, u_size;
  int32_t has_shared;        /* num_shared_experts > 0                      */
  int32_t all_resident;      /* every expert in HBM (roofline reference)     */
  int32_t cache_policy;      /* 0 = workload, 1 = lru, 2 = score            */
  int32_t insert_demand;     /* insert_demand_fetched toggle                */
  int32_t insert_prefetched; /* insert_prefetched toggle                    */
  int32_t beam_width;        /* 1..DALI_MAX_BEAM                            */
  int32_t exact_solver_limit;
  int32_t has_threshold;     /* static-threshold: 0 = median of positives   */
  int32_t pad;
  double scheduling_overhead_ms;
  double solver_node_cost_ms;
  double prefetch_compute_ms;
  double non_moe;            /* resolved non_moe_override / table value     */
  double threshold;
} dali_policy_config;

#define DALI_MAX_BEAM 32

/* ---- library ----------------------------------------------------------- */
const char* dali_last_error(void);
int dali_version(void);
/* Number of kernel launches issued by this library since load (for the
 * bench's gpu_launches claim). */
int64_t dali_launch_count(void);

/* ---- host expert store --------------------------------------------------
 * Page-locked host memory for the per-(layer, expert) weight blocks that
 * the H2D copy stream and the CPU expert worker read: anonymous mmap with
 * transparent huge pages, parallel first touch on `nthreads` threads, then
 * cudaHostRegister (portable).  Exact size (no power-of-two rounding). */
int dali_host_alloc(size_t bytes, int32_t nthreads, void** out);
int dali_host_free(void* p, size_t bytes);
/* Shared variant for one store per node (data-parallel replicas): with
 * create != 0 a memfd of `bytes` is created, touched and registered and its
 * descriptor returned in *fd; with create == 0 the owner's memfd is opened
 * through /proc/<owner_pid>/fd/<*fd> (or, with owner_pid < 0, *fd is a
 * descriptor this process already holds, e.g. received with SCM_RIGHTS),
 * mapped MAP_SHARED and registered. */
int dali_host_alloc_shared(size_t bytes, int32_t nthreads, int32_t create,
                           int32_t* fd, int32_t owner_pid, void** out);

/* ---- (1) gating: route + softmax + stable top-k + histogram --------------
 * Replaces derive_workloads / gate_scores / topk_indices
 * (trace.py:229-265) and, with `residual` != NULL, the residual shift of
 * predict_next_layer (prefetch.py:127-136).
 *   hidden   [dev] (T, d) row-major, f64 or bf16 (raw uint16 bits)
 *   residual [dev] (d,) f64 added to every row first, or NULL
 *   gate     [dev] (d, N) row-major, f64 or bf16 (layout of GateParams,
 *            trace.py:89-113)
 *   topk_idx [dev] (T, k) int32 or NULL; topk_w [dev] (T, k) f32 or NULL
 *            (selected softmax probabilities; renormalised over the k when
 *            renorm != 0)
 *   workloads[dev] (N,) int64, overwritten.
 * Arithmetic: fp64 products and sums, fp64 softmax; ranks by descending
 * probability with ties to the lower index. */
int dali_route_f64(const double* hidden, const double* residual,
                   const double* gate, int64_t T, int32_t d, int32_t N,
                   int32_t k, int32_t renorm, int32_t* topk_idx,
                   float* topk_w, int64_t* workloads, void* stream);
int dali_route_bf16(const uint16_t* hidden, const double* residual,
                    const uint16_t* gate, const float* gate_norm2, int64_t T,
                    int32_t d, int32_t N,
                    int32_t k, int32_t renorm, int32_t* topk_idx,
                    float* topk_w, int64_t* workloads, void* stream);

/* bf16 inputs take the certified fp32 path when d % 8 == 0, 4 <= N <= 256,
 * N % 4 == 0 and gate_norm2 != NULL (csrc/route_guard.cu; gate_norm2 [dev]
 * (N,) f32 = squared column norms of `gate`, an upper bound is enough):
 * fp32 FFMA logits, and a row whose k+1
 * leading logits are not separated by the rigorous summation-error bound
 * gamma_H * ||x|| * (||W_:a|| + ||W_:b||) is recomputed in fp64 as above.
 * Indices and workloads equal the fp64 path's; topk_w of certified rows is
 * an fp32 softmax.  Fire counter (rows recomputed / rows routed since the
 * last reset) and a test hook scaling the bound (scale < 0: every row takes
 * the fp64 recompute). */
int dali_route_fire_count(uint64_t* fires, uint64_t* rows, int32_t reset);
/* dali_route_bf16 (no residual) followed by dali_moe_plan_permute, in ONE
 * launch for decode-sized batches (T <= 16, T*k + N < 256): the routing
 * kernel's batch-owning CTA computes the plan and gathers the permuted rows
 * (derive_workloads + the engine's permute; trace.py:253-265).  Larger
 * batches run the two as separate launches.  Outputs as the two functions'. */
int dali_route_plan_bf16(const uint16_t* hidden, const uint16_t* gate, const float* gate_norm2,
                         int64_t T, int32_t d, int32_t N, int32_t k, int32_t renorm,
                         int32_t* topk_idx, float* topk_w, int64_t* workloads,
                         int32_t* offsets, int32_t* perm_token, int32_t* pos, uint16_t* xp,
                         void* stream);
int dali_route_guard_scale(double scale);
/* A/B hook for T > 16 batches: 0 picks by shape, 1 forces the round-1
   d-chunked kernel, 2 the fixed-geometry prefill kernel (same outputs). */
int dali_route_prefill_variant(int32_t variant);

/* Prefetch-set selection: stable top-P of predicted workloads
 * (prefetch.py:153-156).  predicted [dev] (N,) int64 -> set [dev] (P,) i32 */
int dali_prefetch_select(const int64_t* predicted, int32_t N, int32_t P,
                         int32_t* set, void* stream);

/* Per-token gate scores softmax(hidden @ W_g) in fp64 (gate_scores,
 * trace.py:242-250) -> probs [dev] (T, N) f64; the score cache policy sums
 * them over tokens (simulator.py:426-429).  Same arithmetic as dali_route. */
int dali_gate_probs_f64(const double* hidden, const double* gate, int64_t T,
                        int32_t d, int32_t N, double* probs, void* stream);
int dali_gate_probs_bf16(const uint16_t* hidden, const uint16_t* gate,
                         int64_t T, int32_t d, int32_t N, double* probs,
                         void* stream);

/* ---- (2) greedy assignment (single CTA) ----------------------------------
 * Replaces AssignmentInstance times + sorted_order + greedy_assign
 * (assignment.py:53-123,172-199; cost_model.py:19-27,70-103).
 * If cpu_times/gpu_times are NULL they are evaluated on device from *cm
 * (no-FMA np.interp formula); otherwise the given times are used
 * (AssignmentInstance.from_times, assignment.py:81-103).
 *   workloads [dev] (N,) int64; resident [dev] (N,) uint8
 *   gpu_capacity < 0 means None.
 *   C, G [dev] (N,) int8; order [dev] (N,) int32 (-1 padded);
 *   times_out [dev] (2N,) f64 or NULL (cpu times then gpu times). */
int dali_greedy(const int64_t* workloads, const uint8_t* resident, int32_t N,
                int32_t gpu_capacity, const dali_cost_model* cm,
                const double* cpu_times, const double* gpu_times, int8_t* C,
                int8_t* G, int32_t* order, double* times_out, void* stream);

/* Cost-model evaluation only (CostModel.t_cpu / t_gpu_compute, batch).
 *   w [dev] (n,) f64 -> cpu_out, gpu_out [dev] (n,) f64 */
int dali_cost_eval(const dali_cost_model* cm, const double* w, int64_t n,
                   double* cpu_out, double* gpu_out, void* stream);

/* ---- (4) workload-aware cache window update (single CTA) -----------------
 * Replaces record_and_maybe_replace for the workload policy
 * (cache.py:146-214).  State lives on device:
 *   on_gpu [dev] (N,) uint8, scores [dev] (N,) f64,
 *   counters [dev] int32[2] = {tokens_in_window, stopped}
 *   workload [dev] (N,) f64 (the reference casts to float64)
 *   ev [dev] int32[2 + 2*DALI_MAX_EXPERTS] =
 *        {valid, n_swap, evicted[u]..., admitted[u]...} */
int dali_cache_record(uint8_t* on_gpu, double* scores, int32_t* counters,
                      int32_t N, int32_t w_size, int32_t u_size,
                      const double* workload, int32_t is_eos, int32_t* ev,
                      void* stream);

/* One assignment instance with any reference solver (assignment.py:172-402):
 *   policy 0 greedy, 1 all-cpu, 2 all-gpu, 3 beam (beam_width <= DALI_MAX_BEAM),
 *   4 optimal (branch and bound; *nodes = explored nodes, -1 when more than
 *   exact_solver_limit experts are activated -- the caller raises), 5
 *   static-threshold (has_threshold = 0: median positive workload).
 *   Times from the cost model or explicit [dev] vectors as in dali_greedy;
 *   C, G [dev] (N,) int8; nodes [dev] int64 (may be NULL). */
int dali_assign(int32_t policy, const int64_t* workloads, const uint8_t* resident,
                int32_t N, int32_t gpu_capacity, const dali_cost_model* cm,
                const double* cpu_times, const double* gpu_times, int32_t beam_width,
                int32_t exact_solver_limit, int32_t has_threshold, double threshold,
                int8_t* C, int8_t* G, int64_t* nodes, void* stream);

/* One cache operation on a layer's state (cache.py:104-143): op 0 = lookup
 * (LRU: clock tick, refresh on hit, insert + evict least recently used on a
 * miss), op 1 = force_insert (evict the lowest score / oldest clock).
 *   on_gpu [dev] (N,) u8, scores [dev] (N,) f64, lru_state [dev] (N+1) i64
 *   (clock last; may be NULL unless use_lru); out [dev] int32[2] =
 *   {hit | inserted, victim or -1}. */
int dali_cache_op(uint8_t* on_gpu, const double* scores, int64_t* lru_state, int32_t N,
                  int32_t use_lru, int32_t expert, int32_t op, int32_t* out, void* stream);

/* ---- fused per-layer policy step -----------------------------------------
 * One single-CTA kernel per (step, layer) that performs, in the reference
 * driver's order (simulator.py:359-444): residency = cache | arrived,
 * cost evaluation + greedy, GPU-lane timeline, cache lookups of the GPU
 * experts, prefetch candidates for layer+1 and the virtual-clock arrival
 * rule, and the cache window update; the decision is written to *rec
 * (device or mapped-host memory).
 *   workloads [dev] (N,) int64 this layer's true workloads
 *   predicted [dev] (N,) int64 residual-predicted workloads of layer+1
 *             (NULL when prefetch is off or layer == L-1)
 *   on_gpu    [dev] (L, N) uint8 cache residency, updated in place
 *   scores    [dev] (L, N) f64 window scores, updated in place
 *   counters  [dev] (L, 2) int32 {window, stopped}, updated in place
 *   arrived   [dev] (L, N) uint8 prefetched-and-arrived flags of the
 *             current step; row layer+1 is written, row layer is consumed
 *   slot_of   [dev] (L, N) int32 HBM slot per cached expert or -1; swaps
 *             move the victim's slot to the admitted expert (may be NULL)
 *   lru_state [dev] (L, N+1) int64 LRU clocks (+ the layer's clock last);
 *             used by cache_policy 1 (may be NULL otherwise)
 *   gate_probs [dev] (n_tokens, N) f64 this layer's gate scores
 *             (dali_gate_probs); used by cache_policy 2 (may be NULL)
 * predicted also carries the statistical / random predictors' vectors
 * (frequency-table row, permutation): the kernel only ranks it.
 */
int dali_policy_layer(const dali_policy_config* cfg, const dali_cost_model* cm,
                      int32_t step, int32_t layer, int32_t token_index,
                      int32_t is_eos, const int64_t* workloads,
                      const int64_t* predicted, uint8_t* on_gpu,
                      double* scores, int32_t* counters, uint8_t* arrived,
                      int32_t* slot_of, int64_t* lru_state,
                      const double* gate_probs, int32_t n_tokens,
                      dali_layer_record* rec, void* stream);

/* Same step with the per-step scalars read from a DEVICE descriptor so the
 * launch can live inside a CUDA graph replayed every decode step:
 *   desc [dev] int32[8] = {step, token_index, eos_at_step, record_index,
 *                          pos, len, L, unused}
 *   is_eos = (step == eos_at_step); the record written is
 *   rec_base[record_index + layer].  dali_step_advance moves the
 *   descriptor to the next step (step, token_index, pos, len += 1;
 *   record_index += L) on device. */
int dali_policy_layer_desc(const dali_policy_config* cfg,
                           const dali_cost_model* cm, int32_t layer,
                           const int32_t* desc, const int64_t* workloads,
                           const int64_t* predicted, uint8_t* on_gpu,
                           double* scores, int32_t* counters, uint8_t* arrived,
                           int32_t* slot_of, int64_t* lru_state,
                           const double* gate_probs, int32_t n_tokens,
                           dali_layer_record* rec_base, void* stream);
int dali_step_advance(int32_t* desc, void* stream);

/* ---- (5) expert execution -------------------------------------------------
 * Plan: stable counting sort of the T*k (token, slot) pairs by expert.
 *   topk_idx [dev] (T,k) i32 -> offsets [dev] (N+1) i32,
 *   perm_token [dev] (T*k) i32 (source token of each permuted row),
 *   pos [dev] (T,k) i32 (permuted row of each (token, slot)) */
int dali_moe_plan(const int32_t* topk_idx, int64_t T, int32_t k, int32_t N,
                  int32_t* offsets, int32_t* perm_token, int32_t* pos,
                  void* stream);

/* dali_moe_plan followed by dali_permute; decode-sized batches (T*k <= 64)
 * do both in one single-CTA launch.  x (T, d) bf16 [dev] -> xp (T*k, d). */
int dali_moe_plan_permute(const int32_t* topk_idx, int64_t T, int32_t k, int32_t N,
                          const uint16_t* x, int32_t d, int32_t* offsets,
                          int32_t* perm_token, int32_t* pos, uint16_t* xp,
                          void* stream);

/* Coalesced 128-bit gather: out[r,:] = x[perm_token[r],:]  (bf16, d % 8 == 0) */
int dali_permute(const uint16_t* x, const int32_t* perm_token, int64_t rows,
                 int32_t d, uint16_t* out, void* stream);

/* Grouped SwiGLU expert FFN over the experts with expert_ptr[e] != 0.
 *   xp   [dev] (rows, d) bf16 permuted tokens, rows grouped by offsets
 *   expert_ptr [dev] (N,) u64: base address of expert e's weight block
 *        [W13 interleaved (2f, d) | W2 (d, f)] bf16, or 0 = not on GPU
 *   hbuf [dev] (rows, f) bf16 workspace; yp [dev] (rows, d) f32 out.
 *   Rows of experts with expert_ptr[e] == 0 are left untouched. */
int dali_expert_ffn(const uint16_t* xp, const int32_t* offsets, int32_t N,
                    const uint64_t* expert_ptr, int32_t d, int32_t f,
                    int64_t rows, int32_t max_rows_per_expert, uint16_t* hbuf,
                    float* yp, void* stream);

/* Same contract, forcing the weight-streaming CUDA-core kernels (one warp
 * per weight row, 8 tokens per pass) used for small per-expert token counts. */
int dali_expert_ffn_simt(const uint16_t* xp, const int32_t* offsets, int32_t N,
                         const uint64_t* expert_ptr, int32_t d, int32_t f,
                         uint16_t* hbuf, float* yp, void* stream);

/* Tensor-core path (tcgen05 + TMA), same FFN contract as dali_expert_ffn:
 *   expert_maps [dev] (N,) u64: device address of expert e's 256-byte pair of
 *       CUtensorMaps (W13 map, W2 map; built by dali_expert_maps), 0 = the
 *       expert is not on the GPU.
 *   max_rows_per_expert selects the token tile BN in {16,32,64,128,256};
 *   n_gpu_experts bounds the grid; yp is `splits` planes of (rows, d) f32
 *   (split-K of the down projection; splits must divide f/64). */
int dali_expert_ffn_tc(const uint16_t* xp, const int32_t* offsets, int32_t N,
                       const uint64_t* expert_maps, int32_t d, int32_t f,
                       int64_t rows, int32_t max_rows_per_expert,
                       int32_t n_gpu_experts, uint16_t* hbuf, float* yp,
                       int32_t splits, void* stream);

/* Host: encode the two weight tensor maps of one expert block at device
 * address `block` into out[256] (host memory; copy it to device memory). */
int dali_expert_maps(const void* block, int32_t d, int32_t f, void* out);

/* Eq. (2) combine fused with the residual add and 128-bit scatter:
 *   out[t,:] = x[t,:] + sum_j w[t,j] * row(t,j) (+ extra[t,:]),
 *   row(t,j) = sum_{s<splits} yp[s][pos[t,j],:]   if gpu_mask == NULL or
 *                                                 gpu_mask[idx[t,j]] (GPU expert)
 *            = cpu_rows[pos[t,j],:]               otherwise, if cpu_rows != NULL
 *              (rows the host worker computed for CPU-assigned experts)
 * x, out [dev] (T,d) bf16 (may alias); yp splits x (rows,d) f32; cpu_rows
 * (rows,d) f32 or NULL; topk_idx / pos / topk_w (T,k); gpu_mask [dev] (N,)
 * int8 (the G vector); extra (T,d) f32 token-level addend (shared experts)
 * or NULL. */
int dali_unpermute_combine(const uint16_t* x, const float* yp,
                           const int32_t* topk_idx, const int32_t* pos,
                           const float* topk_w, const int8_t* gpu_mask,
                           const float* cpu_rows, const float* extra, int64_t T,
                           int32_t k, int32_t d, int32_t splits, int64_t rows,
                           uint16_t* out, void* stream);

/* Same as dali_unpermute_combine, launchable before the host worker has
 * produced the CPU experts' rows: every CTA first waits until the mapped
 * pinned word *rows_ready (stored by the worker's last unit, see
 * dali_cpu_submit_layer) is >= rows_want.  rows_ready NULL = no wait.  The
 * wait is bounded (4 s of device time; dali_host_wait_timeouts counts
 * expiries).  The word is polled with ld.global.cv (never a stale L2
 * line); the rows are read once after it. */
int dali_unpermute_combine_wait(const uint16_t* x, const float* yp,
                                const int32_t* topk_idx, const int32_t* pos,
                                const float* topk_w, const int8_t* gpu_mask,
                                const float* cpu_rows, const float* extra, int64_t T,
                                int32_t k, int32_t d, int32_t splits, int64_t rows,
                                uint16_t* out, const uint64_t* rows_ready,
                                uint64_t rows_want, void* stream);
int dali_host_wait_timeouts(uint64_t* out, int32_t reset);

/* Engine plumbing: copy nbytes between UVA addresses (device memory and/or
 * mapped pinned host memory, either direction) with a kernel instead of a
 * copy engine, so small per-layer control transfers and per-token reads never
 * queue behind expert-block DMA.  16-byte aligned pointers take the vector
 * path; unaligned copies are byte-wise and limited to 1 MiB. */
int dali_copy_mapped(void* dst, const void* src, int64_t nbytes, void* stream);
/* Two 16-byte aligned ranges in one kernel launch (same copies as two
 * dali_copy_mapped calls): the decode head's D2H mirrors of the routing block
 * and the permuted rows the CPU experts read. */
int dali_copy_mapped2(void* dst0, const void* src0, int64_t n0, void* dst1,
                      const void* src1, int64_t n1, void* stream);
/* Engine plumbing: cudaMemcpyAsync(cudaMemcpyDefault) of nbytes on `stream`
 * -- the copy-engine expert-block transfers (pinned host store -> HBM cache
 * slot / staging slot) without a host-side stream switch.  The H2D leg of
 * the prefetch and cache-replacement transfers (simulator.py:398-420 times
 * them; moesim moves no bytes). */
int dali_memcpy_async(void* dst, const void* src, size_t nbytes, void* stream);

/* Engine plumbing: bulk host->device copy (expert blocks) driven by `nctas`
 * CTAs of 512 threads reading mapped pinned memory, instead of a copy engine.
 * The CTA count bounds the bytes in flight on PCIe, so latency-critical small
 * transfers issued meanwhile are not queued behind a copy engine's deep read
 * queue.  Pointers and size must be 16-byte aligned. */
int dali_copy_h2d_sm(void* dst, const void* src, int64_t nbytes, int32_t nctas, void* stream);

/* Shared expert(s) finish (engine plumbing): out[t,:] = sum over `splits`
 * planes of ys (splits, T, d) f32, times sigmoid(h[t,:] . gate_w) when
 * gate_w (d,) bf16 is given (Qwen-style gated shared expert), else 1.
 * h (T, d) bf16; out (T, d) f32 [dev]. */
int dali_shared_finish(const float* ys, int32_t splits, int64_t T, int32_t d,
                       const uint16_t* h, const uint16_t* gate_w, float* out, void* stream);

/* Decode GEMV (engine plumbing, attention projections): y (B, M) bf16 =
 * x (B, K) bf16 . W^T with W (M, K) bf16 row-major, 1 <= B <= 8, K % 8 == 0;
 * fp32 accumulation, weight-streaming (one warp per output row). */
int dali_gemv_bf16(const uint16_t* x, const uint16_t* w, int32_t B, int32_t M, int32_t K,
                   uint16_t* y, void* stream);

/* Decode GEMV with the attention block's RMSNorms fused in (engine plumbing;
 * same arithmetic as dali_add_rmsnorm + dali_gemv_bf16, bit for bit):
 *   norm_in_w != NULL: the GEMV input is RMSNorm(x) * norm_in_w (x is the raw
 *     residual stream; eps as in dali_add_rmsnorm);
 *   res != NULL (M == row width): after y, x2_out = res + y and
 *     h_out = RMSNorm(x2_out) * norm_out_w, computed by the last CTA to
 *     finish (counter [dev] u32, zero-initialised, left zero).
 * 1 <= B <= 8, K % 8 == 0, M % 8 == 0, M >= 16. */
int dali_gemv_norm_bf16(const uint16_t* x, const uint16_t* w, int32_t B, int32_t M, int32_t K,
                        uint16_t* y, const uint16_t* norm_in_w, float eps, const uint16_t* res,
                        const uint16_t* norm_out_w, uint16_t* x2_out, uint16_t* h_out,
                        uint32_t* counter, void* stream);
/* Engine plumbing: fused residual add + RMSNorm over (T, d) bf16 rows:
 *   x_out = x + a (a may be NULL: x_out untouched, x used as is);
 *   h = bf16(bf16(x_out * rsqrt(mean(x_out^2) + eps)) * w). */
int dali_add_rmsnorm(const uint16_t* x, const uint16_t* a, const uint16_t* w,
                     float eps, int64_t T, int32_t d, uint16_t* x_out,
                     uint16_t* h, void* stream);

/* Decode attention plumbing (one query token per sequence; position and
 * valid length read from device scalars, graph-capturable):
 *   dali_rope_append: qkv (B, (H+2KV)*hd) bf16 -> q (B,H,hd) rotated (rotate-
 *     half RoPE, fp32 tables cos/sin (max_pos, hd/2)); rotated k and v stored
 *     at *pos in caches laid out (B, KV, max_len, hd).
 *   dali_decode_attention: split-K GQA attention over positions [0, *len),
 *     head_dim 64 or 128; workspace f32 (B*H*splits*(hd+2)). */
int dali_rope_append(const uint16_t* qkv, const float* cos_t, const float* sin_t,
                     const int32_t* pos, int32_t B, int32_t H, int32_t KV,
                     int32_t hd, int32_t max_len, uint16_t* q_out,
                     uint16_t* k_cache, uint16_t* v_cache, void* stream);
int dali_decode_attention(const uint16_t* q, const uint16_t* k_cache,
                          const uint16_t* v_cache, const int32_t* len, int32_t B,
                          int32_t H, int32_t KV, int32_t hd, int32_t max_len,
                          int32_t splits, float scale, float* workspace,
                          uint16_t* out, void* stream);

/* ---- expert-parallel exchange over peer memory ---------------------------
 * The EP MoE layer's dispatch and return all-to-alls, fused with the permute
 * / unpermute around them: ranks store rows straight into each other's
 * receive buffers (CUDA IPC mappings over NVLink/NVSwitch) and bump a
 * system-scope arrival counter (one per rank and direction) instead of
 * calling a collective.  Per-rank buffer (dali_ep_layout, out[5] =
 * {recv, ret, cnt, flags, total} byte offsets):
 *   recv [G][cap][d] bf16, ret [G][cap][d] f32, cnt [G][NL] i32, flags u64[2].
 * Source block s of a receiver's recv / ret is written only by rank s.
 *   dali_ipc_alloc / open / close / free: cudaMalloc + IPC handles (64 B).
 *   dali_ep_dispatch: row r of this rank's permuted rows (grouped by global
 *     expert by dali_moe_plan; offsets (N+1) [dev]) -> owner q = e / NL at
 *     recv_q[rank][r - offsets[q*NL]] (gathered from x via perm_token),
 *     counts -> cnt_q[rank][:]; then every peer's flags[0] += 1.
 *   dali_ep_wait: spin until *flag >= target (bounded; *err = 1 on timeout).
 *   dali_ep_recv: cnt (G, NL) -> grouped order (local expert, source):
 *     offs_l (NL+1), workloads (NL) i64, meta[0] = rows, and the regrouped
 *     rows out (rows, d) bf16.
 *   dali_ep_return: grouped result rows (sum of `splits` planes of yp, or
 *     cpu_rows where gmask[j] == 0) -> ret_s[rank][idx] of their source s;
 *     then every peer's flags[1] += 1.
 *   dali_ep_gather_back: ret (G, cap, d) -> back (rows, d) f32 in this
 *     rank's permuted order (for dali_unpermute_combine with splits 1).
 * peer_* are [dev] (G,) u64 tables of the ranks' buffer addresses. */
int dali_ipc_alloc(size_t bytes, void** ptr, void* handle);
int dali_ipc_open(const void* handle, void** ptr);
int dali_ipc_close(void* ptr);
int dali_ipc_free(void* ptr);
int dali_ep_layout(int32_t G, int32_t NL, int64_t cap, int32_t d, int64_t* out);
int dali_ep_dispatch(const uint16_t* x, const int32_t* perm_token, const int32_t* offsets,
                     int32_t N, int32_t NL, int32_t G, int32_t rank, int64_t cap, int32_t d,
                     int64_t max_rows, const uint64_t* peer_recv, const uint64_t* peer_cnt,
                     const uint64_t* peer_flag, void* stream);
int dali_ep_wait(const uint64_t* flag, uint64_t target, int64_t max_spins, int32_t* err,
                 void* stream);
int dali_ep_recv(const int32_t* cnt, int32_t G, int32_t NL, int64_t cap, const uint16_t* recv,
                 int32_t d, int64_t max_rows, int32_t* perm2, int32_t* offs_l,
                 int64_t* workloads, int32_t* meta, uint16_t* out, void* stream);
int dali_ep_return(const float* yp, int32_t splits, int64_t plane, const float* cpu_rows,
                   const int8_t* gmask, const int32_t* offs_l, const int32_t* cnt, int32_t G,
                   int32_t NL, int32_t rank, int64_t cap, int32_t d, int64_t max_rows,
                   const uint64_t* peer_ret, const uint64_t* peer_flag, void* stream);
int dali_ep_gather_back(const float* ret, const int32_t* offsets, int32_t N, int32_t NL,
                        int64_t cap, int32_t d, int64_t max_rows, float* back, void* stream);

/* ---- CPU expert worker (host; DALI hybrid execution) ---------------------
 * SwiGLU of R token rows x (R, d) bf16 [host] with one expert block [host]
 * (the engine's W13/W2 layout), y (R, d) f32 [host]; AVX-512 BF16
 * weight-streaming kernel on a persistent pool of `nthreads` threads.  The
 * SwiGLU intermediate is rounded to bf16 like the GPU kernel's. */
int dali_cpu_expert(const uint16_t* block, int32_t d, int32_t f,
                    const uint16_t* x, int32_t R, float* y, int32_t nthreads);
/* R > 16 rows (prefill) run on AMX-BF16 tiles when the host has them (1 if
 * so; DALI_CPU_AMX=0 disables): fp32 accumulation and fp32 outputs, only the
 * SwiGLU intermediate rounded to bf16 -- the GPU kernel's rounding points.
 * Without AMX the rows are processed 16 at a time by the AVX-512 kernel. */
int dali_cpu_expert_amx_available(void);

/* Asynchronous form for the engine: experts i < n (block[i], rows x[i]
 * (rows[i] <= 16, d) bf16 -> y[i] (rows[i], d) f32, [host] pointers as
 * uint64) start on the pool's worker threads and the call returns at once,
 * so the caller can dispatch the GPU side of the same layer.  The work is a
 * queue of stages (expert i gate/up, expert i down, ...) cut into ~1 MB
 * units; dali_cpu_expert_wait makes the caller take the remaining units and
 * returns when all are done.  One submission in flight: a second submit, or
 * a synchronous dali_cpu_expert call, before the wait returns DALI_ESIM. */
int dali_cpu_expert_submit(int32_t n, const uint64_t* blocks, const uint64_t* xs,
                           const int32_t* rows, const uint64_t* ys, int32_t d,
                           int32_t f, int32_t nthreads);
int dali_cpu_expert_wait(void);

/* One decode layer's CPU experts in one call (engine hot path): the experts e
 * with C[e] != 0 (the decision record's C vector) and rows offsets[e] ..
 * offsets[e+1] of the permuted activations xp (R, d) bf16 are started on the
 * worker pool, results into out (R, d) f32 (rows of other experts untouched).
 * blocks (N,) = host address of each expert's weight block.  When the job's
 * last work unit finishes (at once if there is none), done_value is stored
 * to *done_flag (release) -- the word dali_unpermute_combine_wait polls.
 * *n_experts = experts started, or -1 if an expert has more than 16 rows
 * (nothing started, flag untouched: prefill-sized work goes through
 * dali_cpu_expert).  Join with dali_cpu_expert_wait. */
int dali_cpu_submit_layer(const int8_t* C, const int32_t* offsets, int32_t N,
                          const uint64_t* blocks, const uint16_t* xp, float* out,
                          int32_t d, int32_t f, int32_t nthreads, uint64_t* done_flag,
                          uint64_t done_value, int32_t* n_experts);

/* Deterministic counter-hash weight init (uniform, given std):
 * out[i] = bf16(std * sqrt(3) * (2*u(seed, offset+i) - 1)). */
int dali_init_uniform_bf16(uint16_t* out, int64_t n, uint64_t seed,
                           uint64_t offset, float stdev, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DALI_H_ */
