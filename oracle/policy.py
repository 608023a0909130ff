"""numpy restatement of the reference hot-path policies (TEST INFRASTRUCTURE).

Every function cites the reference file:line (relative to
``/root/reference/pkg/src/moesim``) whose behaviour it restates.  The
restatement is independent code: it is pinned against the reference itself
through the frozen fixtures in ``tests/golden`` (see ``make_golden.py``).

Exactness notes
---------------
* Gating ranks fp64 softmax scores with a stable descending sort (ties go to
  the lower expert index), exactly as ``trace.py:229-265``.
* ``interp_ms`` evaluates numpy's ``np.interp`` formula
  ``slope*(w - x[j]) + y[j]`` with the slope computed first and no fused
  multiply-add; in Python this is bit-identical to ``np.interp`` and to the
  CUDA kernel compiled with ``-fmad=false``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Gating (reference trace.py:229-265)
# ---------------------------------------------------------------------------


def row_softmax(logits: np.ndarray) -> np.ndarray:
    """Max-shifted softmax over the last axis (trace.py:229-233)."""
    shifted = logits - np.max(logits, axis=-1, keepdims=True)
    ex = np.exp(shifted)
    return ex / np.sum(ex, axis=-1, keepdims=True)


def stable_topk(values, k: int) -> np.ndarray:
    """k largest entries, ties toward the lower index (trace.py:236-239)."""
    v = np.asarray(values, dtype=np.float64)
    return np.argsort(-v, kind="stable")[:k]


def gate_probs(hidden, gate_matrix) -> np.ndarray:
    """softmax(hidden @ W_g) in fp64 (trace.py:242-250)."""
    h = np.atleast_2d(np.asarray(hidden, dtype=np.float64))
    g = np.asarray(gate_matrix, dtype=np.float64)
    if h.shape[1] != g.shape[0]:
        raise ValueError(f"hidden dim {h.shape[1]} does not match gate matrix "
                         f"rows {g.shape[0]}")
    return row_softmax(h @ g)


def route(hidden, gate_matrix, k: int):
    """Per-token top-k experts, their scores, and the per-expert histogram.

    Restates ``derive_workloads`` (trace.py:253-265) and additionally returns
    the per-token selection so the routing kernel's index output can be
    compared.  Returns (topk_idx (T,k) int64, topk_score (T,k) f64,
    workloads (N,) int64).
    """
    probs = gate_probs(hidden, gate_matrix)
    T, N = probs.shape
    if not 1 <= k <= N:
        raise ValueError(f"top_k {k} out of range for {N} experts")
    # stable argsort on the negated rows == per-row topk_indices
    order = np.argsort(-probs, axis=1, kind="stable")[:, :k]
    hist = np.bincount(order.reshape(-1), minlength=N).astype(np.int64)
    score = np.take_along_axis(probs, order, axis=1)
    return order.astype(np.int64), score, hist


def derive_workloads(hidden, gate_matrix, k: int) -> np.ndarray:
    return route(hidden, gate_matrix, k)[2]


# ---------------------------------------------------------------------------
# Cost model (reference cost_model.py:19-155)
# ---------------------------------------------------------------------------


def interp_ms(w: float, xs, ys) -> float:
    """Piecewise-linear lookup with last-segment extrapolation.

    Restates ``_interp`` (cost_model.py:19-27), which defers to ``np.interp``
    inside the table.  numpy evaluates ``slope*(x - xp[j]) + fp[j]`` for
    ``xp[j] <= x < xp[j+1]``, returns ``fp[j]`` on an exact knot and ``fp[-1]``
    at or beyond the last knot; beyond it the reference extrapolates with the
    last segment's slope.
    """
    n = len(xs)
    if w > xs[-1]:
        slope = (ys[-1] - ys[-2]) / (xs[-1] - xs[-2]) if n >= 2 else 0.0
        return float(ys[-1] + slope * (w - xs[-1]))
    if w >= xs[-1]:
        return float(ys[-1])
    if w <= xs[0]:
        return float(ys[0])
    j = int(np.searchsorted(xs, w, side="right")) - 1
    if w == xs[j]:
        return float(ys[j])
    slope = (ys[j + 1] - ys[j]) / (xs[j + 1] - xs[j])
    return float(slope * (w - xs[j]) + ys[j])


@dataclass
class CostTables:
    """Sample tables incl. the (0,0) anchor (cost_model.py:54-68)."""

    cpu_xs: np.ndarray
    cpu_ys: np.ndarray
    gpu_xs: np.ndarray
    gpu_ys: np.ndarray
    trans_time: float
    shared_expert_gpu_time: float = 0.0
    non_moe_layer_time: float = 0.0

    def t_cpu(self, w) -> float:
        return 0.0 if w == 0 else interp_ms(w, self.cpu_xs, self.cpu_ys)

    def t_gpu_compute(self, w) -> float:
        return 0.0 if w == 0 else interp_ms(w, self.gpu_xs, self.gpu_ys)

    def t_gpu(self, w, resident) -> float:
        if w == 0:
            return 0.0
        return max(0.0 if resident else self.trans_time, self.t_gpu_compute(w))


def tables_from_samples(cpu_samples, gpu_samples, trans_time,
                        shared_expert_gpu_time=0.0, non_moe_layer_time=0.0):
    """Anchor and sort samples (restates fit_cost_model, cost_model.py:117-138;
    validation errors are the product's job, the oracle assumes valid input)."""
    def table(samples):
        pts = sorted((float(a), float(b)) for a, b in samples)
        xs, ys = [0.0], [0.0]
        for a, b in pts:
            if a == 0.0 and b == 0.0:
                continue
            xs.append(a)
            ys.append(b)
        return np.asarray(xs), np.asarray(ys)
    cx, cy = table(cpu_samples)
    gx, gy = table(gpu_samples)
    return CostTables(cx, cy, gx, gy, float(trans_time),
                      float(shared_expert_gpu_time), float(non_moe_layer_time))


def default_tables(shared_expert_gpu_time=0.0, non_moe_layer_time=0.0):
    """The bundled "3090-like" profile (cost_model.py:141-155)."""
    return tables_from_samples([(1, 2.0), (16, 32.0), (64, 128.0), (256, 512.0)],
                               [(1, 0.10), (16, 1.60), (64, 6.40), (256, 25.6)],
                               3.0, shared_expert_gpu_time, non_moe_layer_time)


# ---------------------------------------------------------------------------
# Greedy assignment (reference assignment.py:53-199)
# ---------------------------------------------------------------------------


def expert_times(tables: CostTables, workloads, resident):
    """Per-expert CPU and GPU times (assignment.py:75-79)."""
    cpu = np.array([tables.t_cpu(int(w)) for w in workloads], dtype=np.float64)
    gpu = np.array([tables.t_gpu(int(w), bool(r))
                    for w, r in zip(workloads, resident)], dtype=np.float64)
    return cpu, gpu


def visit_order(workloads, cpu_t, gpu_t) -> np.ndarray:
    """Activated experts by descending |gpu-cpu|, ties to lower index
    (assignment.py:119-123)."""
    act = np.flatnonzero(np.asarray(workloads) > 0)
    gap = np.abs(gpu_t[act] - cpu_t[act])
    return act[np.argsort(-gap, kind="stable")]


def greedy(workloads, resident, cpu_t, gpu_t, capacity=None):
    """Algorithm 1 with the transfer-slot guard (assignment.py:172-199).

    Returns (C int8[N], G int8[N], order int64[n_act]).
    """
    n = len(workloads)
    C = np.zeros(n, np.int8)
    G = np.zeros(n, np.int8)
    lane_cpu = 0.0
    lane_gpu = 0.0
    slots = capacity
    order = visit_order(workloads, cpu_t, gpu_t)
    for e in order:
        may_gpu = slots is None or slots > 0 or bool(resident[e])
        if may_gpu and lane_gpu + gpu_t[e] <= lane_cpu + cpu_t[e]:
            G[e] = 1
            lane_gpu += gpu_t[e]
            if slots is not None and not resident[e]:
                slots -= 1
        else:
            C[e] = 1
            lane_cpu += cpu_t[e]
    return C, G, order


def all_gpu(workloads, resident, capacity=None):
    """Everything on the GPU, capacity overflow to the CPU (assignment.py:387-402)."""
    w = np.asarray(workloads)
    C = np.zeros(len(w), np.int8)
    G = np.zeros(len(w), np.int8)
    slots = capacity
    for e in np.flatnonzero(w > 0):
        if slots is None or slots > 0 or bool(resident[e]):
            G[e] = 1
            if slots is not None and not resident[e]:
                slots -= 1
        else:
            C[e] = 1
    return C, G


def all_cpu(workloads):
    """All activated experts on the CPU (assignment.py:380-384)."""
    w = np.asarray(workloads)
    return (w > 0).astype(np.int8), np.zeros(len(w), np.int8)


# ---------------------------------------------------------------------------
# Baseline solvers (reference assignment.py:154-402)
# ---------------------------------------------------------------------------


def makespan(cpu_t, gpu_t, C, G):
    """(T_cpu, T_gpu, max) with numpy dot products (assignment.py:154-169)."""
    tc = float(cpu_t @ C)
    tg = float(gpu_t @ G)
    return tc, tg, max(tc, tg)


def beam(workloads, resident, cpu_t, gpu_t, capacity, beam_width: int):
    """Beam search over the greedy visit order (assignment.py:202-247).

    States (t_cpu, t_gpu, used, gpu tuple, cpu tuple); each expands to its
    greedy-preferred child first, children are stably sorted by makespan and
    the first ``beam_width`` survive; the greedy schedule wins if strictly
    better.  Returns (C, G)."""
    order = visit_order(workloads, cpu_t, gpu_t)
    states = [(0.0, 0.0, 0, (), ())]
    for idx in order:
        g, c = float(gpu_t[idx]), float(cpu_t[idx])
        needs = not bool(resident[idx])
        kids = []
        for (tc, tg, used, gs, cs) in states:
            gk = None
            if capacity is None or not needs or used < capacity:
                gk = (tc, tg + g, used + (1 if needs else 0), gs + (int(idx),), cs)
            ck = (tc + c, tg, used, gs, cs + (int(idx),))
            if gk is not None and tg + g <= tc + c:
                kids += [gk, ck]
            elif gk is not None:
                kids += [ck, gk]
            else:
                kids.append(ck)
        kids.sort(key=lambda st: max(st[0], st[1]))
        states = kids[:beam_width]
    best = states[0]
    gC, gG, _ = greedy(workloads, resident, cpu_t, gpu_t, capacity)
    if makespan(cpu_t, gpu_t, gC, gG)[2] < max(best[0], best[1]):
        return gC, gG
    n = len(workloads)
    C = np.zeros(n, np.int8)
    G = np.zeros(n, np.int8)
    G[list(best[3])] = 1
    C[list(best[4])] = 1
    return C, G


def optimal(workloads, resident, cpu_t, gpu_t, capacity, limit: int = 24):
    """Branch and bound for the minimum makespan (assignment.py:268-346):
    lower bound max(Tc, Tg, (Tc+Tg+rem)/2), locally better device first,
    ties toward fewer GPU experts then the smallest sorted GPU index tuple.
    Returns (C, G, nodes); raises ValueError above ``limit`` activated."""
    order = visit_order(workloads, cpu_t, gpu_t)
    n_act = len(order)
    if n_act > limit:
        raise ValueError(f"exact solver limited to {limit} activated experts, "
                         f"instance has {n_act}")
    ct, gt = cpu_t[order], gpu_t[order]
    needs = (~np.asarray(resident, bool)[order]).astype(np.int64)
    rem = np.concatenate([np.cumsum(np.minimum(ct, gt)[::-1])[::-1], [0.0]])
    gC, gG, _ = greedy(workloads, resident, cpu_t, gpu_t, capacity)
    best = [makespan(cpu_t, gpu_t, gC, gG)[2], int(gG.sum()),
            tuple(np.flatnonzero(gG).tolist())]
    best_choice = [None]
    nodes = [0]
    choice = np.zeros(n_act, np.int8)

    def dfs(depth, tc, tg, used, ng):
        nodes[0] += 1
        lb = max(tc, tg, (tc + tg + rem[depth]) / 2.0)
        if lb > best[0]:
            return
        if lb == best[0] and ng > best[1]:
            return
        if depth == n_act:
            gidx = tuple(sorted(int(order[i]) for i in range(n_act) if choice[i]))
            key = [max(tc, tg), len(gidx), gidx]
            if key < best:
                best[:] = key
                best_choice[0] = choice.copy()
            return
        ok = capacity is None or used + needs[depth] <= capacity
        first_gpu = tg + gt[depth] <= tc + ct[depth]
        for dev in ((1, 0) if first_gpu else (0, 1)):
            if dev == 1:
                if not ok:
                    continue
                choice[depth] = 1
                dfs(depth + 1, tc, tg + gt[depth], used + needs[depth], ng + 1)
            else:
                choice[depth] = 0
                dfs(depth + 1, tc + ct[depth], tg, used, ng)
        choice[depth] = 0

    dfs(0, 0.0, 0.0, 0, 0)
    if best_choice[0] is None:
        return gC, gG, nodes[0]
    n = len(workloads)
    C = np.zeros(n, np.int8)
    G = np.zeros(n, np.int8)
    for i, dv in enumerate(best_choice[0]):
        (G if dv else C)[order[i]] = 1
    return C, G, nodes[0]


def static_threshold(workloads, resident, capacity, threshold=None):
    """GPU iff w >= threshold (default: median positive workload), capacity
    overflow to the CPU in descending-workload order (assignment.py:349-377)."""
    w = np.asarray(workloads)
    n = len(w)
    C = np.zeros(n, np.int8)
    G = np.zeros(n, np.int8)
    act = np.flatnonzero(w > 0)
    if len(act) == 0:
        return C, G
    if threshold is None:
        threshold = float(np.median(w[act]))
    slots = capacity
    for e in act[np.argsort(-w[act], kind="stable")]:
        if w[e] >= threshold and (slots is None or slots > 0 or bool(resident[e])):
            G[e] = 1
            if slots is not None and not resident[e]:
                slots -= 1
        else:
            C[e] = 1
    return C, G


# ---------------------------------------------------------------------------
# Residual prefetch (reference prefetch.py:88-168)
# ---------------------------------------------------------------------------


def calibrate(hidden_steps) -> np.ndarray:
    """Mean inter-layer gate-input shift (prefetch.py:88-104).

    ``hidden_steps`` is an iterable of (L, T_s, d) arrays; returns (L-1, d).
    """
    acc = None
    count = 0
    for h in hidden_steps:
        h = np.asarray(h, dtype=np.float64)
        delta = h[1:].sum(axis=1) - h[:-1].sum(axis=1)
        acc = delta if acc is None else acc + delta
        count += h.shape[1]
    return acc / count


def predict_next(hidden_l, residual_l, gate_next, k: int, prefetch_size: int):
    """Residual predictor: shift, gate with layer l+1, rank (prefetch.py:107-156).

    Returns (predicted workloads int64[N], prefetch_set int64[P]).
    """
    shifted = np.atleast_2d(np.asarray(hidden_l, dtype=np.float64))
    if residual_l is not None:
        shifted = shifted + np.asarray(residual_l, dtype=np.float64)
    predicted = derive_workloads(shifted, gate_next, k)
    pset = stable_topk(predicted.astype(np.float64), min(prefetch_size, len(predicted)))
    return predicted, pset


def frequency_table(step_workloads) -> np.ndarray:
    """Per-layer summed workloads over calibration steps, (L, N) int64
    (activation_frequency_table, prefetch.py:76-85)."""
    table = None
    for w in step_workloads:
        w = np.asarray(w, dtype=np.int64)
        table = w.copy() if table is None else table + w
    return table


def accuracy(pset, true_workloads, k: int) -> float:
    """|set[:k] & topk(true, k)| / k (prefetch.py:159-168)."""
    truth = stable_topk(np.asarray(true_workloads, dtype=np.float64), k)
    return len(set(np.asarray(pset)[:k].tolist()) & set(truth.tolist())) / k


# ---------------------------------------------------------------------------
# Workload-aware cache (reference cache.py:39-214)
# ---------------------------------------------------------------------------


@dataclass
class LayerCache:
    """One layer's cache bookkeeping (cache.py:39-64)."""

    on_gpu: np.ndarray
    w_size: int
    u_size: int
    scores: np.ndarray = None
    window: int = 0
    stopped: bool = False
    policy: str = "workload"          # "workload" | "lru" | "score"
    lru_clock: np.ndarray = None
    clock: int = 0

    def __post_init__(self):
        if self.scores is None:
            self.scores = np.zeros(len(self.on_gpu), np.float64)
        if self.lru_clock is None:
            self.lru_clock = np.zeros(len(self.on_gpu), np.int64)


def lookup(c: LayerCache, e: int) -> tuple[bool, int | None]:
    """Hit iff cached; LRU refreshes on a hit and inserts on a miss, evicting
    the least recently used (first minimum in index order) (cache.py:104-125).
    Returns (hit, LRU victim or None)."""
    hit = bool(c.on_gpu[e])
    victim = None
    if c.policy == "lru":
        c.clock += 1
        if hit:
            c.lru_clock[e] = c.clock
        else:
            cached = np.flatnonzero(c.on_gpu)
            victim = int(cached[np.argmin(c.lru_clock[cached])])
            c.on_gpu[victim] = False
            c.on_gpu[e] = True
            c.lru_clock[e] = c.clock
    return hit, victim


def force_insert(c: LayerCache, e: int) -> int | None:
    """Insert outside the window (demand / prefetch toggles, cache.py:128-143):
    evict the lowest-score cached expert (LRU: least recently used)."""
    if c.on_gpu[e]:
        return None
    cached = np.flatnonzero(c.on_gpu)
    if c.policy == "lru":
        victim = int(cached[np.argmin(c.lru_clock[cached])])
    else:
        victim = int(cached[np.argsort(c.scores[cached], kind="stable")[0]])
    c.on_gpu[victim] = False
    c.on_gpu[e] = True
    return victim


def initial_residents(layer: int, num_experts: int, capacity: int, seed: int):
    """Seeded initial resident set (cache.py:85-88)."""
    rng = np.random.default_rng([seed, layer])
    mask = np.zeros(num_experts, dtype=bool)
    mask[rng.permutation(num_experts)[:capacity]] = True
    return mask


def new_cache(layer, num_experts, capacity, w_size, u_size, seed=0,
              policy: str = "workload") -> LayerCache:
    return LayerCache(initial_residents(layer, num_experts, capacity, seed),
                      int(w_size), int(u_size), policy=policy)


def window_update(c: LayerCache, workload, is_eos: bool, gate_score_sums=None):
    """Workload (score) policy: accumulate workloads (summed gate scores),
    and at the window boundary swap up to u pairs while the incoming score
    >= outgoing; LRU only honours EOS (cache.py:146-214).

    Returns None (no window boundary) or (evicted list, admitted list).
    """
    if c.stopped:
        return None
    if c.policy in ("workload", "score"):
        vec = (np.asarray(workload, dtype=np.float64) if c.policy == "workload"
               else np.asarray(gate_score_sums, dtype=np.float64))
        c.scores = c.scores + vec
        c.window += 1
    if is_eos:
        c.stopped = True
        return None
    if c.policy == "lru" or c.window < c.w_size:
        return None
    off = np.flatnonzero(~c.on_gpu)
    on = np.flatnonzero(c.on_gpu)
    cand = off[np.argsort(-c.scores[off], kind="stable")][:c.u_size]
    vict = on[np.argsort(c.scores[on], kind="stable")][:c.u_size]
    m = 0
    while m < min(len(cand), len(vict)) and c.scores[cand[m]] >= c.scores[vict[m]]:
        m += 1
    evicted = [int(x) for x in vict[:m]]
    admitted = [int(x) for x in cand[:m]]
    c.on_gpu[evicted] = False
    c.on_gpu[admitted] = True
    c.scores = np.zeros_like(c.scores)
    c.window = 0
    return evicted, admitted


def default_u_size(num_experts: int, capacity: int) -> int:
    """simulator.py:38-42."""
    u = 8 if num_experts >= 32 else 1
    return max(0, min(u, capacity, num_experts - capacity))


def hit_rates(records, group_size: int = 8):
    """Overall / per-layer / per-token-group hit rates (cache.py:234-266).

    ``records`` is a list of (layer, token_index, hit).
    """
    if not records:
        return None, {}, {}, []
    hits = sum(1 for r in records if r[2])
    overall = hits / len(records)
    per_layer: dict = {}
    per_group: dict = {}
    for layer, tok, hit in records:
        a = per_layer.setdefault(layer, [0, 0])
        a[0] += int(hit)
        a[1] += 1
        g = per_group.setdefault(tok // group_size, [0, 0])
        g[0] += int(hit)
        g[1] += 1
    pl = {k: v[0] / v[1] for k, v in sorted(per_layer.items())}
    pg = {k: v[0] / v[1] for k, v in sorted(per_group.items())}
    top = max(per_group) if per_group else 0
    empty = [g for g in range(top + 1) if g not in per_group]
    return overall, pl, pg, empty


# ---------------------------------------------------------------------------
# Synthetic trace generator (reference trace.py:274-375) -- input fixture
# ---------------------------------------------------------------------------


@dataclass
class SynthStep:
    token_index: int
    tokens: int
    workloads: np.ndarray
    hidden: np.ndarray
    eos: bool


@dataclass
class SynthTrace:
    L: int
    N: int
    k: int
    d: int
    gates: np.ndarray            # (L, d, N) fp64
    drifts: np.ndarray           # (L-1, d)
    steps: list = field(default_factory=list)


def synth_trace(L, N, k, d, batch_size, num_steps, locality=0.9,
                drift_scale=0.0, noise_scale=0.0, seed=0, phase="decode"):
    """Same RNG draw order as ``generate_synthetic_trace`` so a seed yields the
    reference's arrays bit-for-bit (pinned by the golden tests)."""
    rng = np.random.default_rng(seed)
    norm = math.sqrt(d)

    def renorm(rows):
        n = np.linalg.norm(rows, axis=1, keepdims=True)
        n[n == 0.0] = 1.0
        return rows * (norm / n)

    base = rng.normal(size=(L, d, N)) * (0.4 / np.sqrt(d))
    scale = rng.permuted(np.tile(np.linspace(0.15, 1.85, N), (L, 1)), axis=1)
    gates = base * scale[:, None, :]
    if L > 1:
        dirs = rng.normal(size=(L - 1, d))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        drifts = drift_scale * norm * dirs
    else:
        drifts = np.zeros((0, d))
    state = renorm(rng.normal(size=(batch_size, d)))

    def stack_of(rows):
        out = np.empty((L,) + rows.shape)
        out[0] = rows
        for l in range(1, L):
            out[l] = out[l - 1] + drifts[l - 1] + rng.normal(size=rows.shape) * noise_scale
        return out

    def loads(stack):
        return np.stack([derive_workloads(stack[l], gates[l], k) for l in range(L)])

    def advance(s):
        fresh = rng.normal(size=s.shape)
        return renorm(locality * s + (1.0 - locality) * fresh)

    tr = SynthTrace(L, N, k, d, gates, drifts)
    if phase == "prefill":
        rows = np.empty((batch_size * num_steps, d))
        for t in range(num_steps):
            rows[t * batch_size:(t + 1) * batch_size] = state
            if t < num_steps - 1:
                state = advance(state)
        st = stack_of(rows)
        tr.steps.append(SynthStep(0, rows.shape[0], loads(st), st, True))
    else:
        for t in range(num_steps):
            st = stack_of(state)
            tr.steps.append(SynthStep(t, batch_size, loads(st), st, t == num_steps - 1))
            if t < num_steps - 1:
                state = advance(state)
    return tr
