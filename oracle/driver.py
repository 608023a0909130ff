"""Decision-recording restatement of ``simulate_run`` (TEST INFRASTRUCTURE).

Follows reference ``simulator.py:318-522`` (and ``simulate_layer``
``:151-197``) for the hot-path policy set: greedy (or all-cpu) assignment,
residual prefetch, workload-aware cache.  Besides the aggregate report it
returns one record per (step, layer) holding every decision, so the GPU
engine's device-side decision log can be compared entry by entry.

Floating-point evaluation order follows the reference expression by
expression (sequential lane sums, ``cpu_times @ C`` through numpy, Python
float floor division for the prefetch window) so the oracle reproduces the
reference report bit-for-bit; ``tests/test_oracle_golden.py`` asserts that
against the frozen ``moesim.simulate_run`` outputs.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import policy as P


@dataclass
class DriverConfig:
    """Subset of the reference ``SimConfig`` (simulator.py:45-74) on the path."""

    tables: P.CostTables
    assignment_policy: str = "greedy"          # greedy | all-cpu | all-gpu | beam |
    #                                            optimal | static-threshold
    gpu_capacity: int | None = None
    beam_width: int = 2
    threshold: float | None = None
    exact_solver_limit: int = 24
    prefetch_size: int = 0                     # 0 = prefetch off
    prefetch_kind: str = "residual"            # residual | feature | statistical | random
    residuals: np.ndarray | None = None        # (L-1, d)
    frequency_table: np.ndarray | None = None  # (L, N) statistical predictor
    cache_capacity: int = 0                    # 0 = cache off
    cache_policy: str = "workload"             # workload | lru | score
    w_size: int = 4
    u_size: int | None = None
    insert_demand_fetched: bool = False
    insert_prefetched: bool = False
    scheduling_overhead_ms: float = 0.0
    solver_node_cost_ms: float = 0.0
    prefetch_compute_ms: float = 0.0
    non_moe_override: float | None = None
    seed: int = 0
    num_shared_experts: int = 0
    initial_on_gpu: np.ndarray | None = None   # (L, N) carry-over residency
    all_resident: bool = False                 # every expert in HBM


@dataclass
class StepInput:
    token_index: int
    tokens: int
    workloads: np.ndarray        # (L, N) int64
    hidden: np.ndarray | None    # (L, T, d) gate inputs, needed for prefetch
    eos: bool
    # (L-1, N) next-layer predicted workloads supplied by the caller instead of
    # the residual predictor over ``hidden`` -- the expert-parallel shard
    # semantics: the owner's slice of the prediction summed over every rank's
    # tokens (repo engine/ep.py), not a reference feature
    predicted: np.ndarray | None = None


@dataclass
class LayerRecord:
    step: int
    layer: int
    workloads: np.ndarray
    resident: np.ndarray
    C: np.ndarray
    G: np.ndarray
    lookups: list                 # [(expert, hit)]
    inserts: list = field(default_factory=list)   # [(layer, victim, expert, kind)]
    predicted: np.ndarray | None = None
    prefetch_set: np.ndarray | None = None
    candidates: list = field(default_factory=list)
    completed: list = field(default_factory=list)
    event: tuple | None = None    # (evicted, admitted) at a window boundary
    cpu_busy: float = 0.0
    gpu_makespan: float = 0.0
    latency: float = 0.0
    demand_end: float = 0.0


def layer_schedule(w, resident, C, G, order, tables, cpu_t):
    """Timeline of ``simulate_layer`` (simulator.py:169-193) without overheads.

    Returns (cpu_busy, gpu_makespan, demand intervals list).
    """
    cpu_busy = float(cpu_t @ C)
    pcie_t = 0.0
    engine_t = 0.0
    demand = []
    for e in order:
        if not G[e]:
            continue
        comp = tables.t_gpu_compute(int(w[e]))
        if resident[e]:
            start = engine_t
        else:
            end = pcie_t + tables.trans_time
            demand.append((pcie_t, end))
            pcie_t = end
            start = max(engine_t, end)
        engine_t = start + comp
    return cpu_busy, engine_t, demand


def run(steps, gates, cfg: DriverConfig, L: int, N: int, k: int):
    """Drive ``steps`` through the policies; returns (report dict, records)."""
    tb = cfg.tables
    shared_ms = tb.shared_expert_gpu_time if cfg.num_shared_experts > 0 else 0.0
    non_moe = cfg.non_moe_override if cfg.non_moe_override is not None \
        else tb.non_moe_layer_time
    prefetch_on = cfg.prefetch_size > 0
    rng = np.random.default_rng(cfg.seed) if cfg.prefetch_kind == "random" else None
    caches = None
    if cfg.cache_capacity > 0:
        u = cfg.u_size if cfg.u_size is not None \
            else P.default_u_size(N, cfg.cache_capacity)
        caches = [P.new_cache(l, N, cfg.cache_capacity, cfg.w_size, u, cfg.seed,
                              policy=cfg.cache_policy)
                  for l in range(L)]
        if cfg.initial_on_gpu is not None:
            for l in range(L):
                caches[l].on_gpu = np.asarray(cfg.initial_on_gpu[l], dtype=bool).copy()

    pcie_demand = np.zeros(L)
    pcie_prefetch = np.zeros(L)
    pcie_replace = np.zeros(L)
    layer_time = np.zeros(L)
    cpu_busy_tot = 0.0
    gpu_busy_tot = 0.0
    acc1: dict = {}
    acck: dict = {}
    replacements = []
    lookups_all = []
    token_lat = []
    records = []
    tokens = 0
    n_steps = 0

    for si, st in enumerate(steps):
        token_ms = 0.0
        arrivals: dict = {}
        for l in range(L):
            w = np.asarray(st.workloads[l], dtype=np.int64)
            resident = np.zeros(N, bool)
            if caches is not None:
                resident |= caches[l].on_gpu
            got = arrivals.get(l)
            if got is not None and len(got):
                resident[got] = True
            if cfg.all_resident:
                resident[:] = True
            extra = cfg.prefetch_compute_ms if prefetch_on and l < L - 1 else 0.0

            cpu_t, gpu_t = P.expert_times(tb, w, resident)
            if cfg.assignment_policy == "greedy":
                C, G, order = P.greedy(w, resident, cpu_t, gpu_t, cfg.gpu_capacity)
                nodes = int((w > 0).sum())
            elif cfg.assignment_policy == "all-gpu":
                C, G = P.all_gpu(w, resident, cfg.gpu_capacity)
                order = P.visit_order(w, cpu_t, gpu_t)
                nodes = 0
            elif cfg.assignment_policy == "all-cpu":
                C, G = P.all_cpu(w)
                order = P.visit_order(w, cpu_t, gpu_t)
                nodes = 0
            elif cfg.assignment_policy == "beam":
                C, G = P.beam(w, resident, cpu_t, gpu_t, cfg.gpu_capacity, cfg.beam_width)
                order = P.visit_order(w, cpu_t, gpu_t)
                nodes = int((w > 0).sum()) * cfg.beam_width
            elif cfg.assignment_policy == "optimal":
                C, G, nodes = P.optimal(w, resident, cpu_t, gpu_t, cfg.gpu_capacity,
                                        cfg.exact_solver_limit)
                order = P.visit_order(w, cpu_t, gpu_t)
            elif cfg.assignment_policy == "static-threshold":
                C, G = P.static_threshold(w, resident, cfg.gpu_capacity, cfg.threshold)
                order = P.visit_order(w, cpu_t, gpu_t)
                nodes = 0
            else:
                raise ValueError(cfg.assignment_policy)
            cpu_busy, gpu_mk, demand = layer_schedule(w, resident, C, G, order, tb, cpu_t)
            latency = (max(cpu_busy, gpu_mk) + shared_ms + cfg.scheduling_overhead_ms
                       + cfg.solver_node_cost_ms * nodes + extra)
            rec = LayerRecord(si, l, w.copy(), resident.copy(), C, G, [],
                              cpu_busy=cpu_busy, gpu_makespan=gpu_mk,
                              latency=latency)

            if caches is not None:
                for e in np.flatnonzero(G):
                    hit, victim = P.lookup(caches[l], int(e))
                    rec.lookups.append((int(e), hit))
                    lookups_all.append((l, st.token_index, hit))
                    if victim is not None:
                        rec.inserts.append((l, victim, int(e), "lru"))
                    if (not hit and cfg.insert_demand_fetched and cfg.cache_policy != "lru"
                            and not resident[e]):
                        v = P.force_insert(caches[l], int(e))
                        if v is not None:
                            rec.inserts.append((l, v, int(e), "demand"))

            demand_end = demand[-1][1] if demand else 0.0
            rec.demand_end = demand_end
            if prefetch_on and l < L - 1:
                if st.predicted is not None:
                    predicted = np.asarray(st.predicted[l], np.int64).copy()
                    pset = P.stable_topk(predicted.astype(np.float64),
                                         min(cfg.prefetch_size, N))
                elif cfg.prefetch_kind in ("residual", "feature"):
                    res = (cfg.residuals[l] if cfg.residuals is not None
                           and cfg.prefetch_kind == "residual" else None)
                    predicted, pset = P.predict_next(st.hidden[l], res, gates[l + 1],
                                                     k, cfg.prefetch_size)
                else:
                    predicted = (np.asarray(cfg.frequency_table[l + 1], np.int64).copy()
                                 if cfg.prefetch_kind == "statistical"
                                 else rng.permutation(N).astype(np.int64))
                    pset = P.stable_topk(predicted.astype(np.float64),
                                         min(cfg.prefetch_size, N))
                rec.predicted, rec.prefetch_set = predicted, pset
                true_next = st.workloads[l + 1]
                acc1.setdefault(l + 1, []).append(P.accuracy(pset, true_next, 1))
                acck.setdefault(l + 1, []).append(
                    P.accuracy(pset, true_next, min(cfg.prefetch_size, N)))
                nxt = caches[l + 1].on_gpu if caches is not None else np.zeros(N, bool)
                cands = [int(e) for e in pset if not nxt[e]]
                idle = max(0.0, latency + non_moe - demand_end)
                if tb.trans_time > 0:
                    n_fit = int(idle // tb.trans_time)
                    done = cands[:n_fit]
                    consumed = min(len(cands) * tb.trans_time, idle)
                else:
                    done = cands
                    consumed = 0.0
                pcie_prefetch[l] += consumed
                arrivals[l + 1] = np.asarray(done, dtype=np.int64)
                rec.candidates, rec.completed = cands, list(done)
                if caches is not None and cfg.insert_prefetched:
                    for e in done:
                        v = P.force_insert(caches[l + 1], int(e))
                        if v is not None:
                            rec.inserts.append((l + 1, v, int(e), "prefetch"))

            boundary = 0.0
            if caches is not None:
                gss = None
                if cfg.cache_policy == "score":
                    gss = P.gate_probs(st.hidden[l], gates[l]).sum(axis=0)
                ev = P.window_update(caches[l], w, st.eos, gss)
                if ev is not None:
                    evicted, admitted = ev
                    boundary = len(admitted) * tb.trans_time
                    pcie_replace[l] += boundary
                    rec.event = (evicted, admitted)
                    if admitted:
                        replacements.append({
                            "token_index": st.token_index, "layer": l,
                            "evicted": evicted, "admitted": admitted,
                            "transfer_cost_ms": boundary})

            pcie_demand[l] += sum(e - s for s, e in demand)
            layer_time[l] += latency + boundary + non_moe
            cpu_busy_tot += cpu_busy
            gpu_busy_tot += gpu_mk + shared_ms
            token_ms += latency + boundary
            records.append(rec)

        token_ms += L * non_moe
        token_lat.append(token_ms)
        tokens += st.tokens
        n_steps += 1
        if st.eos:
            break

    total = float(sum(token_lat))
    busy = float(pcie_demand.sum() + pcie_prefetch.sum() + pcie_replace.sum())
    per_layer = {}
    for l in range(L):
        lt = layer_time[l]
        per_layer[str(l)] = float((pcie_demand[l] + pcie_prefetch[l]
                                   + pcie_replace[l]) / lt) if lt > 0 else 0.0
    overall, hl, hg, empty = (P.hit_rates(lookups_all) if caches is not None
                              else (None, {}, {}, []))
    report = {
        "tokens": tokens,
        "steps": n_steps,
        "total_time_ms": total,
        "tokens_per_second": tokens / (total / 1000.0) if total > 0 else 0.0,
        "mean_token_latency_ms": total / n_steps if n_steps else 0.0,
        "cpu_busy_ms": float(cpu_busy_tot),
        "gpu_busy_ms": float(gpu_busy_tot),
        "pcie_demand_ms": float(pcie_demand.sum()),
        "pcie_prefetch_ms": float(pcie_prefetch.sum()),
        "pcie_replacement_ms": float(pcie_replace.sum()),
        "pcie_busy_ms": busy,
        "pcie_busy_fraction": busy / total if total > 0 else 0.0,
        "per_layer_pcie_fraction": per_layer,
        "prefetch_accuracy_top1": {str(a): float(np.mean(b)) for a, b in sorted(acc1.items())},
        "prefetch_accuracy_topk": {str(a): float(np.mean(b)) for a, b in sorted(acck.items())},
        "prefetch_size": cfg.prefetch_size,
        "cache_hit_rate": overall,
        "cache_hit_rate_per_layer": {str(a): b for a, b in hl.items()},
        "cache_hit_rate_per_group": {str(a): b for a, b in hg.items()},
        "cache_empty_groups": empty,
        "replacement_events": replacements,
    }
    return report, records
