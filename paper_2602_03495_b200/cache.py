"""Workload-aware expert cache (drop-in for reference cache.py, workload policy).

``CacheState`` keeps the reference's host-visible fields (``on_gpu``,
``scores``, ``tokens_in_window``, ``stopped``) so callers can inspect and
seed it; ``record_and_maybe_replace`` runs the window update on device
(``dali_cache_record``: score accumulation, stable candidate/victim ranking,
dominance-guarded swaps) and writes the state back.  The engine keeps the
same state resident in HBM and updates it inside the fused policy kernel.
The LRU and score policies and the insert toggles (the reference's
comparison baselines) use the same device state: ``lookup`` /
``force_insert`` run ``dali_cache_op``, the score policy feeds the summed
gate scores through the window kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .errors import CacheError

CACHE_POLICIES = ("workload", "lru", "score")


@dataclass
class ReplacementEvent:
    token_index: int
    evicted: list[int]
    admitted: list[int]
    transfer_cost_ms: float = 0.0


@dataclass
class CacheState:
    layer: int
    num_experts: int
    capacity: int
    window_size: int
    update_size: int
    policy: str
    on_gpu: np.ndarray = field(default=None)
    scores: np.ndarray = field(default=None)
    tokens_in_window: int = 0
    stopped: bool = False
    lru_clock: np.ndarray = field(default=None)
    clock: int = 0
    insert_demand_fetched: bool = False
    insert_prefetched: bool = False

    @property
    def expert_on_gpu(self) -> np.ndarray:
        return np.flatnonzero(self.on_gpu)

    @property
    def expert_on_cpu(self) -> np.ndarray:
        return np.flatnonzero(~self.on_gpu)


def initial_resident_set(layer: int, num_experts: int, capacity: int, seed: int) -> np.ndarray:
    """Seeded initial residents: default_rng([seed, layer]).permutation(N)[:cap]
    (cache.py:85-88).  Host-side, once at init (not on the hot path)."""
    rng = np.random.default_rng([seed, layer])
    mask = np.zeros(num_experts, dtype=bool)
    mask[rng.permutation(num_experts)[:capacity]] = True
    return mask


def init_cache(layer: int, num_experts: int, capacity: int, w_size: int, u_size: int,
               policy: str = "workload", seed: int = 0, insert_demand_fetched: bool = False,
               insert_prefetched: bool = False) -> CacheState:
    if policy not in CACHE_POLICIES:
        raise CacheError(f"unknown cache policy {policy!r}; choose from {CACHE_POLICIES}")
    if not (0 < capacity < num_experts):
        raise CacheError(f"capacity must satisfy 0 < capacity < num_experts, got "
                         f"capacity={capacity}, num_experts={num_experts}")
    if w_size < 1:
        raise CacheError(f"w_size must be >= 1, got {w_size}")
    if not (0 <= u_size <= min(capacity, num_experts - capacity)):
        raise CacheError(f"u_size must be in [0, min(capacity, N - capacity)] = "
                         f"[0, {min(capacity, num_experts - capacity)}], got {u_size}")
    return CacheState(layer=layer, num_experts=num_experts, capacity=capacity,
                      window_size=w_size, update_size=u_size, policy=policy,
                      on_gpu=initial_resident_set(layer, num_experts, capacity, seed),
                      scores=np.zeros(num_experts, dtype=np.float64),
                      lru_clock=np.zeros(num_experts, dtype=np.int64),
                      insert_demand_fetched=insert_demand_fetched,
                      insert_prefetched=insert_prefetched)


def _cache_op(state: CacheState, expert: int, op: int) -> tuple[int, int]:
    N = state.num_experts
    on = _dev.to_dev(state.on_gpu.astype(np.uint8), torch.uint8)
    sc = _dev.to_dev(state.scores, torch.float64)
    lru = _dev.to_dev(np.concatenate([state.lru_clock, [state.clock]]).astype(np.int64),
                      torch.int64)
    out = _dev.zeros((2,), torch.int32)
    _lib.call("dali_cache_op", on.data_ptr(), sc.data_ptr(), lru.data_ptr(), N,
              int(state.policy == "lru"), int(expert), op, out.data_ptr(), _dev.stream_ptr())
    state.on_gpu = on.cpu().numpy().astype(bool)
    lv = lru.cpu().numpy()
    state.lru_clock, state.clock = lv[:N].copy(), int(lv[N])
    o = out.cpu().numpy()
    return int(o[0]), int(o[1])


def lookup(state: CacheState, expert: int) -> bool:
    """Hit iff cached (cache.py:104-117); under LRU the call also ticks the
    clock, refreshes a hit and inserts a miss over the least recently used."""
    if not (0 <= expert < state.num_experts):
        raise CacheError(f"expert {expert} out of range [0, {state.num_experts})")
    if state.policy != "lru":
        return bool(state.on_gpu[expert])
    hit, _ = _cache_op(state, expert, 0)
    return bool(hit)


def force_insert(state: CacheState, expert: int) -> int | None:
    """Insert outside the windowed mechanism (demand / prefetch toggles,
    cache.py:128-143): evicts the lowest-score (LRU: least recently used)
    cached expert and returns it, or None if already cached."""
    if not (0 <= expert < state.num_experts):
        raise CacheError(f"expert {expert} out of range [0, {state.num_experts})")
    if state.on_gpu[expert]:
        return None
    _, victim = _cache_op(state, expert, 1)
    return victim


def record_and_maybe_replace(state: CacheState, workload, token_index: int,
                             is_eos: bool = False, gate_scores=None,
                             trans_time_ms: float = 0.0) -> ReplacementEvent | None:
    if state.stopped:
        return None
    workload = np.asarray(workload)
    if workload.shape != (state.num_experts,):
        raise CacheError(f"workload vector length {workload.shape} != ({state.num_experts},)")
    N = state.num_experts
    if state.policy == "score":
        if gate_scores is None:
            raise CacheError("score policy requires per-expert gate scores")
        gate_scores = np.asarray(gate_scores, dtype=np.float64)
        if gate_scores.shape != (N,):
            raise CacheError(f"gate score vector length {gate_scores.shape} != ({N},)")
    if state.policy == "lru":          # no windowing; EOS still stops it
        if is_eos:
            state.stopped = True
        return None
    vec = workload if state.policy == "workload" else gate_scores
    on = _dev.to_dev(state.on_gpu.astype(np.uint8), torch.uint8)
    sc = _dev.to_dev(state.scores, torch.float64)
    ctr = _dev.to_dev(np.array([state.tokens_in_window, int(state.stopped)], np.int32),
                      torch.int32)
    wl = _dev.to_dev(np.asarray(vec, dtype=np.float64), torch.float64)
    ev = _dev.zeros((2 + 2 * _lib.MAX_EXPERTS,), torch.int32)
    _lib.call("dali_cache_record", on.data_ptr(), sc.data_ptr(), ctr.data_ptr(), N,
              state.window_size, state.update_size, wl.data_ptr(), int(bool(is_eos)),
              ev.data_ptr(), _dev.stream_ptr())
    state.on_gpu = on.cpu().numpy().astype(bool)
    state.scores = sc.cpu().numpy()
    c = ctr.cpu().numpy()
    state.tokens_in_window, state.stopped = int(c[0]), bool(c[1])
    e = ev.cpu().numpy()
    if not e[0]:
        return None
    m = int(e[1])
    evicted = [int(x) for x in e[2:2 + m]]
    admitted = [int(x) for x in e[2 + _lib.MAX_EXPERTS:2 + _lib.MAX_EXPERTS + m]]
    return ReplacementEvent(token_index=token_index, evicted=evicted, admitted=admitted,
                            transfer_cost_ms=len(admitted) * trans_time_ms)


@dataclass
class CacheStats:
    """Hit/miss accounting (cache.py:217-266)."""

    records: list = field(default_factory=list)

    def record(self, layer: int, token_index: int, hit: bool) -> None:
        self.records.append((layer, token_index, hit))

    @property
    def hits(self) -> int:
        return sum(1 for r in self.records if r[2])

    @property
    def misses(self) -> int:
        return sum(1 for r in self.records if not r[2])

    def hit_rate(self, grouping: str = "overall", group_size: int = 8):
        if not self.records:
            raise CacheError("no lookups recorded")
        if grouping == "overall":
            return self.hits / len(self.records)
        if grouping == "per-layer":
            acc: dict = {}
            for layer, _, h in self.records:
                a = acc.setdefault(layer, [0, 0])
                a[0] += int(h)
                a[1] += 1
            return {k: v[0] / v[1] for k, v in sorted(acc.items())}
        if grouping == "per-token-group":
            if group_size < 1:
                raise CacheError("group_size must be >= 1")
            acc = {}
            for _, tok, h in self.records:
                a = acc.setdefault(tok // group_size, [0, 0])
                a[0] += int(h)
                a[1] += 1
            rates = {k: v[0] / v[1] for k, v in sorted(acc.items())}
            top = max(acc) if acc else 0
            return rates, [g for g in range(top + 1) if g not in acc]
        raise CacheError(f"unknown grouping {grouping!r}")
