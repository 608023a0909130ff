"""Device-resident DALI policy state + the per-layer decision step.

One ``PolicyEngine`` holds, in HBM, everything the reference driver keeps
per layer (simulator.py:331-338,354-364): cache residency / window scores /
window counters (``init_cache``), the arrived-prefetch flags of the current
step and the physical slot table.  ``layer_step`` launches, on the caller's
stream:

  1. (prefetch on, layer < L-1) the routing kernel on ``hidden + res[l]``
     with gate ``l+1`` -> predicted workloads of layer l+1;
  2. the fused single-CTA policy kernel -> decision record.

Decision records go to pinned host memory that the kernel writes directly
(UVA), so the host reads them after an event wait without a copy.  The
report assembly (``build_report``) follows the reference's float
accumulation order expression by expression (simulator.py:446-522).
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _dev, _lib
from .cache import initial_resident_set
from .cost_model import CostModel
from .errors import AssignmentError, CacheError, SimulationError
from .trace import route_device, topk_indices


ASSIGNMENT_CODES = {"greedy": 0, "all-cpu": 1, "all-gpu": 2, "beam": 3, "optimal": 4,
                    "static-threshold": 5}
CACHE_CODES = {"workload": 0, "lru": 1, "score": 2}


def default_u_size(num_experts: int, capacity: int) -> int:
    """8 for wide expert pools, 1 for narrow ones, clamped (simulator.py:38-42)."""
    u = 8 if num_experts >= 32 else 1
    return max(0, min(u, capacity, num_experts - capacity))


class PolicyEngine:
    def __init__(self, L: int, N: int, k: int, cost_model: CostModel, *,
                 assignment: str = "greedy", gpu_capacity: int | None = None,
                 prefetch_size: int = 0, residuals: torch.Tensor | None = None,
                 cache_capacity: int = 0, w_size: int = 4, u_size: int | None = None,
                 seed: int = 0, num_shared_experts: int = 0,
                 scheduling_overhead_ms: float = 0.0, solver_node_cost_ms: float = 0.0,
                 prefetch_compute_ms: float = 0.0, non_moe_override: float | None = None,
                 max_records: int = 4096, all_resident: bool = False,
                 initial_on_gpu: np.ndarray | None = None, beam_width: int = 2,
                 threshold: float | None = None, exact_solver_limit: int = 24,
                 cache_policy: str = "workload", insert_demand_fetched: bool = False,
                 insert_prefetched: bool = False, prefetch_kind: str = "residual",
                 frequency_table: np.ndarray | None = None):
        if N > _lib.MAX_EXPERTS:
            raise SimulationError(f"at most {_lib.MAX_EXPERTS} experts per layer")
        if assignment not in ASSIGNMENT_CODES:
            raise SimulationError(f"unknown assignment policy {assignment!r}; choose from "
                                  f"{tuple(ASSIGNMENT_CODES)}")
        if cache_policy not in CACHE_CODES:
            raise SimulationError(f"unknown cache policy {cache_policy!r}")
        if prefetch_kind not in ("residual", "feature", "statistical", "random"):
            raise SimulationError(f"unknown prefetch kind {prefetch_kind!r}")
        if assignment == "beam" and not (1 <= beam_width <= _lib.MAX_BEAM):
            raise SimulationError(f"beam_width must be in [1, {_lib.MAX_BEAM}] on the device "
                                  f"solver, got {beam_width}")
        if prefetch_kind == "statistical" and prefetch_size > 0 and frequency_table is None:
            raise SimulationError("statistical prefetching requires a calibration frequency "
                                  "table")
        dev = _dev.require_cuda()
        self.L, self.N, self.k = L, N, k
        self.cm = cost_model
        self.cm_c = cost_model.to_c()
        self.prefetch_size = int(prefetch_size)
        self.cache_enabled = cache_capacity > 0
        if self.cache_enabled and not (0 < cache_capacity < N):
            raise SimulationError(f"cache capacity must be in (0, {N}), got {cache_capacity}")
        self.u_size = (u_size if u_size is not None
                       else default_u_size(N, cache_capacity)) if self.cache_enabled else 0
        non_moe = (non_moe_override if non_moe_override is not None
                   else cost_model.non_moe_layer_time)
        cfg = _lib.PolicyConfigC()
        cfg.L, cfg.N, cfg.k = L, N, k
        cfg.assignment = ASSIGNMENT_CODES[assignment]
        cfg.beam_width = int(beam_width)
        cfg.exact_solver_limit = int(exact_solver_limit)
        cfg.has_threshold = int(threshold is not None)
        cfg.threshold = float(threshold) if threshold is not None else 0.0
        cfg.cache_policy = CACHE_CODES[cache_policy]
        cfg.insert_demand = int(bool(insert_demand_fetched))
        cfg.insert_prefetched = int(bool(insert_prefetched))
        self.assignment = assignment
        self.cache_policy = cache_policy
        self.prefetch_kind = prefetch_kind
        self.seed = int(seed)
        cfg.gpu_capacity = -1 if gpu_capacity is None else int(gpu_capacity)
        cfg.prefetch_size = self.prefetch_size
        cfg.cache_enabled = int(self.cache_enabled)
        cfg.w_size, cfg.u_size = int(w_size), int(self.u_size)
        cfg.has_shared = int(num_shared_experts > 0)
        cfg.all_resident = int(bool(all_resident))
        cfg.scheduling_overhead_ms = float(scheduling_overhead_ms)
        cfg.solver_node_cost_ms = float(solver_node_cost_ms)
        cfg.prefetch_compute_ms = float(prefetch_compute_ms)
        cfg.non_moe = float(non_moe)
        self.cfg = cfg
        self.non_moe = float(non_moe)
        self.shared_ms = cost_model.shared_expert_gpu_time if num_shared_experts > 0 else 0.0

        on = np.zeros((L, N), np.uint8)
        slot = np.full((L, N), -1, np.int32)
        if self.cache_enabled:
            for l in range(L):
                mask = (initial_resident_set(l, N, cache_capacity, seed) if initial_on_gpu is None
                        else np.asarray(initial_on_gpu[l], dtype=bool))
                if int(mask.sum()) != cache_capacity:
                    raise SimulationError("initial residency does not match cache capacity")
                on[l] = mask
                slot[l, np.flatnonzero(mask)] = np.arange(cache_capacity) + l * cache_capacity
        self.initial_on_gpu = on.copy()
        self.on_gpu = torch.from_numpy(on).to(dev)
        self.slot_of = torch.from_numpy(slot).to(dev)
        self.scores = torch.zeros((L, N), dtype=torch.float64, device=dev)
        self.counters = torch.zeros((L, 2), dtype=torch.int32, device=dev)
        self.arrived = torch.zeros((L, N), dtype=torch.uint8, device=dev)
        self.predicted = torch.zeros((N,), dtype=torch.int64, device=dev)
        # LRU clocks (cache.py:96-99): (L, N+1) int64, the layer's clock last
        self.lru_state = torch.zeros((L, N + 1), dtype=torch.int64, device=dev)
        self._probs = None                  # score policy: (T, N) f64 gate scores
        self.residuals = residuals
        if self.prefetch_size > 0 and residuals is None and prefetch_kind in ("residual",
                                                                               "feature"):
            raise SimulationError("residual prefetching requires calibrated residual vectors; "
                                  "run the calibrate step first")
        self.freq = (torch.from_numpy(np.ascontiguousarray(frequency_table, dtype=np.int64))
                     .to(dev) if frequency_table is not None else None)
        self.max_records = max_records
        # random predictor: numpy's PCG64 stream (prefetch.py:58-60,150-151) drawn
        # on the host, one permutation per decision, staged in pinned memory
        self._rng = None
        self._perm_host = (torch.zeros((max_records, N), dtype=torch.int64, pin_memory=True)
                           if prefetch_kind == "random" and self.prefetch_size > 0 else None)
        self._perm_dev = (torch.zeros((N,), dtype=torch.int64, device=dev)
                          if self._perm_host is not None else None)
        self.records = (_lib.LayerRecordC * max_records)()
        self._rec_buf = torch.empty((max_records * _lib.RECORD_BYTES,), dtype=torch.uint8,
                                    pin_memory=True)
        self.n_records = 0

    def new_run(self) -> np.ndarray:
        """Start a new run (one request): window scores, counters, arrivals
        and the decision log reset, cache residency and slots carry over.
        Returns the residency the run starts from (the oracle's input)."""
        torch.cuda.current_stream().synchronize()
        self.scores.zero_()
        self.counters.zero_()
        self.arrived.zero_()
        self.lru_state.zero_()
        self.n_records = 0
        if self.prefetch_kind == "random":
            self._rng = np.random.default_rng(self.seed)
        return self.on_gpu.cpu().numpy().astype(bool)

    # -- stepping --------------------------------------------------------------
    def record_ptr(self, i: int) -> int:
        return self._rec_buf.data_ptr() + i * _lib.RECORD_BYTES

    def record(self, i: int) -> _lib.LayerRecordC:
        return _lib.LayerRecordC.from_address(self.record_ptr(i))

    def layer_step(self, step: int, layer: int, token_index: int, is_eos: bool,
                   workloads: torch.Tensor, hidden: torch.Tensor | None,
                   gate_next: torch.Tensor | None, stream=None,
                   predicted: torch.Tensor | None = None,
                   gate_this: torch.Tensor | None = None,
                   gate_next_norm2: torch.Tensor | None = None) -> int:
        """Queue the decision of (step, layer) on ``stream``; returns the
        record index (valid on the host once the stream reaches it).
        ``predicted`` supplies layer+1's predicted workloads directly (the
        expert-parallel path all-reduces them across ranks first);
        ``gate_this`` (this layer's gate) feeds the score cache policy."""
        if self.n_records >= self.max_records:
            raise SimulationError("decision log full")
        sp = _dev.stream_ptr(stream)
        i = self.n_records
        pred_p = self.predicted_ptr(layer, hidden, gate_next, stream, predicted, i,
                                    gate_next_norm2=gate_next_norm2)
        probs_p, n_tok = self.gate_probs_ptr(hidden, gate_this, stream)
        _lib.call("dali_policy_layer", C.addressof(self.cfg), C.addressof(self.cm_c), step,
                  layer, token_index, int(bool(is_eos)), workloads.data_ptr(), pred_p,
                  self.on_gpu.data_ptr(), self.scores.data_ptr(), self.counters.data_ptr(),
                  self.arrived.data_ptr(), self.slot_of.data_ptr(), self.lru_state.data_ptr(),
                  probs_p, n_tok, self.record_ptr(i), sp)
        self.n_records += 1
        return i

    def predicted_ptr(self, layer: int, hidden, gate_next, stream=None, predicted=None,
                      rec_index: int = 0, gate_next_norm2=None):
        """Device pointer to layer+1's predicted workloads for the configured
        predictor (None when nothing is prefetched after this layer):
        residual / feature -> routing kernel on the (shifted) gate inputs;
        statistical -> the calibration table row; random -> the next numpy
        permutation, staged through pinned memory by a kernel copy."""
        if self.prefetch_size <= 0 or layer >= self.L - 1:
            return None
        if predicted is not None:
            return predicted.data_ptr()
        if self.prefetch_kind == "statistical":
            return self.freq[layer + 1].data_ptr()
        if self.prefetch_kind == "random":
            if self._rng is None:
                self._rng = np.random.default_rng(self.seed)
            row = self._perm_host[rec_index]
            row.copy_(torch.from_numpy(self._rng.permutation(self.N).astype(np.int64)))
            _lib.call("dali_copy_mapped", self._perm_dev.data_ptr(), row.data_ptr(), self.N * 8,
                      _dev.stream_ptr(stream))
            return self._perm_dev.data_ptr()
        if hidden is None or gate_next is None:
            raise SimulationError("prefetching requires the layer's gate inputs")
        _, _, wl = route_device(hidden, gate_next, self.k, residual=self.residuals[layer],
                                want_idx=False, want_weights=False, stream=stream,
                                out=(None, None, self.predicted), norm2=gate_next_norm2)
        return wl.data_ptr()

    def gate_probs_ptr(self, hidden, gate_this, stream=None):
        """(pointer, tokens) of this layer's fp64 gate scores for the score
        cache policy (gate_scores, trace.py:242-250), else (None, 0)."""
        if not (self.cache_enabled and self.cache_policy == "score"):
            return None, 0
        if hidden is None or gate_this is None:
            raise CacheError("score policy requires per-expert gate scores")
        T = hidden.shape[0]
        if self._probs is None or self._probs.shape[0] < T:
            self._probs = torch.empty((max(T, 1), self.N), dtype=torch.float64,
                                      device=hidden.device)
        fn = "dali_gate_probs_f64" if hidden.dtype == torch.float64 else "dali_gate_probs_bf16"
        g = gate_this.to(hidden.dtype).contiguous()
        _lib.call(fn, hidden.data_ptr(), g.data_ptr(), T, hidden.shape[1], self.N,
                  self._probs.data_ptr(), _dev.stream_ptr(stream))
        return self._probs.data_ptr(), T

    def check_errors(self) -> None:
        """Raise what the reference raises for refused instances (the exact
        solver's activated-expert limit, assignment.py:284-288)."""
        for i in range(self.n_records):
            r = self.record(i)
            if r.err:
                raise AssignmentError(
                    f"exact solver limited to {self.cfg.exact_solver_limit} activated experts, "
                    f"instance has {r.n_act}; use greedy_assign instead")

    # -- reporting -------------------------------------------------------------
    def build_report(self, step_tokens: list[int], true_workloads: dict, spec: dict) -> dict:
        """RunReport dict from the decision log.  ``true_workloads[(step,
        layer)]`` gives the realised workloads (for prefetch accuracy)."""
        L, N = self.L, self.N
        pcie_demand = np.zeros(L)
        pcie_prefetch = np.zeros(L)
        pcie_replace = np.zeros(L)
        layer_time = np.zeros(L)
        cpu_busy = 0.0
        gpu_busy = 0.0
        acc1: dict = {}
        acck: dict = {}
        lookups = []
        replacements = []
        token_lat = []
        tokens = 0
        cur_step = None
        token_ms = 0.0
        for i in range(self.n_records):
            r = self.record(i)
            if r.step != cur_step:
                if cur_step is not None:
                    token_lat.append(token_ms + L * self.non_moe)
                cur_step = r.step
                token_ms = 0.0
            l = r.layer
            if self.cache_enabled:
                for e in range(N):
                    if r.G[e]:
                        lookups.append((l, r.token_index, bool(r.hit[e])))
            if self.prefetch_size > 0 and l < L - 1:
                pset = np.array([r.pset[j] for j in range(r.n_pset)], dtype=np.int64)
                true_next = true_workloads[(r.step, l + 1)]
                acc1.setdefault(l + 1, []).append(_accuracy(pset, true_next, 1))
                acck.setdefault(l + 1, []).append(
                    _accuracy(pset, true_next, min(self.prefetch_size, N)))
                pcie_prefetch[l] += r.consumed
            boundary = 0.0
            if r.ev_valid:
                boundary = r.boundary
                pcie_replace[l] += boundary
                if r.ev_n:
                    replacements.append({
                        "token_index": r.token_index, "layer": l,
                        "evicted": [int(r.evicted[j]) for j in range(r.ev_n)],
                        "admitted": [int(r.admitted[j]) for j in range(r.ev_n)],
                        "transfer_cost_ms": boundary})
            pcie_demand[l] += r.demand_ms
            layer_time[l] += r.latency + boundary + self.non_moe
            cpu_busy += r.cpu_busy
            gpu_busy += r.gpu_makespan + self.shared_ms
            token_ms += r.latency + boundary
        if cur_step is not None:
            token_lat.append(token_ms + L * self.non_moe)
        tokens = int(sum(step_tokens[:len(token_lat)]))
        n_steps = len(token_lat)
        total = float(sum(token_lat))
        busy = float(pcie_demand.sum() + pcie_prefetch.sum() + pcie_replace.sum())
        per_layer = {}
        for l in range(L):
            lt = layer_time[l]
            per_layer[str(l)] = float((pcie_demand[l] + pcie_prefetch[l] + pcie_replace[l]) / lt) \
                if lt > 0 else 0.0
        overall, hl, hg, empty = None, {}, {}, []
        if self.cache_enabled and lookups:
            from .cache import CacheStats
            cs = CacheStats(lookups)
            overall = cs.hit_rate("overall")
            hl = cs.hit_rate("per-layer")
            hg, empty = cs.hit_rate("per-token-group", group_size=8)
        return {
            "tokens": tokens, "steps": n_steps, "total_time_ms": total,
            "tokens_per_second": tokens / (total / 1000.0) if total > 0 else 0.0,
            "mean_token_latency_ms": total / n_steps if n_steps else 0.0,
            "cpu_busy_ms": float(cpu_busy), "gpu_busy_ms": float(gpu_busy),
            "pcie_demand_ms": float(pcie_demand.sum()),
            "pcie_prefetch_ms": float(pcie_prefetch.sum()),
            "pcie_replacement_ms": float(pcie_replace.sum()),
            "pcie_busy_ms": busy,
            "pcie_busy_fraction": busy / total if total > 0 else 0.0,
            "per_layer_pcie_fraction": per_layer,
            "prefetch_accuracy_top1": {str(a): float(np.mean(b)) for a, b in sorted(acc1.items())},
            "prefetch_accuracy_topk": {str(a): float(np.mean(b)) for a, b in sorted(acck.items())},
            "prefetch_size": self.prefetch_size,
            "cache_hit_rate": overall,
            "cache_hit_rate_per_layer": {str(a): b for a, b in hl.items()},
            "cache_hit_rate_per_group": {str(a): b for a, b in hg.items()},
            "cache_empty_groups": empty,
            "replacement_events": replacements,
            "spec": spec,
            "timelines": [],
        }

    def decision_log(self) -> list[dict]:
        """Host copy of every record as plain dicts (for parity checks)."""
        out = []
        N = self.N
        for i in range(self.n_records):
            r = self.record(i)
            out.append({
                "step": r.step, "layer": r.layer,
                "C": np.array(r.C[:N], np.int8), "G": np.array(r.G[:N], np.int8),
                "resident": np.array(r.resident[:N], bool),
                "hits": [(e, bool(r.hit[e])) for e in range(N) if r.G[e]],
                "pset": [int(r.pset[j]) for j in range(r.n_pset)],
                "cand": [int(r.cand[j]) for j in range(r.n_cand)],
                "done": [int(r.cand[j]) for j in range(r.n_done)],
                "event": ((([int(r.evicted[j]) for j in range(r.ev_n)],
                            [int(r.admitted[j]) for j in range(r.ev_n)]))
                          if r.ev_valid else None),
                "cpu_busy": r.cpu_busy, "gpu_makespan": r.gpu_makespan,
                "latency": r.latency, "demand_end": r.demand_end,
                "inserts": [(r.layer + (1 if r.ins_kind[j] == 2 else 0), int(r.ins_victim[j]),
                             int(r.ins_expert[j]), ("lru", "demand", "prefetch")[r.ins_kind[j]])
                            for j in range(r.n_ins)],
            })
        return out


def _accuracy(pset, true_workloads, k):
    truth = topk_indices(np.asarray(true_workloads, dtype=np.float64), k)
    return len(set(np.asarray(pset)[:k].tolist()) & set(truth.tolist())) / k
