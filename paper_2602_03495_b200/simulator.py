"""Trace-driven run of the DALI policies on the GPU (drop-in for
reference simulator.py's ``SimConfig`` / ``simulate_run`` / ``RunReport``).

``simulate_run`` replays a trace's per-(step, layer) workloads and gate
inputs through the device-resident ``PolicyEngine``: the residual predictor
runs on the routing kernel and every assignment / lookup / prefetch-window /
cache decision is made by the fused single-CTA policy kernel.  The report is
assembled from the device decision log with the reference's accumulation
order, so on identical inputs it equals ``moesim.simulate_run(...).to_dict()``
(minus the ``timelines`` detail).  Every reference policy runs on the
device: greedy / beam / branch-and-bound optimal / static-threshold /
all-cpu / all-gpu assignment, residual / feature / statistical / random
predictors (the random predictor's numpy PCG64 draws are made on the host),
workload / LRU / score caches and the insert toggles.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _dev
from .cost_model import CostModel
from .errors import SimulationError
from .policy_engine import PolicyEngine, default_u_size  # noqa: F401  (re-export)
from .trace import ResidualVectors, Trace

ASSIGNMENT_POLICIES = ("greedy", "optimal", "beam", "all-cpu", "all-gpu", "static-threshold")


@dataclass
class SimConfig:
    """Same field names and defaults as the reference (simulator.py:45-106)."""

    cost_model: CostModel
    assignment_policy: str = "greedy"
    beam_width: int = 2
    threshold: float | None = None
    gpu_capacity: int | None = None
    exact_solver_limit: int = 24

    prefetch_kind: str | None = None
    prefetch_size: int = 0
    residuals: ResidualVectors | None = None
    frequency_table: np.ndarray | None = None

    cache_policy: str | None = None
    cache_capacity: int = 0
    w_size: int = 4
    u_size: int | None = None
    insert_demand_fetched: bool = False
    insert_prefetched: bool = False

    scheduling_overhead_ms: float = 0.0
    solver_node_cost_ms: float = 0.0
    prefetch_compute_ms: float = 0.0
    non_moe_override: float | None = None

    seed: int = 0
    keep_timelines: bool = False

    @property
    def prefetch_enabled(self) -> bool:
        return self.prefetch_kind is not None and self.prefetch_size > 0

    @property
    def cache_enabled(self) -> bool:
        return self.cache_policy is not None and self.cache_capacity > 0

    def to_dict(self) -> dict:
        return {
            "assignment_policy": self.assignment_policy, "beam_width": self.beam_width,
            "threshold": self.threshold, "gpu_capacity": self.gpu_capacity,
            "exact_solver_limit": self.exact_solver_limit, "prefetch_kind": self.prefetch_kind,
            "prefetch_size": self.prefetch_size, "has_residuals": self.residuals is not None,
            "cache_policy": self.cache_policy, "cache_capacity": self.cache_capacity,
            "w_size": self.w_size, "u_size": self.u_size,
            "insert_demand_fetched": self.insert_demand_fetched,
            "insert_prefetched": self.insert_prefetched,
            "scheduling_overhead_ms": self.scheduling_overhead_ms,
            "solver_node_cost_ms": self.solver_node_cost_ms,
            "prefetch_compute_ms": self.prefetch_compute_ms,
            "non_moe_override": self.non_moe_override, "seed": self.seed,
            "cost_model": self.cost_model.to_dict(),
        }


@dataclass
class RunReport:
    data: dict

    def to_dict(self) -> dict:
        return {k: v for k, v in self.data.items() if not k.startswith("_")}

    @property
    def decisions(self) -> list:
        return self.data.get("_decisions", [])

    def __getattr__(self, name):
        d = self.__dict__.get("data", {})
        if name in d:
            return d[name]
        raise AttributeError(name)


def _check(trace: Trace, config: SimConfig) -> None:
    """Configuration checks with the reference's messages
    (_validate_run_config / _build_predictor, simulator.py:266-315)."""
    cfg = trace.model_config
    if config.assignment_policy not in ASSIGNMENT_POLICIES:
        raise SimulationError(f"unknown assignment policy {config.assignment_policy!r}; "
                              f"choose from {ASSIGNMENT_POLICIES}")
    if config.prefetch_enabled:
        if not trace.has_features:
            raise SimulationError("prefetching requires a trace with hidden states")
        if config.prefetch_kind in ("residual", "feature") and trace.gate_params is None:
            raise SimulationError("feature-based prefetching requires the trace's gate "
                                  "parameters (sidecar file)")
        if config.prefetch_size > cfg.num_routed_experts:
            raise SimulationError("prefetch_size cannot exceed the expert count")
    if config.cache_enabled:
        if not (0 < config.cache_capacity < cfg.num_routed_experts):
            raise SimulationError(f"cache capacity must be in (0, {cfg.num_routed_experts}), "
                                  f"got {config.cache_capacity}")
        if config.cache_policy == "score" and not (trace.has_features
                                                   and trace.gate_params is not None):
            raise SimulationError("score cache policy requires a featureful trace with gate "
                                  "parameters")
    if config.threshold is not None and config.threshold < 0:
        raise SimulationError("static threshold must be >= 0")
    if config.prefetch_enabled:
        kind = config.prefetch_kind
        if kind == "residual":
            if config.residuals is None:
                raise SimulationError("residual prefetching requires calibrated residual "
                                      "vectors; run the calibrate step first")
            config.residuals.check_shape(cfg)
        elif kind == "statistical":
            if config.frequency_table is None:
                raise SimulationError("statistical prefetching requires a calibration "
                                      "frequency table")
        elif kind not in ("feature", "random"):
            raise SimulationError(f"unknown prefetch kind {kind!r}")


def simulate_run(trace: Trace, config: SimConfig) -> RunReport:
    _check(trace, config)
    cfg = trace.model_config
    L, N, k, d = cfg.num_layers, cfg.num_routed_experts, cfg.top_k, cfg.hidden_dim
    dev = _dev.require_cuda()
    pre = config.prefetch_enabled
    feat = pre and config.prefetch_kind in ("residual", "feature")
    score = config.cache_enabled and config.cache_policy == "score"
    res_dev = None
    if feat:
        res = (config.residuals.values if config.prefetch_kind == "residual"
               else np.zeros((L - 1, d)))
        res_dev = torch.from_numpy(np.ascontiguousarray(res)).to(dev)
    gates = None
    if feat or score:
        gates = torch.from_numpy(np.ascontiguousarray(trace.gate_params.weights)).to(dev)
    n_steps = len(trace.steps)
    eng = PolicyEngine(L, N, k, config.cost_model, assignment=config.assignment_policy,
                       gpu_capacity=config.gpu_capacity,
                       prefetch_size=config.prefetch_size if pre else 0, residuals=res_dev,
                       cache_capacity=config.cache_capacity if config.cache_enabled else 0,
                       w_size=config.w_size, u_size=config.u_size, seed=config.seed,
                       num_shared_experts=cfg.num_shared_experts,
                       scheduling_overhead_ms=config.scheduling_overhead_ms,
                       solver_node_cost_ms=config.solver_node_cost_ms,
                       prefetch_compute_ms=config.prefetch_compute_ms,
                       non_moe_override=config.non_moe_override,
                       max_records=max(1, n_steps * L), beam_width=config.beam_width,
                       threshold=config.threshold,
                       exact_solver_limit=config.exact_solver_limit,
                       cache_policy=config.cache_policy or "workload",
                       insert_demand_fetched=config.insert_demand_fetched,
                       insert_prefetched=config.insert_prefetched,
                       prefetch_kind=config.prefetch_kind or "residual",
                       frequency_table=(np.asarray(config.frequency_table)
                                        if pre and config.prefetch_kind == "statistical"
                                        else None))
    eng.new_run()
    true_wl = {}
    tokens = []
    for si, st in enumerate(trace.steps):
        wl = torch.from_numpy(np.ascontiguousarray(st.workloads, dtype=np.int64)).to(dev)
        hid = (torch.from_numpy(np.ascontiguousarray(st.hidden)).to(dev)
               if (feat or score) and st.hidden is not None else None)
        for l in range(L):
            true_wl[(si, l)] = st.workloads[l]
            eng.layer_step(si, l, st.token_index, st.eos, wl[l],
                           hid[l] if hid is not None else None,
                           gates[l + 1] if (feat and l < L - 1) else None,
                           gate_this=gates[l] if score else None)
        tokens.append(st.tokens)
        if st.eos:
            break
    torch.cuda.synchronize()
    eng.check_errors()
    rep = eng.build_report(tokens, true_wl, config.to_dict())
    rep["_decisions"] = eng.decision_log()
    return RunReport(rep)
