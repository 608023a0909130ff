"""Data model and gating entry points of the drop-in API.

Mirrors the reference data model (trace.py:34-226: ``ModelConfig``,
``GateParams`` (L, d, N), ``ResidualVectors`` (L-1, d), ``TokenStep``,
``Trace``) with the same field names, invariants and error messages.  The
gating math (``derive_workloads``, trace.py:253-265) runs on the GPU routing
kernel (``dali_route_f64`` / ``dali_route_bf16``); there is no host
implementation of it in this package.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .errors import TraceError

TRACE_FORMAT = "moesim-trace-v1"
GATES_FORMAT = "moesim-gates-v1"
RESIDUALS_FORMAT = "moesim-residuals-v1"

MODEL_PRESETS = {
    "deepseek": dict(num_layers=27, num_routed_experts=64, num_shared_experts=2,
                     top_k=6, hidden_dim=2048),
    "qwen": dict(num_layers=48, num_routed_experts=128, num_shared_experts=0,
                 top_k=8, hidden_dim=2048),
    "mixtral": dict(num_layers=32, num_routed_experts=8, num_shared_experts=0,
                    top_k=2, hidden_dim=4096),
}

_FIELDS = ("num_layers", "num_routed_experts", "num_shared_experts", "top_k", "hidden_dim")


@dataclass(frozen=True)
class ModelConfig:
    """MoE routing shape (reference trace.py:44-86)."""

    num_layers: int
    num_routed_experts: int
    num_shared_experts: int
    top_k: int
    hidden_dim: int

    def __post_init__(self):
        if self.num_layers < 1:
            raise TraceError(f"num_layers must be >= 1, got {self.num_layers}")
        if self.hidden_dim < 1:
            raise TraceError(f"hidden_dim must be >= 1, got {self.hidden_dim}")
        if not (1 <= self.top_k <= self.num_routed_experts):
            raise TraceError(
                f"top_k must be in [1, num_routed_experts], got "
                f"top_k={self.top_k}, num_routed_experts={self.num_routed_experts}")
        if self.num_shared_experts < 0:
            raise TraceError("num_shared_experts must be >= 0")

    def to_dict(self) -> dict:
        return {f: getattr(self, f) for f in _FIELDS}

    @classmethod
    def from_dict(cls, d: dict) -> "ModelConfig":
        return cls(**{f: int(d[f]) for f in _FIELDS})

    @classmethod
    def preset(cls, name: str) -> "ModelConfig":
        if name not in MODEL_PRESETS:
            raise TraceError(f"unknown model preset {name!r}; choose from {sorted(MODEL_PRESETS)}")
        return cls(**MODEL_PRESETS[name])


@dataclass
class GateParams:
    """Per-layer gate matrices, shape (num_layers, hidden_dim, num_routed_experts)."""

    weights: np.ndarray

    def __post_init__(self):
        self.weights = np.asarray(self.weights, dtype=np.float64)
        if self.weights.ndim != 3:
            raise TraceError(f"gate weights must be 3-d (L, d, N), got shape {self.weights.shape}")

    @property
    def num_layers(self) -> int:
        return self.weights.shape[0]

    def layer(self, l: int) -> np.ndarray:
        return self.weights[l]

    def check_shape(self, config: ModelConfig) -> None:
        expect = (config.num_layers, config.hidden_dim, config.num_routed_experts)
        if self.weights.shape != expect:
            raise TraceError(f"gate weights shape {self.weights.shape} does not match model "
                             f"config {expect}")


@dataclass
class ResidualVectors:
    """Calibrated mean inter-layer feature shift, shape (num_layers - 1, hidden_dim)."""

    values: np.ndarray

    def __post_init__(self):
        self.values = np.asarray(self.values, dtype=np.float64)
        if self.values.ndim != 2:
            raise TraceError(f"residual vectors must be 2-d (L-1, d), got shape "
                             f"{self.values.shape}")

    @property
    def num_layers(self) -> int:
        return self.values.shape[0] + 1

    def layer(self, l: int) -> np.ndarray:
        return self.values[l]

    def check_shape(self, config: ModelConfig) -> None:
        expect = (config.num_layers - 1, config.hidden_dim)
        if self.values.shape != expect:
            raise TraceError(f"residual vectors shape {self.values.shape} does not match "
                             f"model config {expect}")

    @classmethod
    def zeros(cls, num_layers: int, hidden_dim: int) -> "ResidualVectors":
        return cls(np.zeros((num_layers - 1, hidden_dim)))


@dataclass
class TokenStep:
    """One decode step or one aggregated prefill step (trace.py:152-171)."""

    token_index: int
    tokens: int
    workloads: np.ndarray
    hidden: np.ndarray | None = None
    eos: bool = False

    def __post_init__(self):
        self.workloads = np.asarray(self.workloads, dtype=np.int64)
        if self.hidden is not None:
            self.hidden = np.asarray(self.hidden, dtype=np.float64)


@dataclass
class Trace:
    """Ordered token steps + model shape + optional gates (trace.py:174-226)."""

    model_config: ModelConfig
    batch_size: int
    phase: str
    steps: list[TokenStep] = field(default_factory=list)
    generator_seed: int = 0
    gate_params: GateParams | None = None
    generator_params: dict = field(default_factory=dict)

    def __post_init__(self):
        if self.phase not in ("prefill", "decode"):
            raise TraceError(f"phase must be 'prefill' or 'decode', got {self.phase!r}")
        if self.batch_size < 1:
            raise TraceError("batch_size must be >= 1")

    @property
    def has_features(self) -> bool:
        return bool(self.steps) and all(s.hidden is not None for s in self.steps)

    @property
    def num_steps(self) -> int:
        return len(self.steps)

    def validate(self, check_gating: bool = False) -> None:
        cfg = self.model_config
        L, N, d = cfg.num_layers, cfg.num_routed_experts, cfg.hidden_dim
        if self.gate_params is not None:
            self.gate_params.check_shape(cfg)
        for i, step in enumerate(self.steps):
            if step.workloads.shape != (L, N):
                raise TraceError(f"step {i}: workloads shape {step.workloads.shape} != ({L}, {N})")
            if (step.workloads < 0).any():
                lay, exp = np.argwhere(step.workloads < 0)[0]
                raise TraceError(f"step {i} layer {lay}: negative workload at expert {exp}")
            if step.hidden is not None and step.hidden.shape != (L, step.tokens, d):
                raise TraceError(f"step {i}: hidden shape {step.hidden.shape} != "
                                 f"({L}, {step.tokens}, {d})")
            if check_gating and step.hidden is not None and self.gate_params is not None:
                for l in range(L):
                    got = derive_workloads(step.hidden[l], self.gate_params.layer(l), cfg.top_k)
                    if not np.array_equal(got, step.workloads[l]):
                        raise TraceError(f"step {i} layer {l}: stored workloads do not match "
                                         f"gating recomputation")


def topk_indices(scores, k: int) -> np.ndarray:
    """Indices of the k largest entries, ties toward the lower index.

    Host helper for metrics (prefetch accuracy, trace.py:236-239); the
    routing path ranks on device."""
    return np.argsort(-np.asarray(scores, dtype=np.float64), kind="stable")[:k]


# ---------------------------------------------------------------------------
# GPU gating
# ---------------------------------------------------------------------------


def gate_norm2(gate: torch.Tensor) -> torch.Tensor:
    """Squared column norms (N,) f32 of a router matrix (d, N): the input of
    the certified routing kernel's error bound (csrc/route_guard.cu).  fp32
    summation is within gamma_d relative of the exact value, which the
    kernel's 1% safety factor covers."""
    return gate.float().square().sum(dim=0).contiguous()


def route_device(hidden: torch.Tensor, gate: torch.Tensor, k: int,
                 residual: torch.Tensor | None = None, renorm: bool = False,
                 want_idx: bool = True, want_weights: bool = True, stream=None, out=None,
                 norm2: torch.Tensor | None = None):
    """Launch the fused routing kernel on device tensors.

    hidden (T, d) float64 or bfloat16; gate (d, N) same dtype family;
    residual (d,) float64 or None; norm2 (N,) f32 squared column norms of a
    bf16 gate (computed here when None).  Returns (topk_idx int32 (T,k) |
    None, topk_w float32 (T,k) | None, workloads int64 (N,)).
    """
    T, d = hidden.shape
    if gate.shape[0] != d:
        raise TraceError(f"hidden dim {d} does not match gate matrix rows {gate.shape[0]}")
    N = gate.shape[1]
    if not (1 <= k <= N):
        raise TraceError(f"top_k {k} out of range for {N} experts")
    dev = hidden.device
    if out is not None:            # caller-owned (idx, wts, wl) workspaces
        idx, wts, wl = out
    else:
        idx = torch.empty((T, k), dtype=torch.int32, device=dev) if want_idx else None
        wts = torch.empty((T, k), dtype=torch.float32, device=dev) if want_weights else None
        wl = torch.empty((N,), dtype=torch.int64, device=dev)
    res_p = _dev.ptr(residual)
    if hidden.dtype == torch.float64:
        fn = "dali_route_f64"
        hp, gp = hidden.data_ptr(), gate.to(torch.float64).contiguous().data_ptr()
        gkeep = None
    elif hidden.dtype == torch.bfloat16:
        gkeep = gate.to(torch.bfloat16).contiguous()
        nkeep = norm2 if norm2 is not None else gate_norm2(gkeep)
        _lib.call("dali_route_bf16", hidden.data_ptr(), res_p, gkeep.data_ptr(),
                  nkeep.data_ptr(), T, d, N, k, int(renorm), _dev.ptr(idx), _dev.ptr(wts),
                  wl.data_ptr(), _dev.stream_ptr(stream))
        return idx, wts, wl
    else:
        raise TraceError(f"unsupported hidden dtype {hidden.dtype}")
    _lib.call(fn, hp, res_p, gp, T, d, N, k, int(renorm), _dev.ptr(idx), _dev.ptr(wts),
              wl.data_ptr(), _dev.stream_ptr(stream))
    del gkeep
    return idx, wts, wl


def derive_workloads(hidden, gate_matrix, k: int) -> np.ndarray:
    """Per-expert token counts of top-k routing (reference trace.py:253-265),
    computed by the GPU routing kernel in fp64."""
    h = np.atleast_2d(np.asarray(hidden, dtype=np.float64))
    g = np.asarray(gate_matrix, dtype=np.float64)
    if h.shape[1] != g.shape[0]:
        raise TraceError(f"hidden dim {h.shape[1]} does not match gate matrix rows {g.shape[0]}")
    if not (1 <= k <= g.shape[1]):
        raise TraceError(f"top_k {k} out of range for {g.shape[1]} experts")
    hd = _dev.to_dev(h, torch.float64)
    gd = _dev.to_dev(g, torch.float64)
    _, _, wl = route_device(hd, gd, k, want_idx=False, want_weights=False)
    return wl.cpu().numpy()


def route_topk(hidden, gate_matrix, k: int) -> np.ndarray:
    """Per-token top-k expert indices (the rows ``topk_indices`` would pick
    for each token's softmax scores), computed on the GPU."""
    hd = _dev.to_dev(np.atleast_2d(np.asarray(hidden, dtype=np.float64)), torch.float64)
    gd = _dev.to_dev(np.asarray(gate_matrix, dtype=np.float64), torch.float64)
    idx, _, _ = route_device(hd, gd, k, want_weights=False)
    return idx.cpu().numpy().astype(np.int64)


# ---------------------------------------------------------------------------
# Synthetic trace generator (reference trace.py:274-375): input fixture with
# the reference's RNG draw order; gating of every (step, layer) runs on GPU.
# ---------------------------------------------------------------------------

_GATE_LOGIT_SCALE = 0.4
_GATE_NORM_SPREAD = (0.15, 1.85)


def synthetic_gates(rng: np.random.Generator, L: int, d: int, N: int) -> np.ndarray:
    """Skewed gate matrices: normal * 0.4/sqrt(d) * permuted column scales."""
    base = rng.normal(size=(L, d, N)) * (_GATE_LOGIT_SCALE / np.sqrt(d))
    scales = rng.permuted(np.tile(np.linspace(*_GATE_NORM_SPREAD, N), (L, 1)), axis=1)
    return base * scales[:, None, :]


def generate_synthetic_trace(config: ModelConfig, batch_size: int, num_steps: int,
                             locality: float = 0.9, drift_scale: float = 0.0,
                             noise_scale: float = 0.0, seed: int = 0,
                             phase: str = "decode") -> Trace:
    if not (0.0 <= locality <= 1.0):
        raise TraceError(f"locality must be in [0, 1], got {locality}")
    if drift_scale < 0 or noise_scale < 0:
        raise TraceError("drift_scale and noise_scale must be >= 0")
    if num_steps < 1:
        raise TraceError("num_steps must be >= 1")
    if batch_size < 1:
        raise TraceError("batch_size must be >= 1")
    rng = np.random.default_rng(seed)
    L, N, d, k = config.num_layers, config.num_routed_experts, config.hidden_dim, config.top_k
    norm = float(np.sqrt(d))
    gates = synthetic_gates(rng, L, d, N)
    if L > 1:
        dirs = rng.normal(size=(L - 1, d))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        drifts = drift_scale * norm * dirs
    else:
        drifts = np.zeros((0, d))

    def renorm(rows):
        n = np.linalg.norm(rows, axis=1, keepdims=True)
        n[n == 0.0] = 1.0
        return rows * (norm / n)

    def stack_of(rows):
        out = np.empty((L,) + rows.shape)
        out[0] = rows
        for l in range(1, L):
            out[l] = out[l - 1] + drifts[l - 1] + rng.normal(size=rows.shape) * noise_scale
        return out

    gdev = [_dev.to_dev(gates[l], torch.float64) for l in range(L)]

    def loads(stack):
        out = np.empty((L, N), dtype=np.int64)
        for l in range(L):
            _, _, wl = route_device(_dev.to_dev(stack[l], torch.float64), gdev[l], k,
                                    want_idx=False, want_weights=False)
            out[l] = wl.cpu().numpy()
        return out

    state = renorm(rng.normal(size=(batch_size, d)))
    steps = []
    if phase == "prefill":
        rows = np.empty((batch_size * num_steps, d))
        for t in range(num_steps):
            rows[t * batch_size:(t + 1) * batch_size] = state
            if t < num_steps - 1:
                state = renorm(locality * state + (1.0 - locality) * rng.normal(size=state.shape))
        st = stack_of(rows)
        steps.append(TokenStep(0, rows.shape[0], loads(st), st, eos=True))
    else:
        for t in range(num_steps):
            st = stack_of(state)
            steps.append(TokenStep(t, batch_size, loads(st), st, eos=(t == num_steps - 1)))
            if t < num_steps - 1:
                state = renorm(locality * state + (1.0 - locality) * rng.normal(size=state.shape))
    return Trace(model_config=config, batch_size=batch_size, phase=phase, steps=steps,
                 generator_seed=seed, gate_params=GateParams(gates),
                 generator_params={"num_steps": num_steps, "locality": locality,
                                   "drift_scale": drift_scale, "noise_scale": noise_scale,
                                   "drift_vectors": drifts.tolist()})


# ---------------------------------------------------------------------------
# Sidecar I/O in the reference formats (trace.py:385-568), so residuals and
# traces produced on the B200 can be replayed by the reference tools.
# ---------------------------------------------------------------------------

def save_residuals(residuals: ResidualVectors, path, spec: dict | None = None) -> None:
    n1, d = residuals.values.shape
    header = {"format": RESIDUALS_FORMAT, "num_layers": n1 + 1, "hidden_dim": d}
    if spec is not None:
        header["spec"] = spec
    with open(path, "w") as f:
        f.write(json.dumps(header) + "\n")
        for l in range(n1):
            f.write(json.dumps({"layer": l, "values": residuals.values[l].tolist()}) + "\n")


def load_residuals(path) -> ResidualVectors:
    with open(path) as f:
        lines = [ln for ln in f.read().splitlines() if ln.strip()]
    if not lines:
        raise TraceError(f"{path}: empty residual file")
    header = json.loads(lines[0])
    if header.get("format") != RESIDUALS_FORMAT:
        raise TraceError(f"{path}:1: not a residual vector file")
    L, d = int(header["num_layers"]), int(header["hidden_dim"])
    vals = np.zeros((L - 1, d))
    seen = set()
    for ln in lines[1:]:
        rec = json.loads(ln)
        l = int(rec["layer"])
        if not (0 <= l < L - 1):
            raise TraceError(f"{path}: layer {l} out of range")
        vals[l] = np.asarray(rec["values"], dtype=np.float64)
        seen.add(l)
    if len(seen) != L - 1:
        raise TraceError(f"{path}: expected {L - 1} residual vectors, found {len(seen)}")
    return ResidualVectors(vals)


def save_trace(trace: Trace, path) -> None:
    """Write ``moesim-trace-v1`` line-delimited JSON (reference trace.py:
    385-406): one header object, then one record per step.  Lets the
    reference's own tools (simulate / cache-eval / report) replay a run the
    B200 engine executed."""
    header = {"format": TRACE_FORMAT, "model_config": trace.model_config.to_dict(),
              "batch_size": trace.batch_size, "phase": trace.phase,
              "generator_seed": trace.generator_seed, "has_features": trace.has_features,
              "generator_params": trace.generator_params}
    with open(path, "w") as f:
        f.write(json.dumps(header) + "\n")
        for st in trace.steps:
            rec = {"token_index": int(st.token_index), "tokens": int(st.tokens),
                   "eos": bool(st.eos), "workloads": st.workloads.tolist()}
            if st.hidden is not None:
                rec["hidden"] = st.hidden.tolist()
            f.write(json.dumps(rec) + "\n")


def load_trace(path) -> Trace:
    """Read a ``moesim-trace-v1`` file (reference trace.py:409-473 semantics:
    structural validation with the offending line number)."""
    with open(path) as f:
        lines = f.readlines()
    if not lines:
        raise TraceError(f"{path}: empty trace file")
    try:
        header = json.loads(lines[0])
    except json.JSONDecodeError as e:
        raise TraceError(f"{path}:1: malformed record: {e}") from e
    if header.get("format") != TRACE_FORMAT:
        raise TraceError(f"{path}:1: not a trace file (format tag {header.get('format')!r})")
    cfg = ModelConfig.from_dict(header["model_config"])
    L, N, d = cfg.num_layers, cfg.num_routed_experts, cfg.hidden_dim
    B = int(header["batch_size"])
    steps = []
    for lineno, line in enumerate(lines[1:], start=2):
        if not line.strip():
            continue
        try:
            rec = json.loads(line)
        except json.JSONDecodeError as e:
            raise TraceError(f"{path}:{lineno}: malformed record: {e}") from e
        wl = np.asarray(rec.get("workloads"), dtype=np.int64)
        if wl.shape != (L, N) or (wl < 0).any():
            raise TraceError(f"{path}:{lineno}: workloads must be ({L}, {N}) nonnegative ints")
        tokens = int(rec.get("tokens", B))
        hid = None
        if "hidden" in rec:
            hid = np.asarray(rec["hidden"], dtype=np.float64)
            if hid.shape != (L, tokens, d):
                raise TraceError(f"{path}:{lineno}: hidden shape {hid.shape} != ({L}, {tokens}, {d})")
        steps.append(TokenStep(int(rec.get("token_index", lineno - 2)), tokens, wl, hid,
                               bool(rec.get("eos", False))))
    tr = Trace(cfg, B, header["phase"], steps, int(header.get("generator_seed", 0)),
               generator_params=header.get("generator_params", {}))
    tr.validate()
    return tr


def save_gate_params(gate: GateParams, path, spec: dict | None = None) -> None:
    """``moesim-gates-v1`` sidecar (reference trace.py:486-496)."""
    L, d, N = gate.weights.shape
    header = {"format": GATES_FORMAT, "num_layers": L, "hidden_dim": d, "num_routed_experts": N}
    if spec is not None:
        header["spec"] = spec
    with open(path, "w") as f:
        f.write(json.dumps(header) + "\n")
        for l in range(L):
            f.write(json.dumps({"layer": l, "weights": gate.weights[l].tolist()}) + "\n")
