"""Residual-based next-layer prefetch (drop-in for reference prefetch.py).

``predict_next_layer`` shifts the current layer's gate inputs by the
calibrated residual and applies the next layer's gate on device (routing
kernel with the residual fused into its shared-memory staging), then picks
the prefetch set with the stable top-P kernel.  ``calibrate_residuals``
(Eq. 11, prefetch.py:88-104) accumulates in fp64 on device.
``prefetch_accuracy`` is a host metric.  The reference's comparison
predictors are here too: "statistical" ranks a calibration frequency table
and "random" ranks a numpy PCG64 permutation (drawn on the host, the same
stream as the reference), both through the device top-P kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _dev, _lib
from .errors import PrefetchError
from .trace import ResidualVectors, Trace, route_device, topk_indices

PREDICTOR_KINDS = ("residual", "feature", "statistical", "random")


@dataclass
class PrefetchDecision:
    layer: int
    predicted_workloads: np.ndarray
    prefetch_set: np.ndarray


@dataclass
class Predictor:
    kind: str
    residuals: ResidualVectors | None = None
    frequency_table: np.ndarray | None = None
    seed: int = 0
    n_experts: int | None = None
    _rng: np.random.Generator | None = field(default=None, repr=False)

    def __post_init__(self):
        if self.kind not in PREDICTOR_KINDS:
            raise PrefetchError(f"unknown predictor kind {self.kind!r}; choose from "
                                f"{PREDICTOR_KINDS}")
        if self.kind == "residual" and self.residuals is None:
            raise PrefetchError("residual predictor requires calibrated residual vectors")
        if self.kind == "statistical" and self.frequency_table is None:
            raise PrefetchError("statistical predictor requires a calibration frequency table")
        if self.kind == "random":
            self._rng = np.random.default_rng(self.seed)


def statistical_predictor(calibration_trace: Trace) -> Predictor:
    """Rank experts by per-layer activation counts (prefetch.py:63-66)."""
    return Predictor(kind="statistical",
                     frequency_table=activation_frequency_table(calibration_trace))


def random_predictor(seed: int = 0, n_experts: int | None = None) -> Predictor:
    return Predictor(kind="random", seed=seed, n_experts=n_experts)


def activation_frequency_table(trace: Trace) -> np.ndarray:
    """Per-layer summed workloads over all steps, (L, N) (prefetch.py:76-85)."""
    if not trace.steps:
        raise PrefetchError("calibration trace has no steps")
    return np.sum(np.stack([np.asarray(s.workloads, dtype=np.int64) for s in trace.steps]),
                  axis=0)


def residual_predictor(residuals: ResidualVectors) -> Predictor:
    return Predictor(kind="residual", residuals=residuals)


def feature_predictor() -> Predictor:
    return Predictor(kind="feature")


def calibrate_residuals(calibration_trace: Trace) -> ResidualVectors:
    """Mean adjacent-layer gate-input delta over all calibration tokens,
    accumulated in fp64 on device."""
    if not calibration_trace.has_features:
        raise PrefetchError("residual calibration requires a trace with hidden states")
    cfg = calibration_trace.model_config
    if cfg.num_layers < 2:
        raise PrefetchError("residual calibration requires at least two layers")
    acc = None
    count = 0
    for st in calibration_trace.steps:
        h = _dev.to_dev(st.hidden, torch.float64)          # (L, T, d)
        tok = h.sum(dim=1)
        delta = tok[1:] - tok[:-1]
        acc = delta if acc is None else acc + delta
        count += st.hidden.shape[1]
    if count == 0:
        raise PrefetchError("calibration trace contains no tokens")
    return ResidualVectors((acc / count).cpu().numpy())


def select_prefetch_set(predicted: torch.Tensor, prefetch_size: int) -> torch.Tensor:
    """Stable top-P of device workloads (prefetch.py:153-156)."""
    N = predicted.shape[0]
    P = min(prefetch_size, N)
    out = torch.empty((max(P, 0),), dtype=torch.int32, device=predicted.device)
    _lib.call("dali_prefetch_select", predicted.data_ptr(), N, P, out.data_ptr(),
              _dev.stream_ptr())
    return out


def predict_next_layer(predictor: Predictor, hidden_states, gate_next, k: int,
                       prefetch_size: int, current_layer: int) -> PrefetchDecision:
    if prefetch_size < 0:
        raise PrefetchError("prefetch_size must be >= 0")
    if predictor.kind in ("statistical", "random"):
        if predictor.kind == "statistical":
            table = predictor.frequency_table
            if not (0 <= current_layer + 1 < table.shape[0]):
                raise PrefetchError(f"layer {current_layer + 1} outside calibration table with "
                                    f"{table.shape[0]} layers")
            predicted = np.asarray(table[current_layer + 1], dtype=np.int64).copy()
        else:
            n = predictor.n_experts
            if n is None and gate_next is not None:
                n = np.asarray(gate_next).shape[1]
            if n is None:
                raise PrefetchError("random predictor needs n_experts or gate_next to size its "
                                    "score vector")
            predicted = predictor._rng.permutation(n).astype(np.int64)
        pset = select_prefetch_set(_dev.to_dev(predicted, torch.int64), prefetch_size)
        return PrefetchDecision(layer=current_layer + 1, predicted_workloads=predicted,
                                prefetch_set=pset.cpu().numpy().astype(np.int64))
    if hidden_states is None or gate_next is None:
        raise PrefetchError(f"{predictor.kind} predictor requires hidden states and the next "
                            f"layer's gate")
    h = np.atleast_2d(np.asarray(hidden_states, dtype=np.float64))
    res = None
    if predictor.kind == "residual":
        if current_layer >= predictor.residuals.num_layers - 1:
            raise PrefetchError(f"no residual vector for layer {current_layer}; the last layer "
                                f"has nothing to prefetch")
        res = _dev.to_dev(predictor.residuals.layer(current_layer), torch.float64)
    _, _, wl = route_device(_dev.to_dev(h, torch.float64),
                            _dev.to_dev(np.asarray(gate_next, dtype=np.float64), torch.float64),
                            k, residual=res, want_idx=False, want_weights=False)
    pset = select_prefetch_set(wl, prefetch_size)
    return PrefetchDecision(layer=current_layer + 1,
                            predicted_workloads=wl.cpu().numpy(),
                            prefetch_set=pset.cpu().numpy().astype(np.int64))


def prefetch_accuracy(predicted_set, true_workloads, k: int) -> float:
    """Share of the true top-k experts in the predicted top-k (prefetch.py:159-168)."""
    predicted_set = np.asarray(predicted_set)
    if k < 1:
        raise PrefetchError("k must be >= 1")
    if len(predicted_set) < k:
        raise PrefetchError(f"predicted set has {len(predicted_set)} experts, need at least k={k}")
    truth = topk_indices(np.asarray(true_workloads, dtype=np.float64), k)
    return len(set(predicted_set[:k].tolist()) & set(truth.tolist())) / k
