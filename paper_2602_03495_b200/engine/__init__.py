"""Real MoE inference with DALI offloading (new API; the reference pkg only
simulates).  ``build_engine`` wires random-init weights of a preset shape,
a cost model (measured on this box or given), residual vectors and the
``OffloadEngine``; ``OffloadEngine.generate`` is the user-facing call."""

from __future__ import annotations

import numpy as np
import torch

from .arch import PRESETS, MoEArch, preset
from .offload import EngineConfig, OffloadEngine, RunStats
from .weights import ModelWeights


def calibrate_residuals_engine(arch: MoEArch, weights: ModelWeights, cost_model, prompts,
                               max_seq: int = 1024, ep=None) -> np.ndarray:
    """On-GPU residual calibration (Eq. 11, prefetch.py:88-104 semantics):
    run calibration prompts through an all-GPU engine pass, capture every
    layer's gate input and average h_{l+1} - h_l over tokens in fp64."""
    eng = OffloadEngine(arch, weights, cost_model,
                        EngineConfig(capture=True, cache_slots_per_layer=0,
                                     assignment="greedy"),
                        max_batch=prompts.shape[0], max_seq=max_seq, ep=ep)
    eng.generate(prompts, 1)
    L = arch.num_layers
    per_layer = {}
    for (step, l, h) in eng.stats.captured:
        per_layer.setdefault(step, {})[l] = h
    acc = None
    count = 0
    for step, hs in per_layer.items():
        stack = torch.stack([hs[l].to(torch.float64) for l in range(L)]).cuda()   # (L, T, d)
        tok = stack.sum(dim=1)
        delta = tok[1:] - tok[:-1]
        acc = delta if acc is None else acc + delta
        count += stack.shape[1]
    return (acc / count).cpu().numpy()


def build_engine(name: str, cfg: EngineConfig, seed: int = 0, cost_model=None,
                 residuals: np.ndarray | None = None, resident: bool = False,
                 max_batch: int = 1, max_seq: int = 1024, calib_prompt_len: int = 64,
                 log=None, weights: ModelWeights | None = None, ep=None) -> OffloadEngine:
    """``ep``: an ``ep.EPGroup`` for expert parallelism (this rank then holds
    only its expert shard); None = every expert on this GPU's engine."""
    from .profiler import profile_cost_model
    arch = preset(name)
    experts = ep.local_experts if ep is not None else None
    if ep is not None and not resident and weights is None and cfg.cache_gb is not None:
        # EP: the shard stays in HBM whenever the per-GPU expert budget covers
        # it -- aggregate HBM is the point of expert parallelism (Mixtral-8x7B
        # at G >= 4 under 24 GB, Mixtral-8x22B at G = 8 under 34 GB).  A shard
        # the budget does not cover is cached like the 1-GPU engine, with
        # capacity min(budget blocks / L, NL - 1) slots per layer (the
        # reference's 0 < capacity < N rule, cache.py:75-78).
        shard = arch.num_layers * len(experts) * arch.expert_bytes
        if shard <= cfg.cache_gb * 1e9:
            resident = True
            if log is not None:
                log(f"EP shard of {len(experts)} experts x {arch.num_layers} layers "
                    f"({shard / 1e9:.1f} GB) fits the {cfg.cache_gb} GB budget: resident")
    w = weights if weights is not None else ModelWeights(arch, seed=seed, resident=resident,
                                                         experts=experts)
    if cost_model is None:
        cost_model = profile_cost_model(arch, w, log=log, threads=cfg.cpu_threads)
    if residuals is None and cfg.prefetch_size > 0 and not resident:
        g = torch.Generator().manual_seed(seed + 99)
        prompts = torch.randint(0, arch.vocab_size, (1, calib_prompt_len), generator=g)
        residuals = calibrate_residuals_engine(arch, w, cost_model, prompts, max_seq, ep=ep)
    return OffloadEngine(arch, w, cost_model, cfg, residuals=residuals, max_batch=max_batch,
                         max_seq=max_seq, ep=ep)


def smoke_engine() -> None:
    """Tiny config, cache + prefetch on: one short generation on cuda:0."""
    from ..cost_model import default_cost_model
    eng = build_engine("tiny", EngineConfig(cache_slots_per_layer=2, prefetch_size=1),
                       cost_model=default_cost_model(non_moe_layer_time=3.0), max_seq=64)
    prompt = torch.randint(0, eng.arch.vocab_size, (1, 16))
    toks, st = eng.generate(prompt, 4)
    assert toks.shape == (1, 4)
    rep = eng.policy_report()
    assert rep["steps"] == 4 and st.dali_launches > 0


__all__ = ["PRESETS", "MoEArch", "preset", "EngineConfig", "OffloadEngine", "RunStats",
           "ModelWeights", "build_engine", "calibrate_residuals_engine", "smoke_engine"]
