"""CPU reference arm (TEST / BASELINE INFRASTRUCTURE; never the GPU path).

The reference (``moesim``) only simulates; its CPU restatement of the
path, timed on the GPU box's host cores, is the paper's "Naive" hybrid
baseline with no GPU: gating by the reference algorithm
(fp64 softmax + stable top-k, oracle.policy.route restating
trace.py:229-265) and every routed expert executed on the CPU, plus the
same attention.  torch CPU (oneDNN, AMX-bf16) with all host threads.

Two bounds: ``run_full_depth`` (the ``--impl reference`` arm) materialises
every layer and times consecutive decode tokens through all of them, with
no scaling; ``run_sample`` (the GPU arm's in-process ``cpu_baseline``, where
the engine's own 91 GB host store already occupies host memory) times
``layers`` of the model's L layers and scales by L / layers.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np
import torch
import torch.nn.functional as F

from . import policy as P


class CpuMoE:
    def __init__(self, d, f, N, k, H, KV, hd, layers, norm_topk, seed=0, max_seq=1024):
        torch.manual_seed(seed)
        self.d, self.f, self.N, self.k, self.H, self.KV, self.hd = d, f, N, k, H, KV, hd
        self.layers, self.norm_topk = layers, norm_topk
        bf = torch.bfloat16
        tile = (torch.rand(1 << 20) * 2 - 1).to(bf)

        def rnd(shape, std):
            n = math.prod(shape)
            reps = (n + tile.numel() - 1) // tile.numel()
            t = tile.repeat(reps)[:n].view(shape) * (std * math.sqrt(3))
            return t.contiguous()

        self.wqkv = [rnd(((H + 2 * KV) * hd, d), d ** -0.5) for _ in range(layers)]
        self.wo = [rnd((d, H * hd), (H * hd) ** -0.5) for _ in range(layers)]
        rng = np.random.default_rng(seed)
        self.router = []
        for _ in range(layers):
            g = rng.normal(size=(d, N)) * (0.4 / math.sqrt(d))
            g *= rng.permutation(np.linspace(0.15, 1.85, N))[None, :]
            self.router.append(g)
        self.w13 = [[rnd((2 * f, d), d ** -0.5) for _ in range(N)] for _ in range(layers)]
        self.w2 = [[rnd((d, f), f ** -0.5) for _ in range(N)] for _ in range(layers)]
        self.max_seq = max_seq

    def reset(self, B):
        self.kc = [torch.zeros(B, self.KV, self.max_seq, self.hd, dtype=torch.bfloat16)
                   for _ in range(self.layers)]
        self.vc = [torch.zeros_like(c) for c in self.kc]
        self.pos = 0

    def _attn(self, l, x, B, S):
        H, KV, hd = self.H, self.KV, self.hd
        qkv = x @ self.wqkv[l].t()
        q = qkv[:, :H * hd].view(B, S, H, hd).transpose(1, 2)
        kk = qkv[:, H * hd:(H + KV) * hd].view(B, S, KV, hd).transpose(1, 2)
        vv = qkv[:, (H + KV) * hd:].view(B, S, KV, hd).transpose(1, 2)
        p = self.pos
        self.kc[l][:, :, p:p + S] = kk
        self.vc[l][:, :, p:p + S] = vv
        o = F.scaled_dot_product_attention(q, self.kc[l][:, :, :p + S], self.vc[l][:, :, :p + S],
                                           is_causal=(S > 1), enable_gqa=(H != KV))
        return o.transpose(1, 2).reshape(B * S, H * hd) @ self.wo[l].t()

    def _moe(self, l, h):
        idx, score, _ = P.route(h.double().numpy(), self.router[l], self.k)
        if self.norm_topk:
            score = score / score.sum(axis=1, keepdims=True)
        y = torch.zeros(h.shape, dtype=torch.float32)
        f = self.f
        for e in range(self.N):
            tok, slot = np.nonzero(idx == e)
            if len(tok) == 0:
                continue
            xr = h[torch.from_numpy(tok)]
            gu = (xr @ self.w13[l][e].t()).view(len(tok), f // 64, 2, 64)
            g = gu[:, :, 0].reshape(len(tok), f).float()
            u = gu[:, :, 1].reshape(len(tok), f).float()
            out = ((F.silu(g) * u).to(torch.bfloat16) @ self.w2[l][e].t()).float()
            y.index_add_(0, torch.from_numpy(tok),
                         out * torch.from_numpy(score[tok, slot]).float()[:, None])
        return y

    def step(self, x, B, S):
        """One pass of the sampled layers over (B*S, d) bf16 activations."""
        for l in range(self.layers):
            xn = x.float()
            xn = (xn * torch.rsqrt(xn.pow(2).mean(-1, keepdim=True) + 1e-5)).to(torch.bfloat16)
            x = x + self._attn(l, xn, B, S)
            h = x.float()
            h = (h * torch.rsqrt(h.pow(2).mean(-1, keepdim=True) + 1e-5)).to(torch.bfloat16)
            x = (x.float() + self._moe(l, h)).to(torch.bfloat16)
        self.pos += S
        return x


def run_sample(arch_dims: dict, total_layers: int, prefill: int, decode_steps: int, batch=1,
               sample_layers=2, threads=None, seed=0):
    """Time prefill and decode of the sampled layers; return scaled tokens/s."""
    threads = threads or len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    m = CpuMoE(layers=sample_layers, seed=seed, max_seq=prefill + decode_steps + 1, **arch_dims)
    m.reset(batch)
    g = torch.Generator().manual_seed(seed)
    x = (torch.randn(batch * prefill, arch_dims["d"], generator=g)).to(torch.bfloat16)
    t0 = time.perf_counter()
    m.step(x, batch, prefill)
    t_pre = (time.perf_counter() - t0) * total_layers / sample_layers
    t0 = time.perf_counter()
    for _ in range(decode_steps):
        x = torch.randn(batch, arch_dims["d"], generator=g).to(torch.bfloat16)
        m.step(x, batch, 1)
    t_dec = (time.perf_counter() - t0) * total_layers / sample_layers
    return {"prefill_tokens_per_s": batch * prefill / t_pre,
            "decode_tokens_per_s": batch * decode_steps / t_dec,
            "threads": threads,
            "sample": f"{sample_layers} of {total_layers} layers (time x{total_layers}/"
                      f"{sample_layers}), prefill {prefill} x B{batch}, {decode_steps} decode "
                      f"steps, all experts on CPU, fp64 reference gating"}


def run_full_depth(arch_dims: dict, total_layers: int, prefill: int, decode: int, steps: int,
                   warmup: int, batch: int = 1, chunk: int = 8, threads=None, seed: int = 0,
                   log=None):
    """The reference arm at FULL depth: every one of the model's layers is
    materialised (Mixtral-8x7B: 90 GB of host weights) and run; nothing is
    scaled.  One request = a ``prefill``-token prompt, then ``decode`` - 1
    decode tokens (the first generated token comes from the prefill).  One
    bench step = the next ``chunk`` decode tokens of the current request; a
    request that reaches its last decode position is restarted with a new
    prompt (that prefill is timed into ``prefill_tokens_per_s``).  So K steps
    time K x chunk consecutive decode tokens across every decode position,
    each through all layers, and every expert on the host cores."""
    threads = threads or len(os.sched_getaffinity(0))
    torch.set_num_threads(threads)
    t_init = time.perf_counter()
    m = CpuMoE(layers=total_layers, seed=seed, max_seq=prefill + decode + 1, **arch_dims)
    t_init = time.perf_counter() - t_init
    g = torch.Generator().manual_seed(seed)
    d = arch_dims["d"]
    pre = []

    def new_request():
        m.reset(batch)
        x = torch.randn(batch * prefill, d, generator=g).to(torch.bfloat16)
        t0 = time.perf_counter()
        m.step(x, batch, prefill)
        pre.append(time.perf_counter() - t0)
        if log:
            log(f"reference arm: prefill {batch * prefill / pre[-1]:.1f} tok/s")

    new_request()
    left = max(decode - 1, 1)
    dec_tokens, dec_time, per_step = 0, 0.0, []
    for i in range(warmup + steps):
        n = min(chunk, left)
        t0 = time.perf_counter()
        for _ in range(n):
            x = torch.randn(batch, d, generator=g).to(torch.bfloat16)
            m.step(x, batch, 1)
        dt = time.perf_counter() - t0
        if i >= warmup:
            dec_tokens += batch * n
            dec_time += dt
            per_step.append(dt)
        if log:
            log(f"reference arm step {i}: {batch * n / dt:.2f} decode tok/s")
        left -= n
        if left <= 0:
            new_request()
            left = max(decode - 1, 1)
    return {"prefill_tokens_per_s": batch * prefill / float(np.mean(pre)),
            "decode_tokens_per_s": dec_tokens / dec_time,
            "step_seconds": per_step, "threads": threads, "init_s": round(t_init, 1),
            "sample": f"all {total_layers} layers (no scaling); each step = the next {chunk} "
                      f"decode tokens of a prefill {prefill} + decode {decode} request "
                      f"(B{batch}), requests restarted at their last position, so {steps} "
                      f"timed steps cover {dec_tokens} consecutive decode positions; "
                      f"{len(pre)} full-depth prefills timed; all experts on the CPU "
                      f"(torch oneDNN bf16), fp64 reference gating"}


def policy_layer_timing(d: int, N: int, k: int, capacity: int, prefetch_size: int,
                        tokens: int = 1, reps: int = 5, seed: int = 0) -> dict:
    """Per-layer decision latency of the reference policy on the host
    (SURVEY.md section 8d (i)): gating A4 (trace.py:229-265), greedy A6-A8
    (cost_model.py:70-96, assignment.py:53-199), residual prediction A11
    (prefetch.py:107-156) and the cache window update A16 (cache.py:146-214),
    restated in oracle.policy; 1 warm-up + best of ``reps`` per function, in
    microseconds.  ``tokens`` = T of the layer (1 for B=1 decode)."""
    rng = np.random.default_rng(seed)
    h = rng.standard_normal((tokens, d))
    gate = rng.standard_normal((d, N)) * (0.4 / math.sqrt(d))
    gate_next = rng.standard_normal((d, N)) * (0.4 / math.sqrt(d))
    res = rng.standard_normal(d) * 0.01
    tables = P.default_tables()
    cache = P.new_cache(0, N, capacity, 4, P.default_u_size(N, capacity), seed=seed)
    wl = P.derive_workloads(h, gate, k)
    cpu_t, gpu_t = P.expert_times(tables, wl, cache.on_gpu)

    def best(fn):
        fn()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            fn()
            ts.append((time.perf_counter() - t0) * 1e6)
        return min(ts)

    out = {
        "gating_A4": best(lambda: P.derive_workloads(h, gate, k)),
        "greedy_A6_A8": best(lambda: P.greedy(wl, cache.on_gpu,
                                              *P.expert_times(tables, wl, cache.on_gpu),
                                              capacity)),
        "prefetch_A11": best(lambda: P.predict_next(h, res, gate_next, k, prefetch_size)),
        "cache_A16": best(lambda: P.window_update(cache, wl, False)),
    }
    out["total"] = sum(out.values())
    return {key: round(v, 2) for key, v in out.items()}
