"""CPU fp32 restatement of the MoE forward (TEST INFRASTRUCTURE).

Numeric oracle for hidden states and logits.  The reference has no model
(SPEC.md:8 scopes out FFN math), so this is "parity unpinned" by any
reference test: it restates the paper's Eq. (1)-(2) with
Mixtral-convention SwiGLU experts W2 (silu(W1 x) * W3 x), pre-norm
residual blocks, GQA attention with rotate-half RoPE, and the engine's
expert block layout (W13 rows interleaved in 64-row gate/up groups).

Everything is computed in fp32 from the engine's bf16 weights over the full
sequence (no KV cache).  Routing can be teacher-forced with the engine's
per-layer top-k indices (``topk_override``), so one near-tie flip cannot
cascade; the combine weights are always recomputed here from this model's
own gate logits (softmax, optionally renormalised over the selected k).
"""

from __future__ import annotations

import torch
import torch.nn.functional as F


def _rms(x, eps):
    return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps)


def _rope(x, pos, theta):
    hd = x.shape[-1]
    inv = 1.0 / (theta ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    fr = torch.outer(pos.double(), inv)
    c, s = fr.cos().float()[None, :, None, :], fr.sin().float()[None, :, None, :]
    h = hd // 2
    x1, x2 = x[..., :h], x[..., h:]
    return torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)


def expert_forward(x, block, d, f):
    """SwiGLU of rows x (R, d) with one interleaved expert block (fp32)."""
    n13 = 2 * f * d
    W13 = block[:n13].view(2 * f, d).float().view(f // 64, 2, 64, d)
    W1 = W13[:, 0].reshape(f, d)
    W3 = W13[:, 1].reshape(f, d)
    W2 = block[n13:].view(d, f).float()
    return (F.silu(x @ W1.t()) * (x @ W3.t())) @ W2.t()


def forward(arch, dense, expert_block, tokens, topk_override=None):
    """Full-sequence forward.

    dense: dict of CPU tensors (embed, lm_head, final_norm, attn_norm[L],
      moe_norm[L], wqkv[L], wo[L], router[L] (d, N)).
    expert_block(l, e) -> bf16 CPU tensor of the block.
    tokens (B, S) int64.  topk_override: dict l -> (B*S, k) int64 indices.
    Returns (logits (B, S, V) fp32, gate_inputs list[L] of (B*S, d) fp32).
    """
    a = arch
    B, S = tokens.shape
    d, H, KV, hd = a.hidden_dim, a.num_heads, a.num_kv_heads, a.head_dim
    x = dense["embed"][tokens.reshape(-1)].float()
    pos = torch.arange(S)
    gate_inputs = []
    for l in range(a.num_layers):
        hn = _rms(x, a.rms_eps) * dense["attn_norm"][l].float()
        qkv = hn @ dense["wqkv"][l].float().t()
        q = qkv[:, :H * hd].view(B, S, H, hd)
        k = qkv[:, H * hd:(H + KV) * hd].view(B, S, KV, hd)
        v = qkv[:, (H + KV) * hd:].view(B, S, KV, hd)
        q, k = _rope(q, pos, a.rope_theta), _rope(k, pos, a.rope_theta)
        rep = H // KV
        k = k.repeat_interleave(rep, dim=2)
        v = v.repeat_interleave(rep, dim=2)
        o = F.scaled_dot_product_attention(q.transpose(1, 2), k.transpose(1, 2),
                                           v.transpose(1, 2), is_causal=True)
        x = x + o.transpose(1, 2).reshape(B * S, H * hd) @ dense["wo"][l].float().t()
        h = _rms(x, a.rms_eps) * dense["moe_norm"][l].float()
        gate_inputs.append(h)
        probs = torch.softmax(h.double() @ dense["router"][l].double(), dim=-1)
        if topk_override is not None and l in topk_override:
            idx = topk_override[l]
        else:
            idx = torch.sort(-probs, dim=-1, stable=True).indices[:, :a.top_k]
        sel = torch.gather(probs, 1, idx)
        if a.norm_topk_prob:
            sel = sel / sel.sum(-1, keepdim=True)
        y = torch.zeros_like(x)
        for e in range(a.num_experts):
            rows, slot = torch.nonzero(idx == e, as_tuple=True)
            if len(rows) == 0:
                continue
            out = expert_forward(h[rows], expert_block(l, e), d, a.ffn_dim)
            y.index_add_(0, rows, out * sel[rows, slot].float()[:, None])
        if a.num_shared_experts > 0:
            ys = expert_forward(h, dense["shared"][l], d, a.shared_ffn_dim)
            if a.shared_gate:
                ys = ys * torch.sigmoid(h @ dense["shared_gate"][l].float().t())
            y = y + ys
        x = x + y
    xf = _rms(x, a.rms_eps) * dense["final_norm"].float()
    logits = xf @ dense["lm_head"].float().t()
    return logits.view(B, S, -1), gate_inputs


def dense_from_weights(w):
    """CPU copies of an engine ``ModelWeights``' dense tensors."""
    L = w.arch.num_layers
    return {
        "embed": w.embed.cpu(), "lm_head": w.lm_head.cpu(), "final_norm": w.final_norm.cpu(),
        "attn_norm": [w.attn_norm[l].cpu() for l in range(L)],
        "moe_norm": [w.moe_norm[l].cpu() for l in range(L)],
        "wqkv": [w.wqkv[l].cpu() for l in range(L)], "wo": [w.wo[l].cpu() for l in range(L)],
        "router": [w.router[l].cpu() for l in range(L)],
        "shared": [b.cpu() for b in w.shared],
        "shared_gate": [g.cpu() for g in w.shared_gate],
    }
