"""Non-MoE layer pieces (attention, RMSNorm, RoPE, embeddings, LM head).

These are outside the five DALI subsystems ("use
PyTorch"): torch SDPA (flash backend) with a preallocated GQA KV cache.
"""

from __future__ import annotations

import torch
import torch.nn.functional as F

from .arch import MoEArch


def rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps)
    return (y.to(x.dtype) * w)


class Rope:
    def __init__(self, arch: MoEArch, max_pos: int, device):
        hd = arch.head_dim
        inv = 1.0 / (arch.rope_theta ** (torch.arange(0, hd, 2, dtype=torch.float64,
                                                       device=device) / hd))
        t = torch.arange(max_pos, dtype=torch.float64, device=device)
        fr = torch.outer(t, inv)
        self.cos = fr.cos().float()
        self.sin = fr.sin().float()

    def apply(self, x: torch.Tensor, pos0: int) -> torch.Tensor:
        # x (B, S, H, hd), rotate-half convention
        S = x.shape[1]
        c = self.cos[pos0:pos0 + S][None, :, None, :]
        s = self.sin[pos0:pos0 + S][None, :, None, :]
        xf = x.float()
        h = xf.shape[-1] // 2
        x1, x2 = xf[..., :h], xf[..., h:]
        out = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], dim=-1)
        return out.to(x.dtype)


class KVCache:
    def __init__(self, arch: MoEArch, batch: int, max_len: int, device):
        shp = (arch.num_layers, batch, arch.num_kv_heads, max_len, arch.head_dim)
        self.k = torch.zeros(shp, dtype=torch.bfloat16, device=device)
        self.v = torch.zeros(shp, dtype=torch.bfloat16, device=device)
        self.len = 0


def attention(arch: MoEArch, x: torch.Tensor, wqkv: torch.Tensor, wo: torch.Tensor,
              rope: Rope, cache: KVCache, layer: int, B: int, S: int, pos0: int) -> torch.Tensor:
    """x (B*S, d) normalised input -> (B*S, d) attention output."""
    H, KV, hd = arch.num_heads, arch.num_kv_heads, arch.head_dim
    qkv = x @ wqkv.t()
    q = qkv[:, :H * hd].view(B, S, H, hd)
    k = qkv[:, H * hd:(H + KV) * hd].view(B, S, KV, hd)
    v = qkv[:, (H + KV) * hd:].view(B, S, KV, hd)
    q = rope.apply(q, pos0)
    k = rope.apply(k, pos0)
    cache.k[layer, :, :, pos0:pos0 + S] = k.transpose(1, 2)
    cache.v[layer, :, :, pos0:pos0 + S] = v.transpose(1, 2)
    kk = cache.k[layer, :, :, :pos0 + S]
    vv = cache.v[layer, :, :, :pos0 + S]
    o = F.scaled_dot_product_attention(q.transpose(1, 2), kk, vv, is_causal=(S > 1 and pos0 == 0),
                                       enable_gqa=(H != KV))
    o = o.transpose(1, 2).reshape(B * S, H * hd)
    return o @ wo.t()
