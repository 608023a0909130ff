"""Fused decode attention (csrc/attn.cu decode_attn_fused_kernel) against the
three-launch path it replaces (dali_rope_append + dali_decode_attention):
bit-identical attention output and caches, for GQA and MHA, head_dim 64 and
128, positions inside and at the edge of a split, and repeated launches (the
merge counters must come back to zero)."""

import math

import pytest
import torch

from paper_2602_03495_b200 import _lib

pytestmark = pytest.mark.gpu


def _case(B, H, KV, hd, max_len, pos, splits=16, reps=2, seed=0):
    dev = torch.device("cuda")
    g = torch.Generator(device=dev).manual_seed(seed)
    qkv = (torch.randn(B, (H + 2 * KV) * hd, device=dev, generator=g) * 0.5).to(torch.bfloat16)
    half = hd // 2
    inv = 1.0 / (10000 ** (torch.arange(half, device=dev, dtype=torch.float32) / half))
    ang = torch.arange(max_len, device=dev, dtype=torch.float32)[:, None] * inv[None]
    cos, sin = ang.cos().contiguous(), ang.sin().contiguous()
    kc0 = (torch.randn(B, KV, max_len, hd, device=dev, generator=g) * 0.5).to(torch.bfloat16)
    vc0 = (torch.randn(B, KV, max_len, hd, device=dev, generator=g) * 0.5).to(torch.bfloat16)
    desc = torch.tensor([pos, pos + 1], dtype=torch.int32, device=dev)
    scale = 1.0 / math.sqrt(hd)
    st = torch.cuda.current_stream().cuda_stream
    ws = torch.empty(B * H * splits * (hd + 2), dtype=torch.float32, device=dev)
    # reference: three launches
    kc1, vc1 = kc0.clone(), vc0.clone()
    q = torch.empty(B, H, hd, dtype=torch.bfloat16, device=dev)
    o1 = torch.empty(B, H * hd, dtype=torch.bfloat16, device=dev)
    _lib.call("dali_rope_append", qkv.data_ptr(), cos.data_ptr(), sin.data_ptr(),
              desc.data_ptr(), B, H, KV, hd, max_len, q.data_ptr(), kc1.data_ptr(),
              vc1.data_ptr(), st)
    _lib.call("dali_decode_attention", q.data_ptr(), kc1.data_ptr(), vc1.data_ptr(),
              desc.data_ptr() + 4, B, H, KV, hd, max_len, splits, scale, ws.data_ptr(),
              o1.data_ptr(), st)
    # fused, launched `reps` times (counters reset by the merging CTA)
    ctr = torch.zeros(B * H, dtype=torch.int32, device=dev)
    for _ in range(reps):
        kc2, vc2 = kc0.clone(), vc0.clone()
        o2 = torch.full((B, H * hd), 7.0, dtype=torch.bfloat16, device=dev)
        _lib.call("dali_decode_attention_fused", qkv.data_ptr(), cos.data_ptr(), sin.data_ptr(),
                  desc.data_ptr(), desc.data_ptr() + 4, B, H, KV, hd, max_len, splits, scale,
                  kc2.data_ptr(), vc2.data_ptr(), ws.data_ptr(), ctr.data_ptr(), o2.data_ptr(), st)
        torch.cuda.synchronize()
        assert torch.equal(o1.view(torch.int16), o2.view(torch.int16))
        assert torch.equal(kc1[:, :, :pos + 1].view(torch.int16), kc2[:, :, :pos + 1].view(torch.int16))
        assert torch.equal(vc1[:, :, :pos + 1].view(torch.int16), vc2[:, :, :pos + 1].view(torch.int16))
        assert int(ctr.abs().sum()) == 0


@pytest.mark.parametrize("B,H,KV,hd,pos", [(1, 32, 8, 128, 517), (2, 32, 8, 128, 0),
                                            (1, 16, 16, 128, 63), (3, 16, 4, 64, 200),
                                            (1, 32, 8, 128, 15)])
def test_fused_attention_bit_identical(B, H, KV, hd, pos):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    _case(B, H, KV, hd, 1024, pos)
