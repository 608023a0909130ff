"""Decode attention alone (B=1, Mixtral GQA 32/8, hd 128, 16 splits): the
split-K kernel + merge, 50 back-to-back launches in a CUDA graph.

    python tools/prof_attn.py [--len 600] [--max-len 648]
"""
import argparse
import math
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--len", type=int, default=600)
ap.add_argument("--max-len", type=int, default=648)
a = ap.parse_args()
B, H, KV, hd, ML = 1, 32, 8, 128, a.max_len
bf = torch.bfloat16
q = torch.randn(B, H, hd, device="cuda").to(bf)
kc = torch.randn(B, KV, ML, hd, device="cuda").to(bf)
vc = torch.randn(B, KV, ML, hd, device="cuda").to(bf)
ln = torch.tensor([a.len], dtype=torch.int32, device="cuda")
out = torch.empty(B, H * hd, dtype=bf, device="cuda")
ws = torch.empty(B * H * 16 * (hd + 2), dtype=torch.float32, device="cuda")


def fn():
    _lib.call("dali_decode_attention", q.data_ptr(), kc.data_ptr(), vc.data_ptr(), ln.data_ptr(),
              B, H, KV, hd, ML, 16, 1 / math.sqrt(hd), ws.data_ptr(), out.data_ptr(),
              torch.cuda.current_stream().cuda_stream)


for _ in range(3):
    fn()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(50):
        fn()
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
g.replay()
e1.record()
e1.synchronize()
print(f"split-K attention + merge: {e0.elapsed_time(e1) * 1e3 / 50:.2f} us per call (len {a.len})")
