"""Cost of fp64 fires in the certified routing kernels (diagnostic).

Router experts 3 and 4 are identical except one weight (row 7) nudged by a
bf16 ulp, and dominate every token.  A token with a tiny element 7 is a
near-tie the fp32 certificate cannot separate (a fire with 2 candidates); a
token with element 7 = 64 separates them by far more than the bound.  Prints
us per call (50-call CUDA graph) with 0 fires and with the first `--ties`
rows firing.

    python tools/fire_cost.py [--d 4096] [--N 8] [--k 2] [--T 1,4096] [--ties 1]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.trace import gate_norm2, route_device  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--N", type=int, default=8)
ap.add_argument("--k", type=int, default=2)
ap.add_argument("--T", type=str, default="1,4096")
ap.add_argument("--ties", type=int, default=1)
ap.add_argument("--iters", type=int, default=50)
args = ap.parse_args()
torch.manual_seed(0)
d, N, k = args.d, args.N, args.k


def timed(h, g):
    n2 = gate_norm2(g)
    T = h.shape[0]
    out = (torch.empty((T, k), dtype=torch.int32, device="cuda"),
           torch.empty((T, k), dtype=torch.float32, device="cuda"),
           torch.empty((N,), dtype=torch.int64, device="cuda"))
    for _ in range(3):
        route_device(h, g, k, out=out, norm2=n2)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        for _ in range(args.iters):
            route_device(h, g, k, out=out, norm2=n2)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    e1.synchronize()
    _lib.route_fire_count(reset=True)
    route_device(h, g, k, out=out, norm2=n2)
    fires, rows = _lib.route_fire_count(reset=True)
    return e0.elapsed_time(e1) * 1e3 / args.iters, fires


w = torch.randn(d, N) * 0.4 / d ** 0.5
w[:, 3] = w[:, 3].abs() + 1.0 / d ** 0.5          # experts 3 and 4 lead for positive rows
w = w.to(torch.bfloat16)
w[:, 4] = w[:, 3]
w[7, 4] = torch.tensor(w[7, 4].float().item() * (1 + 2 ** -7)).to(torch.bfloat16)
wd = w.cuda()
for T in [int(x) for x in args.T.split(",")]:
    h = torch.randn(T, d).abs() + 0.01
    h[:, 7] = 64.0                                 # separated: no fire
    t0, f0 = timed(h.to(torch.bfloat16).cuda(), wd)
    h[:min(args.ties, T), 7] = 2.0 ** -20          # near-tie rows: fires
    t1, f1 = timed(h.to(torch.bfloat16).cuda(), wd)
    print(f"T={T}: {t0:.1f} us ({f0} fires) | {t1:.1f} us ({f1} fires)", flush=True)
