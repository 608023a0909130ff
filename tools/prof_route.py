"""Time the routing kernel at decode / prefill shapes (diagnostic, ncu target).

    python tools/prof_route.py [--d 4096] [--N 8] [--k 2]
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
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--T", type=str, default="1,4,16,128,512,4096")
ap.add_argument("--prefill-variant", type=int, default=0,
                help="T > 16: 0 by shape, 1 d-chunked kernel, 2 fixed-geometry kernel")
ap.add_argument("--force", action="store_true", help="every row through the fp64 recompute")
ap.add_argument("--scale", type=float, default=1.0,
                help="bound scale (diagnostic: << 1 suppresses fires to time the fire-free kernel)")
args = ap.parse_args()
_lib.call("dali_route_prefill_variant", args.prefill_variant)
_lib.call("dali_route_guard_scale", -1.0 if args.force else args.scale)
torch.manual_seed(0)
g = (torch.randn(args.d, args.N, device="cuda") * 0.02).to(torch.bfloat16)
n2 = gate_norm2(g)             # the engine computes router norms once
for T in [int(x) for x in args.T.split(",")]:
    h = torch.randn(T, args.d, device="cuda").to(torch.bfloat16)
    for _ in range(3):
        route_device(h, g, args.k)
    torch.cuda.synchronize()
    out = (torch.empty((T, args.k), dtype=torch.int32, device="cuda"),
           torch.empty((T, args.k), dtype=torch.float32, device="cuda"),
           torch.empty((args.N,), dtype=torch.int64, device="cuda"))
    graph = torch.cuda.CUDAGraph()            # device time without host launch cost
    with torch.cuda.graph(graph):
        for _ in range(args.iters):
            route_device(h, g, args.k, out=out, norm2=n2)
    graph.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    graph.replay()
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / args.iters
    _lib.route_fire_count(reset=True)
    route_device(h, g, args.k, out=out, norm2=n2)
    fires, rows = _lib.route_fire_count(reset=True)
    byts = T * args.d * 2 + args.d * args.N * 2 + T * args.k * 8 + args.N * 8
    print(f"T={T}: {us:.1f} us per call ({byts / us / 1e3:.1f} GB/s algorithmic, "
          f"fires {fires}/{rows})")
