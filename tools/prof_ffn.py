"""Drive the grouped expert FFN kernels at Mixtral-8x7B shapes (for ncu).

    python tools/prof_ffn.py [--mode decode|prefill|both] [--iters N] [--kernel tc|simt]

decode : 2 GPU experts x 1 token (B=1 top-2), weights resident in HBM
prefill: 8 GPU experts x 128 tokens (512-token prompt, top-2)
Prints CUDA-event timings and achieved HBM GB/s (algorithmic bytes).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.engine.offload import ffn_splits  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mode", default="both", help="both | decode | prefill | one | all | decode-sweep | none")
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--kernel", default="tc", help="tc | simt")
ap.add_argument("--check", action="store_true", help="compare with an fp32 torch reference")
ap.add_argument("--kprof", action="store_true", help="per-kernel CUPTI durations")
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--f", type=int, default=14336)
ap.add_argument("--splits", type=int, default=0, help="override the split-K planes")
ap.add_argument("--counts", default=None, help="RxE: R tokens on each of E experts (e.g. 512x8)")
ap.add_argument("--n", type=int, default=8, help="experts (weight blocks allocated)")
ap.add_argument("--zipf", default=None,
                help="TxK: T tokens routed top-K over the n experts with a seeded skewed "
                     "distribution (DeepSeek-V2-Lite prefill: 4096x6 with --n 64)")
ap.add_argument("--count-list", default=None, help="explicit per-expert rows, comma-separated")
ap.add_argument("--graph", type=int, default=0,
                help="also replay N back-to-back launches captured in one CUDA graph")
args = ap.parse_args()
d, f, N = args.d, args.f, args.n
dev = torch.device("cuda")
blocks = torch.empty((N, 3 * f * d), dtype=torch.bfloat16, device=dev)
for e in range(N):
    _lib.call("dali_init_uniform_bf16", blocks[e].data_ptr(), blocks[e].numel(), 7 + e, 0,
              0.02, torch.cuda.current_stream().cuda_stream)
mp = np.zeros((N, 256), dtype=np.uint8)
for e in range(N):
    _lib.call("dali_expert_maps", blocks[e].data_ptr(), d, f, mp[e].ctypes.data)
maps_dev = torch.from_numpy(mp).to(dev)
nsm = torch.cuda.get_device_properties(dev).multi_processor_count
peak = 6552.3


def run(counts, label):
    rows = sum(counts)
    on = [c > 0 for c in counts]
    offs = torch.tensor(np.concatenate([[0], np.cumsum(counts)]), dtype=torch.int32, device=dev)
    maps = torch.tensor([maps_dev[e].data_ptr() if on[e] else 0 for e in range(N)],
                        dtype=torch.int64, device=dev)
    ptrs = torch.tensor([blocks[e].data_ptr() if on[e] else 0 for e in range(N)],
                        dtype=torch.int64, device=dev)
    xp = torch.randn(rows, d, device=dev).to(torch.bfloat16)
    h = torch.empty(rows, f, dtype=torch.bfloat16, device=dev)
    mr = max(counts)
    bn = 16 if mr <= 16 else 32 if mr <= 32 else 64 if mr <= 64 else 128 if mr <= 128 else 256
    tiles = sum((c + bn - 1) // bn for c in counts if c) * (d // 128)
    splits = args.splits or ffn_splits(mr, tiles, f // 64, nsm)
    y = torch.empty(splits, rows, d, dtype=torch.float32, device=dev)
    cs0 = torch.cuda.current_stream().cuda_stream  # noqa: F841

    def go():
        cs = torch.cuda.current_stream().cuda_stream
        if args.kernel == "tc":
            _lib.call("dali_expert_ffn_tc", xp.data_ptr(), offs.data_ptr(), N, maps.data_ptr(), d,
                      f, rows, mr, sum(on), h.data_ptr(), y.data_ptr(), splits, cs)
        else:
            _lib.call("dali_expert_ffn", xp.data_ptr(), offs.data_ptr(), N, ptrs.data_ptr(), d, f,
                      rows, mr, h.data_ptr(), y.data_ptr(), cs)
    for _ in range(3):
        go()
    torch.cuda.synchronize()
    if args.check:                      # vs an fp32 torch reference of the same FFN
        ysum = y.sum(0)
        err = 0.0
        for e in range(N):
            if not on[e]:
                continue
            r0, r1 = int(offs[e]), int(offs[e + 1])
            blk = blocks[e].float()
            w13 = blk[:2 * f * d].view(2 * f, d)
            idx = torch.arange(2 * f, device=dev).view(-1, 128)
            g_rows, u_rows = idx[:, :64].reshape(-1), idx[:, 64:].reshape(-1)
            x = xp[r0:r1].float()
            gg, uu = x @ w13[g_rows].t(), x @ w13[u_rows].t()
            hh = (torch.nn.functional.silu(gg) * uu).to(torch.bfloat16).float()
            ref = hh @ blk[2 * f * d:].view(d, f).t()
            err = max(err, float((ysum[r0:r1] - ref).abs().max() / ref.abs().max()))
        print(f"{label}: max |err| / max |ref| vs fp32 reference {err:.2e}", flush=True)
    ts = []
    for _ in range(args.iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        go()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    if args.kprof:                      # per-kernel device durations (CUPTI)
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(10):
                go()
            torch.cuda.synchronize()
        for ev in prof.key_averages():
            if ev.device_type.name == "CUDA" and ev.count >= 10:
                print(f"    {ev.key[:60]:60s} n={ev.count} avg {ev.device_time:.1f} us")
    if args.graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(args.graph):
                go()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        e1.synchronize()
        print(f"{label}: graph of {args.graph} launches: {e0.elapsed_time(e1) * 1e3 / args.graph:.1f}"
              f" us per launch", flush=True)
    byts = sum(on) * 3 * f * d * 2 + rows * (d * 2 + 2 * f * 2 + d * 4 * splits)
    flops = 6.0 * rows * d * f
    print(f"{label}: {args.kernel} splits={splits} bn={bn} median {ms * 1e3:.1f} us, "
          f"{byts / ms / 1e6:.0f} GB/s ({byts / ms / 1e6 / peak:.3f} of {peak}), "
          f"{flops / ms / 1e9:.1f} TFLOP/s, bytes {byts}")


if args.zipf:
    T_, K_ = (int(x) for x in args.zipf.split("x"))
    rng = np.random.default_rng(5)
    pr = 1.0 / np.arange(1, N + 1) ** 0.6
    pr = rng.permutation(pr / pr.sum())
    cnt = np.zeros(N, dtype=np.int64)
    for _ in range(T_):
        cnt[rng.choice(N, size=K_, replace=False, p=pr)] += 1
    run(cnt.tolist(), f"zipf {args.zipf} (max {cnt.max()}, min {cnt.min()})")
if args.counts:
    r_, e_ = (int(x) for x in args.counts.split("x"))
    run([r_] * e_ + [0] * (N - e_), f"counts {args.counts}")
if args.count_list:
    run([int(x) for x in args.count_list.split(",")], f"count list {args.count_list}")
if args.mode == "one":
    run([1, 0, 0, 0, 0, 0, 0, 0], "decode 1x1")
if args.mode in ("decode", "both"):
    run([1, 0, 0, 1, 0, 0, 0, 0], "decode 2x1")
if args.mode in ("prefill", "both"):
    run([128] * 8, "prefill 8x128")
if args.mode == "decode-sweep":
    for c in ([1] + [0] * 7, [1, 1] + [0] * 6, [2, 2] + [0] * 6, [2, 1] + [0] * 6, [1] * 8,
              [2] * 8, [1, 2, 0, 0, 2, 0, 0, 0]):
        run(c, f"counts {max(c)}x{sum(1 for x in c if x)}")
if args.mode == "all":
    for c in ([1, 0, 0, 0, 0, 0, 0, 0], [1, 1, 0, 0, 0, 0, 0, 0], [2, 1, 0, 0, 0, 0, 0, 0],
              [4] * 8, [16] * 8, [64] * 8, [128] * 8, [256] * 8, [512] * 8):
        run(c, f"counts {c[0]}x{sum(1 for x in c if x)}")
