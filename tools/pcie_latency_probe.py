"""Latency of small GPU<->host transfers under expert DMA (diagnostic).

Measures, with CUDA events on a high-priority stream, the device time of the
per-layer control transfers of the offloaded decode:
  * read 136 B / 32 KB of pinned host memory by kernel (pointer table, CPU rows)
  * write 16 KB to pinned host memory by kernel (xp mirror)
while the PCIe H2D direction is (a) idle, (b) busy with a copy-engine expert
copy (cudaMemcpyAsync, 352 MB), (c) busy with an SM-driven copy of the same
block (dali_copy_h2d_sm) at 1..16 CTAs, reporting each bulk copy's GB/s.

    python tools/pcie_latency_probe.py
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.engine.weights import HostStore  # noqa: E402

torch.cuda.set_device(0)
BLOCK = 352 * 1024 * 1024
store = HostStore(BLOCK + (8 << 20), 16)
src = store.bytes
big_dev = torch.empty(BLOCK, dtype=torch.uint8, device="cuda")
small_h = torch.zeros(1 << 20, dtype=torch.uint8).pin_memory()
small_d = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
bulk = torch.cuda.Stream()
crit = torch.cuda.Stream(priority=-1)


gw = torch.randn(6144, 4096, device="cuda").to(torch.bfloat16)
gx = torch.randn(1, 4096, device="cuda").to(torch.bfloat16)
gy = torch.empty(1, 6144, device="cuda", dtype=torch.bfloat16)


def small_ops(n=40):
    res = {}
    ts = []
    for _ in range(n):                  # victim: the decode path's persistent GEMV
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(crit)
        for _ in range(4):
            _lib.call("dali_gemv_norm_bf16", gx.data_ptr(), gw.data_ptr(), 1, 6144, 4096,
                      gy.data_ptr(), None, 1e-5, None, None, None, None, None, crit.cuda_stream)
        e1.record(crit)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3 / 4)
    res["gemv"] = (float(np.median(ts)), float(np.percentile(ts, 90)))
    for name, (dst, s_, nb) in {
        "read136": (small_d.data_ptr(), small_h.data_ptr(), 144),
        "read32k": (small_d.data_ptr(), small_h.data_ptr(), 32768),
        "write16k": (small_h.data_ptr(), small_d.data_ptr(), 16384),
    }.items():
        ts = []
        for _ in range(n):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(crit)
            _lib.call("dali_copy_mapped", dst, s_, nb, crit.cuda_stream)
            e1.record(crit)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
            time.sleep(0.0002)
        res[name] = (float(np.median(ts)), float(np.percentile(ts, 90)))
    return res


def fmt(r):
    return "  ".join(f"{k} med {v[0]:6.1f} p90 {v[1]:6.1f} us" for k, v in r.items())


torch.cuda.synchronize()
print("idle:            ", fmt(small_ops()), flush=True)


def with_bulk(kind, nctas=0):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(bulk)
    for _ in range(6):
        if kind == "ce":
            with torch.cuda.stream(bulk):
                big_dev.copy_(src[:BLOCK], non_blocking=True)
        else:
            _lib.call("dali_copy_h2d_sm", big_dev.data_ptr(), src.data_ptr(), BLOCK, nctas,
                      bulk.cuda_stream)
    e1.record(bulk)
    time.sleep(0.003)
    r = small_ops(30)
    e1.synchronize()
    gbs = 6 * BLOCK / (e0.elapsed_time(e1) * 1e-3) / 1e9
    return r, gbs


r, gbs = with_bulk("ce")
print(f"copy engine      ({gbs:5.1f} GB/s): {fmt(r)}", flush=True)
for n, u in ((2, 4), (3, 4), (4, 4), (4, 2), (8, 2), (8, 1), (12, 1), (16, 1), (24, 1), (32, 1)):
    r, gbs = with_bulk("sm", n + 64 * (u - 1))
    print(f"sm copy {n:2d} CTAs x{u} ({gbs:5.1f} GB/s): {fmt(r)}", flush=True)
# bandwidth alone (no small ops)
for n in (2, 4, 8 + 64, 16):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(bulk)
    for _ in range(4):
        _lib.call("dali_copy_h2d_sm", big_dev.data_ptr(), src.data_ptr(), BLOCK, n,
                  bulk.cuda_stream)
    e1.record(bulk)
    e1.synchronize()
    print(f"sm copy {n:2d} CTAs alone: {4 * BLOCK / (e0.elapsed_time(e1) * 1e-3) / 1e9:5.1f} GB/s")
assert torch.equal(big_dev[:4096].cpu(), src[:4096])
