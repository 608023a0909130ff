"""A/B of the prefill-sized CPU expert: native AMX-BF16 (fp32 outputs) vs
torch oneDNN bf16 (the round-1 path), Mixtral-8x7B block, R tokens.

    python tools/cpu_prefill_ab.py [--R 16,32,64,128,256] [--threads N]
"""
import argparse
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--R", default="17,32,64,128,256")
ap.add_argument("--d", type=int, default=4096)
ap.add_argument("--f", type=int, default=14336)
ap.add_argument("--threads", type=int, default=len(os.sched_getaffinity(0)))
ap.add_argument("--blocks", type=int, default=4)
a = ap.parse_args()
d, f = a.d, a.f
torch.set_num_threads(a.threads)
blocks = [(torch.randn(3 * f * d) * 0.02).to(torch.bfloat16) for _ in range(a.blocks)]
print("amx available:", _lib.load().dali_cpu_expert_amx_available(), "threads", a.threads)


def onednn(block, x):
    n = x.shape[0]
    W13 = block[:2 * f * d].view(2 * f, d)
    W2 = block[2 * f * d:].view(d, f)
    gu = (x @ W13.t()).view(n, f // 64, 2, 64)
    g = gu[:, :, 0, :].reshape(n, f).float()
    u = gu[:, :, 1, :].reshape(n, f).float()
    act = (torch.nn.functional.silu(g) * u).to(torch.bfloat16)
    return (act @ W2.t()).float()


def native(block, x):
    y = torch.empty(x.shape[0], d)
    _lib.call("dali_cpu_expert", block.data_ptr(), d, f, x.data_ptr(), x.shape[0], y.data_ptr(),
              a.threads)
    return y


for R in [int(r) for r in a.R.split(",")]:
    x = torch.randn(R, d).to(torch.bfloat16)
    res = {}
    for name, fn in (("amx", native), ("onednn", onednn)):
        for b in blocks[:2]:
            fn(b, x)
        ts = []
        for i in range(3 * len(blocks)):
            t0 = time.perf_counter()
            fn(blocks[i % len(blocks)], x)
            ts.append((time.perf_counter() - t0) * 1e3)
        ts.sort()
        res[name] = ts[len(ts) // 2]
    fl = 6.0 * R * d * f
    print(f"R={R}: amx {res['amx']:.2f} ms ({fl / res['amx'] / 1e9:.2f} TF/s), onednn "
          f"{res['onednn']:.2f} ms ({fl / res['onednn'] / 1e9:.2f} TF/s)", flush=True)
