"""Decode GEMV (dali_gemv_bf16) alone: achieved HBM bandwidth at the
attention-projection shapes, rotating over weight copies larger than L2."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402

dev = torch.device("cuda")
for (M, K) in [(6144, 4096), (4096, 4096), (10240, 6144)]:
    n_copy = max(2, int(400e6 // (M * K * 2)))
    ws = [torch.randn(M, K, device=dev).to(torch.bfloat16) for _ in range(n_copy)]
    x = torch.randn(1, K, device=dev).to(torch.bfloat16)
    y = torch.empty(1, M, dtype=torch.bfloat16, device=dev)
    cs = torch.cuda.current_stream().cuda_stream
    for i in range(6):
        _lib.call("dali_gemv_bf16", x.data_ptr(), ws[i % n_copy].data_ptr(), 1, M, K,
                  y.data_ptr(), cs)
    ts = []
    for _ in range(5):                      # 20 back-to-back launches per sample
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(20):
            _lib.call("dali_gemv_bf16", x.data_ptr(), ws[i % n_copy].data_ptr(), 1, M, K,
                      y.data_ptr(), cs)
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 20)
    ms = float(np.median(ts))
    print(f"gemv M={M} K={K}: {ms * 1e3:.1f} us, {M * K * 2 / ms / 1e6:.0f} GB/s")
