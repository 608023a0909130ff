"""Probe host memory bandwidth and CPU expert GEMV speed on the GPU box."""
import os, time, torch
torch.set_num_threads(len(os.sched_getaffinity(0)))
a = torch.empty(1 << 30, dtype=torch.uint8); a.fill_(1)
b = torch.empty_like(a)
for _ in range(3):
    t = time.perf_counter(); b.copy_(a); el = time.perf_counter() - t
    print("copy 1GiB GB/s (r+w)", 2 * a.numel() / el / 1e9)
x = a.view(torch.float32)
for _ in range(3):
    t = time.perf_counter(); s = x.sum(); el = time.perf_counter() - t
    print("sum 1GiB GB/s", a.numel() / el / 1e9)
W = torch.randn(28672, 4096).to(torch.bfloat16)
for R in (1, 2, 4, 8):
    h = torch.randn(R, 4096).to(torch.bfloat16)
    ts = []
    for _ in range(5):
        t = time.perf_counter(); y = h @ W.t(); ts.append(time.perf_counter() - t)
    print("bf16 gemm R", R, "ms", min(ts) * 1e3, "GB/s", W.numel() * 2 / min(ts) / 1e9)
