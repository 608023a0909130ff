"""Can the GPU add host-DRAM bandwidth to the CPU experts?  (diagnostic)

Measures, on the Mixtral host store: zero-copy reads by SM loads
(dali_copy_mapped host->device), copy-engine H2D DMA, and the native CPU
expert (w=1) -- each alone, then CPU expert + zero-copy and CPU expert + DMA
concurrently (the CPU loop runs in a thread; ctypes drops the GIL)."""
import os
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.engine import ModelWeights, preset  # noqa: E402
from paper_2602_03495_b200.engine.cpu_worker import cpu_expert_rows  # noqa: E402

arch = preset("mixtral-8x7b")
cores = len(os.sched_getaffinity(0))
w = ModelWeights(arch, seed=0)
d, f, L, N = arch.hidden_dim, arch.ffn_dim, arch.num_layers, arch.num_experts
eb = w.expert_bytes
dev_buf = torch.empty((eb,), dtype=torch.uint8, device="cuda")
h1 = torch.randn(1, d).to(torch.bfloat16)
st = torch.cuda.Stream()


def cpu_loop(secs, out, threads=cores):
    t_end, n, i = time.perf_counter() + secs, 0, 0
    t0 = time.perf_counter()
    while time.perf_counter() < t_end:
        cpu_expert_rows(w.expert_host(i % L, 1 + (i // L) % (N - 1)), h1, d, f, threads)
        n += 1
        i += 1
    out.append((time.perf_counter() - t0) / n * 1e3)


def gpu_loop(secs, kind, out):
    t_end, nbytes = time.perf_counter() + secs, 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    i = 0
    while time.perf_counter() < t_end:
        src = w.expert_host(i % L, 0)
        if kind == "zero_copy":
            _lib.call("dali_copy_mapped", dev_buf.data_ptr(), src.data_ptr(), eb, st.cuda_stream)
        else:
            with torch.cuda.stream(st):
                dev_buf.copy_(src.view(torch.uint8).view(-1), non_blocking=True)
        nbytes += eb
        i += 1
        st.synchronize()
    e1.record(st)
    e1.synchronize()
    out.append(nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)


cpu_loop(1.0, [])                       # warm-up
for rnd in range(2):
    r = []
    cpu_loop(1.5, r)
    print(f"cpu expert alone: {r[0]:.3f} ms ({eb / r[0] / 1e6:.0f} GB/s)", flush=True)
    for kind in ("zero_copy", "dma"):
        g = []
        gpu_loop(1.0, kind, g)
        print(f"{kind} alone: {g[0]:.1f} GB/s", flush=True)
        r, g = [], []
        th = threading.Thread(target=cpu_loop, args=(1.5, r))
        th.start()
        gpu_loop(1.5, kind, g)
        th.join()
        cg = eb / r[0] / 1e6
        print(f"cpu + {kind}: cpu {r[0]:.3f} ms ({cg:.0f} GB/s) + gpu {g[0]:.1f} GB/s = "
              f"{cg + g[0]:.0f} GB/s", flush=True)
