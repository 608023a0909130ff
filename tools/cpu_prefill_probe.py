"""Why do prefill-sized CPU experts run 2x slower inside the engine than in
the profile?  (diagnostic)  Times the oneDNN expert path (w rows) after a
sustained warm-up: alone, with H2D expert copies in flight, and right after a
native (decode-path) call whose pool threads are still spinning."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.engine import ModelWeights, preset  # noqa: E402
from paper_2602_03495_b200.engine.cpu_worker import cpu_expert_rows  # noqa: E402

arch = preset("mixtral-8x7b")
cores = len(os.sched_getaffinity(0))
torch.set_num_threads(cores)
w = ModelWeights(arch, seed=0)
d, f, L, N = arch.hidden_dim, arch.ffn_dim, arch.num_layers, arch.num_experts
eb = w.expert_bytes
dev = torch.device("cuda")
dst = torch.empty((eb,), dtype=torch.uint8, device=dev)
side = torch.cuda.Stream()
h1 = torch.randn(1, d).to(torch.bfloat16)
t_end, i = time.perf_counter() + 1.0, 0
while time.perf_counter() < t_end:
    cpu_expert_rows(w.expert_host(i % L, 0), h1, d, f, cores)
    i += 1
rows = int(sys.argv[1]) if len(sys.argv) > 1 else 128
x = torch.randn(rows, d).to(torch.bfloat16)


def blk(i):
    return w.expert_host((i * 7) % L, (i * 3) % N)


def timed(mode, n=12):
    ts = []
    for j in range(n):
        if mode == "dma":
            with torch.cuda.stream(side):
                for q in range(4):
                    dst.copy_(w.host.bytes[eb * (10 + q): eb * (11 + q)], non_blocking=True)
            time.sleep(0.0005)
        if mode == "after_native":
            cpu_expert_rows(blk(j + 100), h1, d, f, cores)
        t0 = time.perf_counter()
        cpu_expert_rows(blk(j), x, d, f, cores)
        ts.append((time.perf_counter() - t0) * 1e3)
        if mode == "dma":
            side.synchronize()
    return f"{mode:13s} rows {rows}: min {min(ts):.2f} med {np.median(ts):.2f} max {max(ts):.2f} ms"


for mode in ("alone", "dma", "after_native", "alone", "dma", "after_native"):
    print(timed(mode), flush=True)
