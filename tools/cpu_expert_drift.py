"""Does the CPU expert cost drift after start-up?  (diagnostic)

Builds the Mixtral-8x7B host store, then times the native CPU expert (w=1)
over distinct layer-0 blocks every couple of seconds and prints the THP
state of the process (AnonHugePages) next to it.
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.engine import ModelWeights, preset  # noqa: E402
from paper_2602_03495_b200.engine.cpu_worker import cpu_expert_rows  # noqa: E402


def thp_kb():
    tot = 0
    with open("/proc/self/smaps_rollup") as f:
        for line in f:
            if line.startswith("AnonHugePages"):
                tot += int(line.split()[1])
    return tot


arch = preset("mixtral-8x7b")
cores = len(os.sched_getaffinity(0))
t0 = time.time()
w = ModelWeights(arch, seed=0)
print(f"store built in {time.time() - t0:.1f}s, THP {thp_kb() / 1e6:.1f} GB of "
      f"{w.host.nbytes / 1e9:.1f} GB", flush=True)
for p in ("/sys/kernel/mm/transparent_hugepage/enabled",
          "/sys/kernel/mm/transparent_hugepage/defrag"):
    try:
        print(p, open(p).read().strip())
    except OSError:
        pass
d, f = arch.hidden_dim, arch.ffn_dim
h = torch.randn(1, d).to(torch.bfloat16)
L, N = arch.num_layers, arch.num_experts
t_start = time.time()
if len(sys.argv) > 2 and sys.argv[2] == "continuous":
    # back-to-back calls over all blocks, stats per 250 ms window
    i, win, ts = 0, time.time(), []
    while time.time() - t_start < float(sys.argv[1]):
        blk = w.expert_host(i % L, (i // L) % N)
        t1 = time.perf_counter()
        cpu_expert_rows(blk, h, d, f, cores)
        ts.append((time.perf_counter() - t1) * 1e3)
        i += 1
        if time.time() - win > 0.25:
            print(f"t={time.time() - t_start:5.2f}s n {len(ts)} min {min(ts):.3f} "
                  f"med {np.median(ts):.3f} max {max(ts):.3f} ms", flush=True)
            win, ts = time.time(), []
    sys.exit(0)
for rnd in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
    for layer in (0, L // 2, L - 1):
        ts = []
        for i in range(16):
            blk = w.expert_host(layer, i % N)
            t1 = time.perf_counter()
            cpu_expert_rows(blk, h, d, f, cores)
            ts.append((time.perf_counter() - t1) * 1e3)
        print(f"t={time.time() - t_start:5.1f}s layer {layer:2d}: min {min(ts):.3f} "
              f"med {np.median(ts):.3f} ms  THP {thp_kb() / 1e6:.1f} GB", flush=True)
    time.sleep(2.0)
