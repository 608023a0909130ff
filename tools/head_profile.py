"""CUPTI (torch.profiler) kernel table of offloaded decode steps at a real
model width with few layers (diagnostic for the per-layer device head).

    python tools/head_profile.py [--model mixtral-8x7b] [--layers 2] [--decode 8]
"""
import argparse
import dataclasses
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.cost_model import default_cost_model  # noqa: E402
from paper_2602_03495_b200.engine import (EngineConfig, ModelWeights, OffloadEngine,  # noqa: E402
                                          preset)

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mixtral-8x7b")
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--decode", type=int, default=8)
ap.add_argument("--out", default="gpurun_out/head_profile.txt")
args = ap.parse_args()

arch = dataclasses.replace(preset(args.model), num_layers=args.layers)
w = ModelWeights(arch, seed=0)
cm = default_cost_model(non_moe_layer_time=0.5)
import numpy as np  # noqa: E402
res = np.zeros((arch.num_layers - 1, arch.hidden_dim))
eng = OffloadEngine(arch, w, cm, EngineConfig(cache_slots_per_layer=2, prefetch_size=1),
                    residuals=res, max_seq=128)
p = torch.randint(0, arch.vocab_size, (1, 32))
eng.generate(p, args.decode)
eng.generate(p, args.decode)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    eng.generate(p, args.decode)
tab = prof.key_averages().table(sort_by="cuda_time_total", row_limit=40)
print(tab)
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    f.write(tab)
prof.export_chrome_trace(args.out.replace(".txt", ".json"))
