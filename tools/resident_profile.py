"""CUPTI kernel table of the all-resident decode (CUDA-graph replay) at the
full Mixtral-8x7B shape (diagnostic for the roofline-reference mode).

    python tools/resident_profile.py [--decode 32]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.cost_model import default_cost_model  # noqa: E402
from paper_2602_03495_b200.engine import EngineConfig, build_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mixtral-8x7b")
ap.add_argument("--decode", type=int, default=32)
ap.add_argument("--out", default="gpurun_out/resident_profile.txt")
args = ap.parse_args()
eng = build_engine(args.model, EngineConfig(), resident=True, max_seq=256,
                   cost_model=default_cost_model())
p = torch.randint(0, eng.arch.vocab_size, (1, 64))
for _ in range(2):
    toks, st = eng.generate(p.cuda(), args.decode, host_io=False)
    print(f"decode {st.decode_tokens / st.decode_ms * 1e3:.1f} tok/s", flush=True)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    toks, st = eng.generate(p.cuda(), args.decode, host_io=False)
print(f"profiled: decode {st.decode_tokens / st.decode_ms * 1e3:.1f} tok/s")
tab = prof.key_averages().table(sort_by="cuda_time_total", row_limit=30)
print(tab)
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    f.write(tab)
