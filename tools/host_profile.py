"""cProfile of the host side of offloaded decode (diagnostic).

    python tools/host_profile.py [--model qwen1.5-moe-a2.7b] [--cache-gb 16]
"""
import argparse
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.engine import EngineConfig, build_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="qwen1.5-moe-a2.7b")
ap.add_argument("--cache-gb", type=float, default=16.0)
ap.add_argument("--prefill", type=int, default=128)
ap.add_argument("--decode", type=int, default=32)
args = ap.parse_args()
cfg = EngineConfig(cache_gb=args.cache_gb, prefetch_size=4, w_size=4, seed=0)
eng = build_engine(args.model, cfg, seed=0, max_seq=args.prefill + args.decode + 8)
p = torch.randint(0, eng.arch.vocab_size, (1, args.prefill))
eng.generate(p, args.decode)
pr = cProfile.Profile()
pr.enable()
toks, st = eng.generate(p, args.decode)
pr.disable()
print(f"decode {st.decode_tokens / st.decode_ms * 1e3:.1f} tok/s")
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
