"""In-process A/B of an engine switch on the bench workload (diagnostic).

Builds the Mixtral-8x7B offloaded engine once (bench.py's settings: 24 GB
cache, residual prefetch P=1, teacher-forced Zipf decode) and alternates
requests between the two settings of an engine attribute, so host-speed
drift of the KVM guest hits both arms equally.  Prints decode tokens/s per
request and the per-arm medians.

    python tools/ab_inproc.py --attr _launch_ahead --a 0 --b 1 [--reps 6] [--decode 64]
"""
import argparse
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import zipf_tokens  # noqa: E402
from paper_2602_03495_b200.engine import EngineConfig, build_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mixtral-8x7b")
ap.add_argument("--attr", default="_launch_ahead")
ap.add_argument("--a", default="0")
ap.add_argument("--b", default="1")
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--prefill", type=int, default=512)
ap.add_argument("--decode", type=int, default=64)
args = ap.parse_args()
cores = len(os.sched_getaffinity(0))
cfg = EngineConfig(cache_gb=24.0, prefetch_size=1, w_size=4, seed=0, cpu_threads=cores)
eng = build_engine(args.model, cfg, seed=0, max_seq=args.prefill + args.decode + 8,
                   log=lambda *a: print(*a, file=sys.stderr))
V = eng.arch.vocab_size
prompt = torch.randint(0, V, (1, args.prefill), generator=torch.Generator().manual_seed(1000))
forced = zipf_tokens(V, (1, args.decode - 1), seed=3000)


def conv(v):
    return type(getattr(eng, args.attr))(int(v)) if v.isdigit() else v


res = {args.a: [], args.b: []}
eng.generate(prompt, 8, forced=forced[:, :7])                       # warm-up
for r in range(args.reps):
    for v in ((args.a, args.b) if r % 2 == 0 else (args.b, args.a)):
        setattr(eng, args.attr, conv(v))
        eng.reset_cache()
        toks, st = eng.generate(prompt, args.decode, forced=forced)
        tps = st.decode_tokens / st.decode_ms * 1e3
        res[v].append(tps)
        print(f"rep {r} {args.attr}={v}: decode {tps:.3f} tok/s", flush=True)
for v, xs in res.items():
    print(f"{args.attr}={v}: median {statistics.median(xs):.3f} tok/s  mean {statistics.mean(xs):.3f}"
          f"  ({', '.join(f'{x:.2f}' for x in xs)})")
