"""Device-side chain of one offloaded decode layer (diagnostic).

Profiles a few teacher-forced decode tokens of the offloaded engine (CUPTI
kernel + memcpy records via torch.profiler) and prints, per kernel name on
the compute stream, the mean duration and the mean idle gap before it --
i.e. where the ~0.1 ms between "CPU rows ready" and "next decision visible"
goes.  Also lists the host-side ranges the profiler saw.

    python tools/offload_chain.py [--model mixtral-8x7b] [--cache-gb 24] [--decode 12]
"""
import argparse
import collections
import json
import os
import re
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.engine import EngineConfig, build_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mixtral-8x7b")
ap.add_argument("--cache-gb", type=float, default=24.0)
ap.add_argument("--prefill", type=int, default=128)
ap.add_argument("--decode", type=int, default=12)
ap.add_argument("--out", default="gpurun_out/offload_chain.txt")
args = ap.parse_args()
cores = len(os.sched_getaffinity(0))
cfg = EngineConfig(cache_gb=args.cache_gb, prefetch_size=1, w_size=4, seed=0, cpu_threads=cores)
eng = build_engine(args.model, cfg, seed=0, max_seq=args.prefill + args.decode + 8,
                   log=lambda *a: print(*a, file=sys.stderr))
from bench import zipf_tokens  # noqa: E402
V = eng.arch.vocab_size
g = torch.Generator().manual_seed(1000)
p = torch.randint(0, V, (1, args.prefill), generator=g)
forced = zipf_tokens(V, (1, args.decode - 1), seed=3000)
for _ in range(2):
    toks, st = eng.generate(p, args.decode, host_io=True, forced=forced)
print(f"decode {st.decode_tokens / st.decode_ms * 1e3:.2f} tok/s", flush=True)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    toks, st = eng.generate(p, args.decode, host_io=True, forced=forced)
tr = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(tr)
ev = [e for e in json.load(open(tr))["traceEvents"] if e.get("ph") == "X" and
      e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
by_stream = collections.defaultdict(list)
for e in ev:
    by_stream[e["args"].get("stream", 0)].append(e)
lines = []
for sid, es in sorted(by_stream.items(), key=lambda x: -len(x[1])):
    es.sort(key=lambda e: e["ts"])
    lines.append(f"stream {sid}: {len(es)} records")
main = max(by_stream.values(), key=len)
main.sort(key=lambda e: e["ts"])
main = main[int(len(main) * 0.4):]              # decode part
dur = collections.defaultdict(list)
gap = collections.defaultdict(list)
prev_end = None
for e in main:
    name = re.sub(r"\(.*", "", e["name"]).replace("void ", "")[:70]
    dur[name].append(e["dur"])
    if prev_end is not None:
        gap[name].append(max(0.0, e["ts"] - prev_end))
    prev_end = e["ts"] + e["dur"] if prev_end is None else max(prev_end, e["ts"] + e["dur"])
lines.append(f"compute stream, last 60% of records ({len(main)}), decode {args.decode} tokens:")
for name in sorted(dur, key=lambda n: -sum(dur[n]) - sum(gap[n])):
    lines.append(f"  {name:70s} n={len(dur[name]):5d} dur={np.mean(dur[name]):8.2f} us "
                 f"gap_before={np.mean(gap[name]) if gap[name] else 0:8.2f} us "
                 f"(median {np.median(gap[name]) if gap[name] else 0:7.2f})")
# one representative layer sequence
lines.append("sample sequence (ts relative, us):")
t0 = main[len(main) // 2]["ts"]
for e in main[len(main) // 2: len(main) // 2 + 40]:
    name = re.sub(r"\(.*", "", e["name"]).replace("void ", "")[:60]
    lines.append(f"  {e['ts'] - t0:9.1f} +{e['dur']:7.1f}  {name}")
print("\n".join(lines))
os.makedirs(os.path.dirname(args.out), exist_ok=True)
open(args.out, "w").write("\n".join(lines) + "\n")
