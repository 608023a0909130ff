"""Critical-path breakdown of a decode step (diagnostic).

Runs decode steps of the engine under the CUDA profiler (CUPTI activity
records: kernel start / end on the device clock) and attributes the step's
device time to kernels along the launching stream: kernel k's share is
end(k) - max(end(k-1), start(k)) plus the idle gap before it.  With PDL a
kernel "starts" early and waits, so only end-to-end deltas are meaningful.

    python tools/critical_path.py [--model mixtral-8x7b] [--resident] [--decode 16]
"""
import argparse
import collections
import json
import os
import re
import sys
import tempfile

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.cost_model import default_cost_model  # noqa: E402
from paper_2602_03495_b200.engine import EngineConfig, build_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mixtral-8x7b")
ap.add_argument("--decode", type=int, default=16)
ap.add_argument("--prompt", type=int, default=512)
ap.add_argument("--out", default="gpurun_out/critical_path.txt")
args = ap.parse_args()
eng = build_engine(args.model, EngineConfig(), resident=True, max_seq=args.prompt + args.decode + 8,
                   cost_model=default_cost_model())
p = torch.randint(0, eng.arch.vocab_size, (1, args.prompt))
for _ in range(2):
    toks, st = eng.generate(p.cuda(), args.decode, host_io=False)
print(f"decode {st.decode_tokens / st.decode_ms * 1e3:.1f} tok/s", flush=True)
from torch.profiler import ProfilerActivity, profile  # noqa: E402
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    toks, st = eng.generate(p.cuda(), args.decode, host_io=False)
tr = os.path.join(tempfile.mkdtemp(), "trace.json")
prof.export_chrome_trace(tr)
ev = [e for e in json.load(open(tr))["traceEvents"]
      if e.get("ph") == "X" and e.get("cat") == "kernel"]
by_stream = collections.defaultdict(list)
for e in ev:
    by_stream[e["args"].get("stream", 0)].append(e)
main = max(by_stream.values(), key=len)
main.sort(key=lambda e: e["ts"])
# the decode steps: after the (long) prefill, i.e. the last decode-1 graph replays;
# take the last 70% of the main-stream kernels
main = main[int(len(main) * 0.3):]
share = collections.defaultdict(float)
count = collections.Counter()
prev_end = main[0]["ts"] + main[0]["dur"]
for e in main[1:]:
    s, end = e["ts"], e["ts"] + e["dur"]
    name = re.sub(r"\(.*", "", e["name"]).replace("void ", "")[:60]
    share[name] += max(0.0, end - max(prev_end, s)) + max(0.0, s - prev_end)
    count[name] += 1
    prev_end = max(prev_end, end)
tot = sum(share.values())
lines = [f"critical path over {len(main)} main-stream kernels, {tot:.0f} us "
         f"({args.model}, resident, decode {st.decode_tokens / st.decode_ms * 1e3:.1f} tok/s)"]
for name, v in sorted(share.items(), key=lambda x: -x[1]):
    lines.append(f"{name:60s} n={count[name]:5d} total={v:9.1f} us  per_launch={v / count[name]:7.2f} us"
                 f"  share={v / tot:.3f}")
print("\n".join(lines))
os.makedirs(os.path.dirname(args.out), exist_ok=True)
open(args.out, "w").write("\n".join(lines) + "\n")
