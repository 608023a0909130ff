"""Stress test of the launch-ahead offloaded decode (diagnostic).

Runs many short requests of varying prompt length through a tiny engine
(cache + prefetch on) and checks after each that the residual stream is
finite and that no launched-ahead combine timed out waiting for its CPU
rows (dali_host_wait_timeouts).  Round 2 found with it that ld.volatile
polls of mapped pinned memory could be served a stale GPU-L2 line for
seconds; host-memory reads on the decode path now use ld.global.cv.

    python tools/stress_launch_ahead.py [tiny|tiny-shared] [iterations]
"""
import ctypes
import faulthandler
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.cost_model import default_cost_model  # noqa: E402
from paper_2602_03495_b200.engine import EngineConfig, build_engine  # noqa: E402

faulthandler.enable()
name = sys.argv[1] if len(sys.argv) > 1 else "tiny-shared"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = EngineConfig(cache_slots_per_layer=2 if name == "tiny" else 6, prefetch_size=2,
                   capture=True, seed=3)
cm = default_cost_model(shared_expert_gpu_time=0.0 if name == "tiny" else 0.5,
                        non_moe_layer_time=3.0)
eng = build_engine(name, cfg, seed=5, cost_model=cm, max_seq=128)
g = torch.Generator().manual_seed(0)
tmo = ctypes.c_uint64()
for it in range(iters):
    p = torch.randint(0, eng.arch.vocab_size, (1, 16 + it % 7), generator=g)
    toks, st = eng.generate(p, 24)
    torch.cuda.synchronize()
    _lib.call("dali_host_wait_timeouts", ctypes.byref(tmo), 0)
    x = eng._wsd.get(("dec_X", torch.bfloat16, False))
    finite = bool(torch.isfinite(x).all()) if x is not None else True
    if tmo.value or not finite:
        sys.exit(f"iteration {it}: {tmo.value} poll timeouts, residual finite={finite}")
print(f"{name}: {iters} requests ok, 0 poll timeouts")
