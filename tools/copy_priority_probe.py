"""Does a demand copy wait behind queued replacement DMA?  (diagnostic)

Queues N expert-sized H2D copies on a 'replacement' stream, then issues one
'demand' copy of the same size and measures its latency from issue to
completion: on a second normal stream, on a high-priority stream, and as a
kernel copy over UVA-mapped pinned memory (dali_copy_mapped, no copy engine).
"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.engine.weights import HostStore  # noqa: E402

mb = float(sys.argv[1]) if len(sys.argv) > 1 else 17.3
n_backlog = int(sys.argv[2]) if len(sys.argv) > 2 else 16
nbytes = int(mb * 1e6) // 16 * 16
store = HostStore(nbytes * (n_backlog + 1), 16)
src = store.bytes
dev = torch.empty((n_backlog + 1, nbytes), dtype=torch.uint8, device="cuda")
repl = torch.cuda.Stream()
lo, hi = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") \
    else (0, -1)
normal = torch.cuda.Stream()
high = torch.cuda.Stream(priority=-1)
comp = torch.cuda.Stream()


def trial(kind):
    torch.cuda.synchronize()
    with torch.cuda.stream(repl):
        for i in range(n_backlog):
            dev[i].copy_(src[i * nbytes:(i + 1) * nbytes], non_blocking=True)
    time.sleep(0.0005)
    s = {"normal": normal, "high": high, "kernel": comp}[kind]
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    if kind == "kernel":
        _lib.call("dali_copy_mapped", dev[n_backlog].data_ptr(),
                  src[n_backlog * nbytes:].data_ptr(), nbytes, s.cuda_stream)
    else:
        with torch.cuda.stream(s):
            dev[n_backlog].copy_(src[n_backlog * nbytes:(n_backlog + 1) * nbytes],
                                 non_blocking=True)
    e1.record(s)
    e1.synchronize()
    t = e0.elapsed_time(e1)
    torch.cuda.synchronize()
    return t


alone = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(normal)
    with torch.cuda.stream(normal):
        dev[0].copy_(src[:nbytes], non_blocking=True)
    e1.record(normal)
    e1.synchronize()
    alone.append(e0.elapsed_time(e1))
print(f"block {mb} MB, backlog {n_backlog} copies; demand copy alone {min(alone):.3f} ms")
for kind in ("normal", "high", "kernel", "normal", "high", "kernel"):
    print(f"  demand copy behind backlog, {kind:6s}: {trial(kind):.3f} ms", flush=True)
