"""Phase timestamps of one fp64 fire (diagnostic; -DDALI_RG_PROF library,
tools/libdali_prof.so via DALI_LIB_PATH): the fire_cost.py near-tie router,
T = 1, CTA 0 (the cluster leader).  Marks: entry, ..., rank (7), cand list
(9), candidate logits reduced (10), fp64 done (8)."""
import ctypes as C
import os
import sys

os.environ.setdefault("DALI_LIB_PATH", os.path.join(os.path.dirname(__file__), "libdali_prof.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.trace import gate_norm2, route_device  # noqa: E402

lib = _lib.load()
d, N, k = (int(x) for x in sys.argv[1:4])
torch.manual_seed(0)
w = torch.randn(d, N) * 0.4 / d ** 0.5
w[:, 3] = w[:, 3].abs() + 1.0 / d ** 0.5
w = w.to(torch.bfloat16)
w[:, 4] = w[:, 3]
w[7, 4] = torch.tensor(w[7, 4].float().item() * (1 + 2 ** -7)).to(torch.bfloat16)
g = w.cuda()
n2 = gate_norm2(g)
names = {0: "entry", 1: "issued", 2: "landed", 3: "loop", 4: "reduce", 5: "pre-cl", 6: "post-cl",
         7: "rank", 9: "cand", 10: "logits64", 8: "fp64"}
for tie in (False, True):
    h = torch.randn(1, d).abs() + 0.01
    h[:, 7] = 2.0 ** -20 if tie else 64.0
    h = h.to(torch.bfloat16).cuda()
    for _ in range(5):
        route_device(h, g, k, norm2=n2)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * 96)()
    lib.dali_rg_prof(buf)
    row = list(buf[0:12])
    t0 = row[0]
    print("tie" if tie else "no tie", " ".join(f"{n}={(row[i] - t0) if row[i] >= t0 else '-'}"
                                              for i, n in names.items()))
