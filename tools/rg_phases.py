"""Phase timestamps (globaltimer, ns) of the certified routing kernel, from a
-DDALI_RG_PROF build (tools/libdali_prof.so via DALI_LIB_PATH): launch ->
loads issued -> first stage landed -> main loop done -> slice reduction ->
cluster gather -> ranking -> fp64 recompute -> end, per CTA (first 8)."""
import ctypes as C
import os
import sys

os.environ.setdefault("DALI_LIB_PATH", os.path.join(os.path.dirname(__file__), "libdali_prof.so"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_03495_b200 import _lib  # noqa: E402
from paper_2602_03495_b200.trace import gate_norm2, route_device  # noqa: E402

lib = _lib.load()
if os.environ.get("RG_FORCE_FP64") == "1":
    lib.dali_route_guard_scale(-1.0)
d, N, k = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4096, 8, 2)))
Ts = [int(x) for x in (sys.argv[4].split(",") if len(sys.argv) > 4 else ["1", "16", "512"])]
g = (torch.randn(d, N, device="cuda") * 0.02).to(torch.bfloat16)
n2 = gate_norm2(g)
names = ["entry", "issued", "landed", "loop", "reduce", "pre-cl", "post-cl", "rank", "fp64"]  # tile kernel: 4 = tree done, no 5-6
for T in Ts:
    h = torch.randn(T, d, device="cuda").to(torch.bfloat16)
    for _ in range(5):
        route_device(h, g, k, norm2=n2)
    torch.cuda.synchronize()
    buf = (C.c_uint64 * 96)()
    lib.dali_rg_prof(buf)
    print(f"T={T}")
    for b in range(8):
        row = list(buf[b * 12:(b + 1) * 12])
        t0 = row[0]
        if not t0:
            continue
        print("  cta", b, " ".join(f"{n}={(row[i] - t0) if row[i] >= t0 else '-'}"
                                  for i, n in enumerate(names)))
