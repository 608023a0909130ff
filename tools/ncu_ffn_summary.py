"""Summarise an ncu --set full --page raw --csv capture of tools/prof_ffn.py
--mode all into per-FFN-call DRAM traffic vs algorithmic bytes.

    python tools/ncu_ffn_summary.py gpurun_out/ffn_full_raw.csv profiles/r01_ncu_ffn_traffic.json

Each FFN call is an (up, down) kernel pair; prof_ffn.py's shapes in order
(after the skipped warm-ups) are 1x1, 1x2, 2x2, 4x8, 16x8 ... (tokens x
experts; 1x2 and 2x2 have identical grids and are grouped as 1x2).  Algorithmic bytes = weight blocks of the GPU experts + token
activations (prof_ffn.py's formula)."""
import csv
import json
import sys

D, F = 4096, 14336
# consecutive launches with identical grids are one group: 1x2 and 2x2 share grids
SHAPES = [(1, 1), (1, 2), (4, 8), (16, 8), (64, 8), (128, 8), (256, 8), (512, 8)]


def alg_bytes(tok, n_exp, splits):
    rows = tok * n_exp
    return n_exp * 3 * F * D * 2 + rows * (D * 2 + 2 * F * 2 + D * 4 * splits)


rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
data = [r for r in rows[hi + 2:] if len(r) > 5]
c = {n: h.index(n) for n in ("Kernel Name", "Grid Size", "gpu__time_duration.sum",
                             "dram__bytes_read.sum", "dram__bytes_write.sum")}
pairs = [(data[i], data[i + 1]) for i in range(0, len(data) - 1, 2)]
out = {"source": "ncu --set full --clock-control none -k regex:ffn_tc (tools/prof_ffn.py --mode "
                 "all --iters 2), per (up, down) kernel pair", "calls": []}
# prof_ffn runs each shape 3 warm-up + iters timed; ncu -s 6 skipped 3 launches (pairs)
per_shape = {}
seen = []
for up, dn in pairs:
    grid = (up[c["Grid Size"]], dn[c["Grid Size"]])
    if not seen or seen[-1][0] != grid:
        seen.append([grid, []])
    seen[-1][1].append((up, dn))
for (grid, calls), (tok, n_exp) in zip(seen, SHAPES):
    t = sum(float(u[c["gpu__time_duration.sum"]]) + float(d_[c["gpu__time_duration.sum"]])
            for u, d_ in calls) / len(calls)
    rd = sum(float(u[c["dram__bytes_read.sum"]]) + float(d_[c["dram__bytes_read.sum"]])
             for u, d_ in calls) / len(calls)
    wr = sum(float(u[c["dram__bytes_write.sum"]]) + float(d_[c["dram__bytes_write.sum"]])
             for u, d_ in calls) / len(calls)
    alg = alg_bytes(tok, n_exp, 1)
    out["calls"].append({"shape": f"{tok} token(s) x {n_exp} expert(s)", "grids": grid,
                         "launches": len(calls), "time_ns": t, "dram_read_bytes": rd,
                         "dram_write_bytes": wr, "algorithmic_bytes_weights_acts": alg,
                         "traffic_over_algorithmic": (rd + wr) / alg})
with open(sys.argv[2], "w") as f:
    json.dump(out, f, indent=1)
for cl in out["calls"]:
    print(cl["shape"], round(cl["time_ns"] / 1e3, 1), "us", round(cl["traffic_over_algorithmic"], 4))
