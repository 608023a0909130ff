"""Print the key fields of a bench.py JSON line (diagnostic helper).

    python tools/bench_summary.py out.json [label]
"""
import json
import sys

d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
lab = sys.argv[2] if len(sys.argv) > 2 else ""
o = d.get("offload_roofline") or {}
p = d.get("prefill_roofline") or {}
print(lab, "value", d["value"], "e2e", d["e2e"]["value"], "prefill", d.get("prefill_tokens_per_s"),
      "e2e_prefill", d["e2e"].get("prefill_tokens_per_s"), "floor_frac", o.get("frac_of_floor"),
      "prefill cpu/h2d", p.get("cpu_experts"), p.get("h2d_copies"), "prefill_floor_frac",
      p.get("frac_of_floor"), "copies", d.get("copies_per_step"), flush=True)
