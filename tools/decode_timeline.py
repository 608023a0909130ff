"""Per-layer host/device timeline of the offloaded engine (diagnostic).

    python tools/decode_timeline.py [--model mixtral-8x7b] [--cache-gb 24] [--decode 48]

Runs one warm-up request and one traced request (EngineConfig.trace_layers)
and prints, for decode layers, where the wall time goes: host phases
(launch, decision wait, GPU dispatch, CPU experts, combine launch, the gap
to the next layer) and device phases (route -> decision, decision -> FFN
start = copy waits, FFN start -> combine end), grouped by how many experts
the layer ran on the CPU and whether the layer waited on a replacement.
"""
import argparse
import collections
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_03495_b200.engine import EngineConfig, build_engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="mixtral-8x7b")
ap.add_argument("--cache-gb", type=float, default=24.0)
ap.add_argument("--prefill", type=int, default=512)
ap.add_argument("--decode", type=int, default=48)
ap.add_argument("--prefetch", type=int, default=1)
ap.add_argument("--forced", type=int, default=1, help="teacher-forced decode like bench.py")
ap.add_argument("--out", default="gpurun_out/timeline.json")
ap.add_argument("--cost-model", default=None,
                help="cost-model JSON: loaded if it exists, else profiled and saved there "
                     "(fixes the decisions across A/B runs)")
args = ap.parse_args()
from paper_2602_03495_b200.cost_model import load_cost_model, save_cost_model  # noqa: E402
cm = None
if args.cost_model and os.path.exists(args.cost_model):
    cm = load_cost_model(args.cost_model)

cores = len(os.sched_getaffinity(0))
cfg = EngineConfig(cache_gb=args.cache_gb, prefetch_size=args.prefetch, w_size=4, seed=0,
                   cpu_threads=cores, trace_layers=True)
eng = build_engine(args.model, cfg, seed=0, max_seq=args.prefill + args.decode + 8,
                   log=lambda *a: print(*a, file=sys.stderr), cost_model=cm)
if args.cost_model and cm is None:
    save_cost_model(eng.cm, args.cost_model)
V = eng.arch.vocab_size
g = torch.Generator().manual_seed(1000)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import zipf_tokens  # noqa: E402  (the bench's teacher-forced decode stream)

for it in range(2):
    p = torch.randint(0, V, (1, args.prefill), generator=g)
    forced = zipf_tokens(V, (1, args.decode - 1), seed=3000 + it) if args.forced else None
    toks, st = eng.generate(p, args.decode, host_io=True, forced=forced)
    print(f"request {it}: prefill {st.prefill_tokens / st.prefill_ms * 1e3:.1f} tok/s decode "
          f"{st.decode_tokens / st.decode_ms * 1e3:.2f} tok/s", flush=True)
torch.cuda.synchronize()
lt = st.layer_trace
L = eng.arch.num_layers
rows, prows = [], []
for i, r in enumerate(lt):
    tp = r["host"]
    ev_r, ev_dec, t0, ev_c = r["ev"]
    nxt = lt[i + 1] if i + 1 < len(lt) else None
    d = dict(step=r["step"], layer=r["layer"], nC=r["nC"], hit=r["hit"], dem=r["dem"],
             pf=r["pf"], rep=r["rep"],
             h_launch=(tp[1] - tp[0]) * 1e3, h_wait=(tp[2] - tp[1]) * 1e3,
             h_presub=(r["tp_sub"] - tp[2]) * 1e3,
             g_rows_comb=(r["ev_rows"].elapsed_time(ev_c) if r.get("ev_rows") is not None
                          else None),
             h_disp=(tp[3] - tp[2]) * 1e3, h_cpu=(tp[4] - tp[3]) * 1e3,
             h_comb=(tp[5] - tp[4]) * 1e3,
             h_gap=((nxt["host"][0] - tp[5]) * 1e3) if nxt else None,
             g_route_dec=ev_r.elapsed_time(ev_dec),
             g_dec_ffn=ev_dec.elapsed_time(t0) if t0 is not None else None,
             g_ffn_comb=t0.elapsed_time(ev_c) if t0 is not None else None,
             g_dec_comb=ev_dec.elapsed_time(ev_c),
             g_prev_comb_to_route=(lt[i - 1]["ev"][3].elapsed_time(ev_r) if i > 0 else None))
    (rows if r["T"] == 1 else prows).append(d)


def mean(key, rs):
    v = [r[key] for r in rs if r[key] is not None]
    return round(float(np.mean(v)), 3) if v else None


keys = ["h_launch", "h_wait", "h_presub", "g_rows_comb", "h_disp", "h_cpu", "h_comb", "h_gap", "g_route_dec",
        "g_dec_ffn", "g_ffn_comb", "g_dec_comb", "g_prev_comb_to_route"]
steps = sorted({r["step"] for r in rows})
per_tok = (sum(r["h_launch"] + r["h_wait"] + r["h_disp"] + r["h_cpu"] + r["h_comb"] +
               (r["h_gap"] or 0) for r in rows) / max(len(steps), 1))
summary = {"decode_layers": len(rows), "steps": len(steps), "host_ms_per_token": per_tok,
           "all": {k: mean(k, rows) for k in keys}}
grp = collections.defaultdict(list)
for r in rows:
    grp[f"nC{r['nC']}_hit{r['hit']}_rep{r['rep']}"].append(r)
summary["groups"] = {g_: dict(n=len(rs), **{k: mean(k, rs) for k in keys})
                     for g_, rs in sorted(grp.items())}
by_layer = collections.defaultdict(list)
for r in rows:
    by_layer[r["layer"]].append(r)
summary["per_layer_wait"] = {l: mean("h_wait", rs) for l, rs in sorted(by_layer.items())}
summary["per_step_ms"] = {s: round(sum(r["h_launch"] + r["h_wait"] + r["h_disp"] + r["h_cpu"] +
                                       r["h_comb"] + (r["h_gap"] or 0)
                                       for r in rows if r["step"] == s), 2) for s in steps}
summary["prefill_layers"] = [
    {k: (round(v, 3) if isinstance(v, float) else v) for k, v in r.items()} for r in prows]
summary["cpu_expert_ms"] = [(int(r), round(float(ms), 3), kind, t0)
                            for r, ms, kind, t0 in st.cpu_expert_ms]
summary["cost_model_cpu"] = eng.cm.to_dict()["cpu_samples"]
summary["stats"] = {k: getattr(st, k) for k in ("demand_copies", "prefetch_copies",
                                                  "replace_copies", "cpu_expert_calls",
                                                  "gpu_expert_calls")}
print(json.dumps(summary, indent=1))
os.makedirs(os.path.dirname(args.out), exist_ok=True)
with open(args.out, "w") as f:
    json.dump(dict(summary=summary, rows=rows), f)
