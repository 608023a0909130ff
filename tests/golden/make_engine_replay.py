"""Freeze B200 engine requests as reference-format replay fixtures
(VERDICT r1 "Engine -> moesim replay").

Run on a GPU box (the engine needs cuda:0; nothing here reads the reference):

    python tests/golden/make_engine_replay.py [out_dir]

For each case one request (a short prefill, then decode steps) runs through
the offloaded engine from its seeded initial cache -- the same residency the
reference's ``init_cache(layer, N, capacity, ..., seed)`` draws
(cache.py:67-101), so ``moesim`` semantics apply unchanged.  The engine's own
exporter (``engine.offload.export_trace``) writes:

* ``<case>.trace.jsonl.gz`` -- ``moesim-trace-v1`` (trace.py:385-406) with the
  per-step x per-layer workloads the engine routed and the bf16 gate inputs it
  captured (as fp64), gzip'd for the repository;
* ``<case>.gates.gz`` / ``<case>.res.gz`` -- the router (GateParams, L x d x N) and
  the engine's calibrated residual vectors (ResidualVectors, L-1 x d);
* ``<case>.cost.json`` -- the cost model the engine decided with (profiled on
  the box, quantised to the 2^-12 ms grid, or the reference default);
* ``<case>.engine.json`` -- the engine's SimConfig-equivalent knobs, its
  ``policy_report()`` (RunReport-shaped) and its per-(step, layer) GPU expert
  sets, cache lookups and replacement events.

``tests/test_engine_replay.py`` (CPU) feeds the artifacts to
``moesim.simulate_run`` (simulator.py:318-522) and requires the reference's
report and per-layer decisions to equal the engine's.
"""

from __future__ import annotations

import gzip
import json
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

# case -> (arch, cache slots/layer, prefetch size, batch, prompt, new tokens, profiled cm)
CASES = {
    "tiny": ("tiny", 2, 2, 1, 16, 24, False),
    "mixtral_L3": ("mixtral-8x7b@L3", 2, 1, 1, 8, 16, True),
    "qwen_L4_b2": ("qwen1.5-moe-a2.7b@L4", 38, 4, 2, 6, 12, True),
}


def _jsonable(x):
    if isinstance(x, dict):
        return {str(k): _jsonable(v) for k, v in x.items()}
    if isinstance(x, (list, tuple)):
        return [_jsonable(v) for v in x]
    if hasattr(x, "tolist"):
        return x.tolist()
    return x


def make_case(name, out_dir):
    from paper_2602_03495_b200.cost_model import default_cost_model, save_cost_model
    from paper_2602_03495_b200.engine import EngineConfig, build_engine
    from paper_2602_03495_b200.engine.offload import export_trace
    arch_name, slots, psize, B, S, new, profiled = CASES[name]
    cfg = EngineConfig(cache_slots_per_layer=slots, prefetch_size=psize, w_size=4, seed=3,
                       capture=True, cpu_threads=len(os.sched_getaffinity(0)))
    cm = None if profiled else default_cost_model(non_moe_layer_time=3.0)
    eng = build_engine(arch_name, cfg, seed=5, cost_model=cm, max_batch=B, max_seq=128)
    eng.reset_cache()
    prompt = torch.randint(0, eng.arch.vocab_size, (B, S),
                           generator=torch.Generator().manual_seed(21))
    toks, st = eng.generate(prompt, new)
    base = os.path.join(out_dir, name)
    export_trace(eng, base + ".trace.jsonl", base + ".gates", base + ".res", batch_size=B)
    for ext in (".trace.jsonl", ".gates", ".res"):
        with open(base + ext, "rb") as fi, gzip.open(base + ext + ".gz", "wb",
                                                     compresslevel=9) as fo:
            shutil.copyfileobj(fi, fo)
        os.remove(base + ext)
    save_cost_model(eng.cm, base + ".cost.json")
    log = eng.policy.decision_log()
    doc = {
        "case": name, "arch": arch_name,
        "sim_config": {"prefetch_kind": "residual", "prefetch_size": psize,
                       "cache_policy": "workload", "cache_capacity": eng.slots_per_layer,
                       "w_size": eng.cfg.w_size, "u_size": eng.cfg.u_size, "seed": eng.cfg.seed},
        "initial_on_gpu": st.initial_on_gpu.astype(int).tolist(),
        "report": _jsonable(eng.policy_report()),
        "decisions": [{"step": r["step"], "layer": r["layer"],
                       "gpu": [int(e) for e in range(len(r["G"])) if r["G"][e]],
                       "cpu": [int(e) for e in range(len(r["C"])) if r["C"][e]],
                       "hits": [[int(e), bool(h)] for e, h in r["hits"]],
                       "pset": r["pset"], "done": r["done"],
                       "event": r["event"], "latency": r["latency"]} for r in log],
        "cpu_expert_calls": st.cpu_expert_calls, "gpu_expert_calls": st.gpu_expert_calls,
        "device": torch.cuda.get_device_name(0),
    }
    with open(base + ".engine.json", "w") as f:
        json.dump(doc, f)
    print(f"{name}: {len(st.steps_meta)} steps, {st.cpu_expert_calls} CPU / "
          f"{st.gpu_expert_calls} GPU expert calls, hit rate {doc['report']['cache_hit_rate']}")
    del eng
    torch.cuda.empty_cache()


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "tests", "golden",
                                                              "engine_replay")
    os.makedirs(out, exist_ok=True)
    torch.cuda.set_device(0)
    for name in CASES:
        make_case(name, out)


if __name__ == "__main__":
    main()
