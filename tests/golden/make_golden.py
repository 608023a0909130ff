"""Freeze reference (``moesim``) outputs into small fixtures.

Run in the BUILD container only (it imports the real reference from
``/root/reference/pkg/src``; that tree does not exist on the GPU box):

    python tests/golden/make_golden.py

Outputs (committed): ``tests/golden/golden.npz`` (arrays) and
``tests/golden/golden.json`` (reports / ragged lists).  Inputs that are large
(synthetic traces at model shapes) are NOT stored: the tests regenerate them
with ``oracle.policy.synth_trace`` (same numpy RNG draw order as the
reference generator, trace.py:274-375) and the fixture stores a sha256 of the
reference's arrays so a regeneration mismatch is caught.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

import moesim  # noqa: E402
from moesim import cache as mc  # noqa: E402
from moesim import prefetch as mp  # noqa: E402
from moesim.assignment import greedy_assign  # noqa: E402
from moesim.cost_model import _interp, default_cost_model, fit_cost_model  # noqa: E402
from moesim.simulator import SimConfig, simulate_run  # noqa: E402
from moesim.trace import (ModelConfig, derive_workloads,  # noqa: E402
                          generate_synthetic_trace, topk_indices)

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from make_golden_cfgs import baseline_cfgs, run_cfgs  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def per_token_topk(hidden, gate, k):
    from moesim.trace import gate_scores
    s = gate_scores(hidden, gate)
    return np.stack([topk_indices(r, k) for r in s]).astype(np.int64)


# Trace shapes: (name, L, N, k, d, batch, steps, phase, gen kwargs)
TRACES = [
    ("tiny_decode", 4, 8, 2, 256, 1, 32, "decode",
     dict(locality=0.9, drift_scale=0.4, noise_scale=0.08, seed=7)),
    ("tiny_prefill", 4, 8, 2, 256, 1, 128, "prefill",
     dict(locality=0.9, drift_scale=0.4, noise_scale=0.08, seed=7)),
    ("headline", 4, 16, 2, 32, 32, 48, "decode",
     dict(locality=0.9, drift_scale=0.4, noise_scale=0.08, seed=7)),
    ("mixtral_decode", 3, 8, 2, 4096, 4, 6, "decode",
     dict(locality=0.9, drift_scale=0.4, noise_scale=0.08, seed=11)),
    ("qwen_decode", 3, 60, 4, 2048, 16, 4, "decode",
     dict(locality=0.9, drift_scale=0.4, noise_scale=0.08, seed=13)),
    ("dsv2_prefill", 2, 64, 6, 2048, 1, 512, "prefill",
     dict(locality=0.9, drift_scale=0.4, noise_scale=0.08, seed=17)),
]


def main():
    arrays = {}
    meta = {"moesim_version": moesim.__version__, "numpy": np.__version__,
            "traces": {}, "runs": {}, "runs_baseline": {}, "greedy": {}, "cache": {}}

    # --- gating hand cases (test_trace.py:37-72) --------------------------
    gate = np.array([[3.0, 1.0, 2.0, 0.0], [0.0, 2.0, 1.0, 3.0], [2.0, 3.0, 0.0, 1.0]])
    arrays["hand_gate"] = gate
    arrays["hand_hidden"] = np.eye(3)
    arrays["hand_workloads_k2"] = derive_workloads(np.eye(3), gate, 2)

    # --- interp (cost_model.py:19-27) -------------------------------------
    cm = default_cost_model()
    ws = np.arange(0, 5000, dtype=np.float64)
    arrays["interp_w"] = ws
    arrays["interp_cpu_default"] = np.array([cm.t_cpu(w) for w in ws])
    arrays["interp_gpu_default"] = np.array([cm.t_gpu_compute(w) for w in ws])
    rng = np.random.default_rng(99)
    rnd_models = []
    for i in range(6):
        xs = np.unique(rng.integers(1, 300, size=int(rng.integers(1, 7))))
        ys = np.cumsum(rng.uniform(0.01, 9.0, size=len(xs)))
        xg = np.unique(rng.integers(1, 300, size=int(rng.integers(1, 7))))
        yg = np.cumsum(rng.uniform(0.001, 2.0, size=len(xg)))
        m = fit_cost_model(list(zip(xs, ys)), list(zip(xg, yg)), trans_time=float(rng.uniform(0.5, 5)))
        rnd_models.append(m.to_dict())
        arrays[f"interp_cpu_rnd{i}"] = np.array([_interp(w, m.cpu_xs, m.cpu_ys) for w in ws[1:]])
        arrays[f"interp_gpu_rnd{i}"] = np.array([_interp(w, m.gpu_xs, m.gpu_ys) for w in ws[1:]])
    meta["interp_models"] = rnd_models

    # --- greedy streams (conftest.py:20-58 generators) --------------------
    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import random_instance, random_times_instance
    for name, gen in [("cost", lambda r: random_instance(r, cm, resident_prob=0.3, capacity_prob=0.5)),
                      ("cost_wide", lambda r: random_instance(r, cm, n_act_range=(20, 60), max_workload=400,
                                                              resident_prob=0.3, capacity_prob=0.5)),
                      ("times", lambda r: random_times_instance(r, resident_prob=0.4, capacity_prob=0.6))]:
        r = np.random.default_rng({"cost": 5, "cost_wide": 6, "times": 23}[name])
        cases = []
        for _ in range(300):
            inst = gen(r)
            a = greedy_assign(inst)
            cases.append({
                "workloads": inst.workloads.tolist(),
                "resident": inst.resident.astype(int).tolist(),
                "capacity": inst.gpu_capacity,
                "cpu_times": inst.cpu_times.tolist(),
                "gpu_times": inst.gpu_times.tolist(),
                "order": inst.sorted_order().tolist(),
                "C": a.C.tolist(), "G": a.G.tolist()})
        meta["greedy"][name] = cases

    # --- cache sequences (cache.py:146-214) --------------------------------
    r = np.random.default_rng(77)
    for ci in range(12):
        n = int(r.integers(4, 70))
        cap = int(r.integers(1, n))
        u = int(r.integers(0, min(cap, n - cap) + 1))
        wsz = int(r.integers(1, 6))
        seed = int(r.integers(0, 100))
        layer = int(r.integers(0, 30))
        st = mc.init_cache(layer, n, cap, wsz, u, seed=seed)
        init = st.on_gpu.copy()
        seq = r.integers(0, 9, size=(40, n))
        if ci % 3 == 0:
            seq[:, : n // 2] = 3  # force ties
        eos_at = int(r.integers(20, 45))
        events = []
        for t in range(40):
            ev = mc.record_and_maybe_replace(st, seq[t], t, is_eos=(t == eos_at), trans_time_ms=3.0)
            events.append(None if ev is None else [ev.evicted, ev.admitted, ev.transfer_cost_ms])
        meta["cache"][f"c{ci}"] = {"n": n, "cap": cap, "u": u, "w": wsz, "seed": seed,
                                   "layer": layer, "eos_at": eos_at,
                                   "init": init.astype(int).tolist(),
                                   "seq": seq.tolist(), "events": events,
                                   "final": st.on_gpu.astype(int).tolist()}

    # --- traces: gating, prefetch, full runs --------------------------------
    for (name, L, N, k, d, B, S, phase, kw) in TRACES:
        cfg = ModelConfig(num_layers=L, num_routed_experts=N, num_shared_experts=0,
                          top_k=k, hidden_dim=d)
        tr = generate_synthetic_trace(cfg, batch_size=B, num_steps=S, phase=phase, **kw)
        hid = np.stack([s.hidden for s in tr.steps])  # (S, L, T, d)
        wl = np.stack([s.workloads for s in tr.steps])
        res = mp.calibrate_residuals(tr)
        info = {"L": L, "N": N, "k": k, "d": d, "B": B, "S": S, "phase": phase, "kw": kw,
                "sha_gates": sha(tr.gate_params.weights), "sha_hidden": sha(hid),
                "sha_res": sha(res.values)}
        arrays[f"{name}_workloads"] = wl
        # per-token top-k of the first step, every layer
        arrays[f"{name}_topk_s0"] = np.stack([per_token_topk(tr.steps[0].hidden[l],
                                                             tr.gate_params.layer(l), k)
                                              for l in range(L)])
        # residual predictions for every (step, layer<L-1), P = 2
        rp = mp.residual_predictor(res)
        pred, psets = [], []
        for s in tr.steps:
            for l in range(L - 1):
                dcs = mp.predict_next_layer(rp, s.hidden[l], tr.gate_params.layer(l + 1), k, 2, l)
                pred.append(dcs.predicted_workloads)
                psets.append(dcs.prefetch_set)
        arrays[f"{name}_pred"] = np.array(pred)
        arrays[f"{name}_psets"] = np.array(psets)
        meta["traces"][name] = info
        for rn, over in run_cfgs(N):
            cm_run = default_cost_model(non_moe_layer_time=3.0 if "nm3" in rn else 0.0)
            sc = dict(cost_model=cm_run)
            sc.update(over)
            if sc.get("prefetch_kind") == "residual":
                sc["residuals"] = res
            rep = simulate_run(tr, SimConfig(**sc)).to_dict()
            rep.pop("spec")
            rep.pop("timelines")
            meta["runs"][f"{name}/{rn}"] = rep
        for rn, over in baseline_cfgs(N):
            cm_run = default_cost_model(non_moe_layer_time=3.0 if "nm3" in rn else 0.0)
            sc = dict(cost_model=cm_run)
            sc.update(over)
            if sc.get("prefetch_kind") == "residual":
                sc["residuals"] = res
            if sc.get("prefetch_kind") == "statistical":
                sc["frequency_table"] = mp.activation_frequency_table(tr)
            try:
                rep = simulate_run(tr, SimConfig(**sc)).to_dict()
                rep.pop("spec")
                rep.pop("timelines")
            except moesim.errors.MoesimError as exc:
                rep = {"error": type(exc).__name__, "message": str(exc)}
            meta["runs_baseline"][f"{name}/{rn}"] = rep

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(meta, f, sort_keys=True)
    print("wrote", len(arrays), "arrays;", len(meta["runs"]), "runs")


if __name__ == "__main__":
    main()
