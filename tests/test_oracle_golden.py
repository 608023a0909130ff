"""Pin the CPU oracle (oracle/) against frozen reference outputs (CPU only)."""

import numpy as np
import pytest

from conftest import sha, trace_from_meta
from oracle import driver as D
from oracle import policy as P


def test_hand_gating(golden):
    a, _ = golden
    assert P.derive_workloads(a["hand_hidden"], a["hand_gate"], 2).tolist() == \
        a["hand_workloads_k2"].tolist() == [2, 2, 1, 1]
    assert P.stable_topk(np.array([1.0, 2.0, 2.0, 0.5]), 2).tolist() == [1, 2]
    assert P.stable_topk(np.array([7.0, 7.0, 7.0]), 3).tolist() == [0, 1, 2]


def test_interp_bitwise(golden):
    a, meta = golden
    tb = P.default_tables()
    ws = a["interp_w"]
    assert np.array_equal(np.array([tb.t_cpu(w) for w in ws]), a["interp_cpu_default"])
    assert np.array_equal(np.array([tb.t_gpu_compute(w) for w in ws]), a["interp_gpu_default"])
    for i, m in enumerate(meta["interp_models"]):
        t = P.tables_from_samples(m["cpu_samples"], m["gpu_samples"], m["trans_time"])
        got_c = np.array([P.interp_ms(w, t.cpu_xs, t.cpu_ys) for w in ws[1:]])
        got_g = np.array([P.interp_ms(w, t.gpu_xs, t.gpu_ys) for w in ws[1:]])
        assert np.array_equal(got_c, a[f"interp_cpu_rnd{i}"])
        assert np.array_equal(got_g, a[f"interp_gpu_rnd{i}"])


@pytest.mark.parametrize("stream", ["cost", "cost_wide", "times"])
def test_greedy_streams(golden, stream):
    _, meta = golden
    tb = P.default_tables()
    for case in meta["greedy"][stream]:
        w = np.array(case["workloads"], np.int64)
        res = np.array(case["resident"], bool)
        if stream.startswith("cost"):
            ct, gt = P.expert_times(tb, w, res)
            assert ct.tolist() == case["cpu_times"] and gt.tolist() == case["gpu_times"]
        else:
            ct, gt = np.array(case["cpu_times"]), np.array(case["gpu_times"])
        C, G, order = P.greedy(w, res, ct, gt, case["capacity"])
        assert order.tolist() == case["order"]
        assert C.tolist() == case["C"] and G.tolist() == case["G"]


def test_cache_sequences(golden):
    _, meta = golden
    for name, c in meta["cache"].items():
        lc = P.new_cache(c["layer"], c["n"], c["cap"], c["w"], c["u"], c["seed"])
        assert lc.on_gpu.astype(int).tolist() == c["init"], name
        for t, want in enumerate(c["events"]):
            ev = P.window_update(lc, np.array(c["seq"][t]), t == c["eos_at"])
            if want is None:
                assert ev is None, (name, t)
            else:
                assert [ev[0], ev[1], len(ev[1]) * 3.0] == want, (name, t)
        assert lc.on_gpu.astype(int).tolist() == c["final"]


@pytest.fixture(scope="module")
def traces(golden):
    _, meta = golden
    return {n: trace_from_meta(i) for n, i in meta["traces"].items()}


def test_generator_regenerates_reference_arrays(golden, traces):
    _, meta = golden
    for name, info in meta["traces"].items():
        tr = traces[name]
        assert sha(tr.gates) == info["sha_gates"], name
        assert sha(np.stack([s.hidden for s in tr.steps])) == info["sha_hidden"], name
        res = P.calibrate([s.hidden for s in tr.steps])
        assert sha(res) == info["sha_res"], name


def test_gating_and_prefetch_on_traces(golden, traces):
    a, meta = golden
    for name, info in meta["traces"].items():
        tr, k, L = traces[name], info["k"], info["L"]
        wl = np.stack([s.workloads for s in tr.steps])
        assert np.array_equal(wl, a[f"{name}_workloads"]), name
        s0 = tr.steps[0]
        top = np.stack([P.route(s0.hidden[l], tr.gates[l], k)[0] for l in range(L)])
        assert np.array_equal(top, a[f"{name}_topk_s0"]), name
        res = P.calibrate([s.hidden for s in tr.steps])
        pred, psets = [], []
        for s in tr.steps:
            for l in range(L - 1):
                p, ps = P.predict_next(s.hidden[l], res[l], tr.gates[l + 1], k, 2)
                pred.append(p)
                psets.append(ps)
        assert np.array_equal(np.array(pred), a[f"{name}_pred"]), name
        assert np.array_equal(np.array(psets), a[f"{name}_psets"]), name


def _driver_cfg(name, over, N):
    nm = 3.0 if "nm3" in name else 0.0
    kw = dict(tables=P.default_tables(non_moe_layer_time=nm))
    m = {"assignment_policy": "assignment_policy", "prefetch_size": "prefetch_size",
         "cache_capacity": "cache_capacity", "w_size": "w_size", "u_size": "u_size",
         "seed": "seed", "gpu_capacity": "gpu_capacity",
         "non_moe_override": "non_moe_override",
         "scheduling_overhead_ms": "scheduling_overhead_ms",
         "solver_node_cost_ms": "solver_node_cost_ms",
         "prefetch_compute_ms": "prefetch_compute_ms", "beam_width": "beam_width",
         "threshold": "threshold", "exact_solver_limit": "exact_solver_limit",
         "prefetch_kind": "prefetch_kind", "cache_policy": "cache_policy",
         "insert_demand_fetched": "insert_demand_fetched",
         "insert_prefetched": "insert_prefetched"}
    for key, val in over.items():
        if key in m:
            kw[m[key]] = val
    return D.DriverConfig(**kw)


def test_driver_reports_match_reference(golden, traces):
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/golden")
    from make_golden_cfgs import run_cfgs  # noqa
    _, meta = golden
    for key, want in meta["runs"].items():
        tname, rname = key.split("/")
        tr = traces[tname]
        info = meta["traces"][tname]
        over = dict(run_cfgs(info["N"]))[rname]
        cfg = _driver_cfg(rname, over, info["N"])
        if over.get("prefetch_size"):
            cfg.residuals = P.calibrate([s.hidden for s in tr.steps])
        steps = [D.StepInput(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                 for s in tr.steps]
        rep, _ = D.run(steps, tr.gates, cfg, info["L"], info["N"], info["k"])
        assert rep == want, key


def test_driver_baseline_reports_match_reference(golden, traces):
    """Alternative policies: beam / optimal / static
    solvers, LRU and score caches, insert toggles, feature / statistical /
    random predictors -- whole reports equal the reference's, and the exact
    solver refuses the same instances."""
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/golden")
    from make_golden_cfgs import baseline_cfgs  # noqa
    _, meta = golden
    assert len(meta["runs_baseline"]) >= 80
    for key, want in meta["runs_baseline"].items():
        tname, rname = key.split("/")
        tr = traces[tname]
        info = meta["traces"][tname]
        over = dict(baseline_cfgs(info["N"]))[rname]
        cfg = _driver_cfg(rname, over, info["N"])
        if over.get("prefetch_kind") == "residual":
            cfg.residuals = P.calibrate([s.hidden for s in tr.steps])
        if over.get("prefetch_kind") == "statistical":
            cfg.frequency_table = P.frequency_table([s.workloads for s in tr.steps])
        steps = [D.StepInput(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                 for s in tr.steps]
        if "error" in want:
            with pytest.raises(ValueError, match="exact solver limited"):
                D.run(steps, tr.gates, cfg, info["L"], info["N"], info["k"])
            continue
        rep, _ = D.run(steps, tr.gates, cfg, info["L"], info["N"], info["k"])
        assert rep == want, key
