"""GPU parity: policy kernels vs the oracle and the frozen reference outputs.

Bit-exact bar: workloads, per-token top-k indices, greedy C/G/order,
interpolated times, prefetch sets, cache events, full run reports and
per-layer decision logs.
"""

import numpy as np
import pytest

from conftest import trace_from_meta
from oracle import driver as D
from oracle import policy as P

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dali():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_2602_03495_b200 as m
    return m


@pytest.fixture(scope="module")
def traces(golden):
    _, meta = golden
    return {n: trace_from_meta(i) for n, i in meta["traces"].items()}


# --- gating -----------------------------------------------------------------

def test_gating_hand_cases(dali, golden):
    a, _ = golden
    assert dali.derive_workloads(a["hand_hidden"], a["hand_gate"], 2).tolist() == [2, 2, 1, 1]
    gate = np.zeros((3, 4))
    gate[0, 1] = 10.0
    assert dali.derive_workloads(np.array([[1.0, 0, 0]]), gate, 1).tolist() == [0, 1, 0, 0]
    rng = np.random.default_rng(0)
    assert dali.derive_workloads(rng.normal(size=(3, 5)), rng.normal(size=(5, 4)), 4).tolist() \
        == [3, 3, 3, 3]
    # exact ties -> lower index (all-zero logits)
    assert dali.trace.route_topk(np.zeros((2, 3)), np.zeros((3, 5)), 3).tolist() == \
        [[0, 1, 2], [0, 1, 2]]
    with pytest.raises(dali.TraceError):
        dali.derive_workloads(np.ones((1, 3)), np.ones((4, 4)), 1)
    with pytest.raises(dali.TraceError):
        dali.derive_workloads(np.ones((1, 4)), np.ones((4, 4)), 5)


def test_gating_empty_and_single_expert(dali):
    import torch
    from paper_2602_03495_b200.trace import route_device
    h = torch.zeros((0, 16), dtype=torch.float64, device="cuda")
    g = torch.ones((16, 4), dtype=torch.float64, device="cuda")
    _, _, wl = route_device(h, g, 2)
    assert wl.cpu().tolist() == [0, 0, 0, 0]
    assert dali.derive_workloads(np.ones((5, 3)), np.ones((3, 1)), 1).tolist() == [5]


def test_gating_on_reference_traces(dali, golden, traces):
    a, meta = golden
    for name, info in meta["traces"].items():
        tr, L, k = traces[name], info["L"], info["k"]
        for si, st in enumerate(tr.steps):
            for l in range(L):
                got = dali.derive_workloads(st.hidden[l], tr.gates[l], k)
                assert np.array_equal(got, a[f"{name}_workloads"][si, l]), (name, si, l)
        s0 = tr.steps[0]
        top = np.stack([dali.trace.route_topk(s0.hidden[l], tr.gates[l], k) for l in range(L)])
        assert np.array_equal(top, a[f"{name}_topk_s0"]), name


def test_gating_bf16_matches_fp64_oracle_on_bf16_values(dali):
    """Engine path: bf16 hidden + bf16 gate, fp64 arithmetic == oracle on the
    same (exactly representable) values, at BASELINE shapes."""
    import torch
    from paper_2602_03495_b200.trace import route_device
    for (T, d, N, k) in [(128, 256, 8, 2), (512, 4096, 8, 2), (16, 2048, 60, 4),
                         (1024, 2048, 64, 6)]:
        g = torch.Generator().manual_seed(T + N)
        h = torch.randn(T, d, generator=g).to(torch.bfloat16)
        w = (torch.randn(d, N, generator=g) * 0.4 / d ** 0.5 *
             torch.linspace(0.15, 1.85, N)[torch.randperm(N, generator=g)]).to(torch.bfloat16)
        idx, wts, wl = route_device(h.cuda(), w.cuda(), k, renorm=True)
        o_idx, o_sc, o_wl = P.route(h.double().numpy(), w.double().numpy(), k)
        assert np.array_equal(idx.cpu().numpy(), o_idx), (T, d, N)
        assert np.array_equal(wl.cpu().numpy(), o_wl)
        ref_w = o_sc / o_sc.sum(axis=1, keepdims=True)
        np.testing.assert_allclose(wts.cpu().numpy(), ref_w, rtol=1e-6)


# --- cost model + greedy ----------------------------------------------------

def test_cost_eval_bitwise(dali, golden):
    a, meta = golden
    cm = dali.default_cost_model()
    ws = a["interp_w"]
    assert np.array_equal(cm.cpu_times(ws), a["interp_cpu_default"])
    assert np.array_equal(cm._eval(ws)[1], a["interp_gpu_default"])
    for i, m in enumerate(meta["interp_models"]):
        c = dali.fit_cost_model(m["cpu_samples"], m["gpu_samples"], m["trans_time"])
        co, go = c._eval(ws[1:])
        assert np.array_equal(co, a[f"interp_cpu_rnd{i}"]), i
        assert np.array_equal(go, a[f"interp_gpu_rnd{i}"]), i


@pytest.mark.parametrize("stream", ["cost", "cost_wide", "times"])
def test_greedy_streams(dali, golden, stream):
    _, meta = golden
    cm = dali.default_cost_model()
    for case in meta["greedy"][stream]:
        w = np.array(case["workloads"], np.int64)
        res = np.array(case["resident"], bool)
        if stream.startswith("cost"):
            inst = dali.AssignmentInstance(w, res, cm, case["capacity"])
            assert inst.cpu_times.tolist() == case["cpu_times"]
            assert inst.gpu_times.tolist() == case["gpu_times"]
        else:
            inst = dali.AssignmentInstance.from_times(case["cpu_times"], case["gpu_times"],
                                                      workloads=w, resident=res,
                                                      gpu_capacity=case["capacity"])
        a = dali.greedy_assign(inst)
        assert a.C.tolist() == case["C"] and a.G.tolist() == case["G"]
        assert inst.sorted_order().tolist() == case["order"]
        assert dali.validate(inst, a) == []


def test_greedy_reference_hand_cases(dali):
    f = dali.AssignmentInstance.from_times
    a = dali.greedy_assign(f([8, 6, 4, 2], [2, 3, 3, 3]))
    assert a.G.tolist() == [1, 1, 0, 0] and a.C.tolist() == [0, 0, 1, 1]
    assert dali.makespan(f([8, 6, 4, 2], [2, 3, 3, 3]), a) == (6.0, 5.0, 6.0)
    assert dali.greedy_assign(f([3], [3])).G.tolist() == [1]          # tie -> GPU
    inst = f([10, 10, 10], [1, 1, 1], gpu_capacity=1)
    assert dali.greedy_assign(inst).G.sum() == 1
    z = dali.AssignmentInstance(np.zeros(5, int), np.zeros(5, bool), dali.default_cost_model())
    a = dali.greedy_assign(z)
    assert a.C.sum() == 0 and a.G.sum() == 0


def test_greedy_max_experts(dali):
    rng = np.random.default_rng(1)
    cm = dali.default_cost_model()
    tb = P.default_tables()
    for n in (128, 256):
        w = rng.integers(0, 50, n)
        res = rng.random(n) < 0.3
        a = dali.greedy_assign(dali.AssignmentInstance(w, res, cm, 7))
        ct, gt = P.expert_times(tb, w, res)
        C, G, _ = P.greedy(w, res, ct, gt, 7)
        assert np.array_equal(a.C, C) and np.array_equal(a.G, G)


# --- prefetch -----------------------------------------------------------------

def test_prefetch_hand_case(dali):
    gate_next = np.array([[1.0, 0.0, 3.0, 0.0], [0.0, 1.0, 0.0, 3.0]])
    res = dali.ResidualVectors(np.array([[-1.0, 2.0]]))
    d = dali.predict_next_layer(dali.residual_predictor(res), np.eye(2), gate_next, k=2,
                                prefetch_size=2, current_layer=0)
    assert d.predicted_workloads.tolist() == [0, 2, 0, 2]
    assert d.prefetch_set.tolist() == [1, 3]
    assert d.layer == 1
    with pytest.raises(dali.PrefetchError, match="last layer"):
        dali.predict_next_layer(dali.residual_predictor(res), np.eye(2), gate_next, 2, 2, 1)


def test_prefetch_on_reference_traces(dali, golden, traces):
    a, meta = golden
    for name, info in meta["traces"].items():
        tr, L, k = traces[name], info["L"], info["k"]
        res = P.calibrate([s.hidden for s in tr.steps])
        rp = dali.residual_predictor(dali.ResidualVectors(res))
        pred, psets = [], []
        for s in tr.steps:
            for l in range(L - 1):
                dcs = dali.predict_next_layer(rp, s.hidden[l], tr.gates[l + 1], k, 2, l)
                pred.append(dcs.predicted_workloads)
                psets.append(dcs.prefetch_set)
        assert np.array_equal(np.array(pred), a[f"{name}_pred"]), name
        assert np.array_equal(np.array(psets), a[f"{name}_psets"]), name


def test_calibration_on_device_close_to_oracle(dali, traces):
    tr = traces["tiny_decode"]
    cfg = dali.ModelConfig(tr.L, tr.N, 0, tr.k, tr.d)
    t = dali.Trace(cfg, 1, "decode", [dali.TokenStep(s.token_index, s.tokens, s.workloads,
                                                     s.hidden, s.eos) for s in tr.steps])
    got = dali.calibrate_residuals(t).values
    np.testing.assert_allclose(got, P.calibrate([s.hidden for s in tr.steps]), rtol=0,
                               atol=1e-12)


# --- cache --------------------------------------------------------------------

def test_cache_sequences(dali, golden):
    _, meta = golden
    for name, c in meta["cache"].items():
        st = dali.init_cache(c["layer"], c["n"], c["cap"], c["w"], c["u"], seed=c["seed"])
        assert st.on_gpu.astype(int).tolist() == c["init"]
        for t, want in enumerate(c["events"]):
            ev = dali.record_and_maybe_replace(st, np.array(c["seq"][t]), t,
                                               is_eos=(t == c["eos_at"]), trans_time_ms=3.0)
            if want is None:
                assert ev is None, (name, t)
            else:
                assert [ev.evicted, ev.admitted, ev.transfer_cost_ms] == want, (name, t)
        assert st.on_gpu.astype(int).tolist() == c["final"]


def test_cache_worked_example(dali):
    st = dali.init_cache(0, 8, 4, 4, 2)
    st.on_gpu[:] = False
    st.on_gpu[[0, 1, 2, 3]] = True
    per_token = np.array([9.0, 1.0, 8.0, 2.0, 7.0, 0.0, 6.0, 0.0]) / 4.0
    evs = [dali.record_and_maybe_replace(st, per_token, t) for t in range(4)]
    assert evs[:3] == [None, None, None]
    assert sorted(evs[3].evicted) == [1, 3] and sorted(evs[3].admitted) == [4, 6]
    assert sorted(st.expert_on_gpu) == [0, 2, 4, 6]
    assert (st.scores == 0.0).all()
    st = dali.init_cache(0, 8, 4, 1, 2)
    st.on_gpu[:] = False
    st.on_gpu[[0, 1, 2, 3]] = True
    ev = dali.record_and_maybe_replace(st, np.zeros(8), 0)
    assert ev.evicted == [0, 1] and ev.admitted == [4, 5]
    st = dali.init_cache(0, 8, 4, 2, 0)
    before = st.on_gpu.copy()
    assert dali.record_and_maybe_replace(st, np.arange(8.0), 0) is None
    ev = dali.record_and_maybe_replace(st, np.arange(8.0), 1)
    assert ev.evicted == [] and ev.admitted == []
    assert np.array_equal(st.on_gpu, before)


# --- full runs ----------------------------------------------------------------

def _sim_config(dali, rname, over, res):
    nm = 3.0 if "nm3" in rname else 0.0
    kw = dict(cost_model=dali.default_cost_model(non_moe_layer_time=nm))
    kw.update(over)
    if kw.get("prefetch_kind") == "residual":
        kw["residuals"] = dali.ResidualVectors(res)
    return dali.SimConfig(**kw)


def test_simulate_run_matches_reference_reports(dali, golden, traces):
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/golden")
    from make_golden_cfgs import run_cfgs
    _, meta = golden
    for key, want in meta["runs"].items():
        tname, rname = key.split("/")
        tr, info = traces[tname], meta["traces"][tname]
        over = dict(run_cfgs(info["N"]))[rname]
        res = P.calibrate([s.hidden for s in tr.steps])
        cfg = dali.ModelConfig(info["L"], info["N"], 0, info["k"], info["d"])
        t = dali.Trace(cfg, info["B"], info["phase"],
                       [dali.TokenStep(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                        for s in tr.steps], gate_params=dali.GateParams(tr.gates))
        rep = dali.simulate_run(t, _sim_config(dali, rname, over, res)).to_dict()
        rep.pop("spec")
        rep.pop("timelines")
        assert rep == want, key


def test_decision_log_matches_oracle(dali, traces):
    """Entry-by-entry: C/G, residency, lookups, prefetch sets, arrivals, events."""
    tr = traces["headline"]
    res = P.calibrate([s.hidden for s in tr.steps])
    for nm, cap, psize in [(3.0, 8, 1), (0.5, 4, 3), (40.0, 8, 4)]:
        tb = P.default_tables(non_moe_layer_time=nm)
        dcfg = D.DriverConfig(tables=tb, prefetch_size=psize, residuals=res,
                              cache_capacity=cap, w_size=4, u_size=1, seed=3)
        steps = [D.StepInput(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                 for s in tr.steps]
        orep, recs = D.run(steps, tr.gates, dcfg, tr.L, tr.N, tr.k)
        cfg = dali.ModelConfig(tr.L, tr.N, 0, tr.k, tr.d)
        t = dali.Trace(cfg, 32, "decode", [dali.TokenStep(s.token_index, s.tokens, s.workloads,
                                                          s.hidden, s.eos) for s in tr.steps],
                       gate_params=dali.GateParams(tr.gates))
        sc = dali.SimConfig(cost_model=dali.default_cost_model(non_moe_layer_time=nm),
                            prefetch_kind="residual", prefetch_size=psize,
                            residuals=dali.ResidualVectors(res), cache_policy="workload",
                            cache_capacity=cap, w_size=4, u_size=1, seed=3)
        run = dali.simulate_run(t, sc)
        got = run.decisions
        assert len(got) == len(recs)
        n_arrived = 0
        for g, o in zip(got, recs):
            assert (g["step"], g["layer"]) == (o.step, o.layer)
            assert np.array_equal(g["C"], o.C) and np.array_equal(g["G"], o.G)
            assert np.array_equal(g["resident"], o.resident)
            assert g["hits"] == o.lookups
            if o.prefetch_set is not None:
                assert g["pset"] == o.prefetch_set.tolist()
                assert g["cand"] == o.candidates and g["done"] == o.completed
                n_arrived += len(o.completed)
            assert g["event"] == o.event
            assert (g["cpu_busy"], g["gpu_makespan"], g["latency"], g["demand_end"]) == \
                (o.cpu_busy, o.gpu_makespan, o.latency, o.demand_end)
        orep.pop("replacement_events")
        rep = run.to_dict()
        rep.pop("replacement_events")
        for k in orep:
            assert rep[k] == orep[k], k
        if nm == 40.0:
            assert n_arrived > 0   # the arrival rule is exercised


# --- alternative policies ---------------------------------

def test_simulate_run_baselines_match_reference_reports(dali, golden, traces):
    """Beam / optimal / static solvers, LRU + score caches, insert toggles,
    feature / statistical / random predictors: whole reports equal the
    frozen moesim reports; the exact solver refuses the same instances."""
    import sys
    sys.path.insert(0, __file__.rsplit("/", 1)[0] + "/golden")
    from make_golden_cfgs import baseline_cfgs
    _, meta = golden
    for key, want in meta["runs_baseline"].items():
        tname, rname = key.split("/")
        tr, info = traces[tname], meta["traces"][tname]
        over = dict(baseline_cfgs(info["N"]))[rname]
        res = P.calibrate([s.hidden for s in tr.steps])
        cfg = dali.ModelConfig(info["L"], info["N"], 0, info["k"], info["d"])
        t = dali.Trace(cfg, info["B"], info["phase"],
                       [dali.TokenStep(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                        for s in tr.steps], gate_params=dali.GateParams(tr.gates))
        sc = _sim_config(dali, rname, over, res)
        if over.get("prefetch_kind") == "statistical":
            sc.frequency_table = P.frequency_table([s.workloads for s in tr.steps])
        if "error" in want:
            with pytest.raises(dali.AssignmentError, match="exact solver limited"):
                dali.simulate_run(t, sc)
            continue
        rep = dali.simulate_run(t, sc).to_dict()
        rep.pop("spec")
        rep.pop("timelines")
        assert rep == want, key


def test_baseline_decision_logs_match_oracle(dali, traces):
    """Entry by entry incl. the LRU / toggle insertions the engine executes."""
    tr = traces["headline"]
    res = P.calibrate([s.hidden for s in tr.steps])
    steps = [D.StepInput(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
             for s in tr.steps]
    cfg = dali.ModelConfig(tr.L, tr.N, 0, tr.k, tr.d)
    t = dali.Trace(cfg, 32, "decode", [dali.TokenStep(s.token_index, s.tokens, s.workloads,
                                                      s.hidden, s.eos) for s in tr.steps],
                   gate_params=dali.GateParams(tr.gates))
    for pol, ins_d, ins_p in [("lru", False, True), ("workload", True, True),
                              ("score", True, False)]:
        dcfg = D.DriverConfig(tables=P.default_tables(non_moe_layer_time=3.0), prefetch_size=2,
                              residuals=res, cache_capacity=4, cache_policy=pol, w_size=4,
                              u_size=1, seed=3, insert_demand_fetched=ins_d,
                              insert_prefetched=ins_p)
        _, recs = D.run(steps, tr.gates, dcfg, tr.L, tr.N, tr.k)
        sc = dali.SimConfig(cost_model=dali.default_cost_model(non_moe_layer_time=3.0),
                            prefetch_kind="residual", prefetch_size=2,
                            residuals=dali.ResidualVectors(res), cache_policy=pol,
                            cache_capacity=4, w_size=4, u_size=1, seed=3,
                            insert_demand_fetched=ins_d, insert_prefetched=ins_p)
        got = dali.simulate_run(t, sc).decisions
        assert len(got) == len(recs)
        n_ins = 0
        for g, o in zip(got, recs):
            assert g["hits"] == o.lookups, (pol, o.step, o.layer)
            assert g["inserts"] == o.inserts, (pol, o.step, o.layer)
            assert g["event"] == o.event
            n_ins += len(o.inserts)
        assert n_ins > 0, pol


def test_single_instance_solvers_vs_oracle(dali):
    """beam_assign / optimal_assign / static_threshold_assign on random
    dyadic-time instances (reference conftest.py:36-58 style) == oracle."""
    rng = np.random.default_rng(41)
    for it in range(120):
        n = int(rng.integers(1, 14))
        w = rng.integers(0, 6, size=n).astype(np.int64)
        res = rng.random(n) < 0.3
        ct = rng.integers(1, 64, size=n) / 64.0
        gt = rng.integers(1, 64, size=n) / 64.0
        ct[w == 0] = 0.0
        gt[w == 0] = 0.0
        cap = None if rng.random() < 0.5 else int(rng.integers(0, 4))
        inst = dali.AssignmentInstance.from_times(ct, gt, resident=res, workloads=w,
                                                  gpu_capacity=cap)
        bw = int(rng.integers(1, 5))
        C, G = P.beam(w, res, ct, gt, cap, bw)
        a = dali.beam_assign(inst, bw)
        assert a.C.tolist() == C.tolist() and a.G.tolist() == G.tolist(), ("beam", it)
        C, G, nodes = P.optimal(w, res, ct, gt, cap)
        a, mk, nd = dali.optimal_assign_with_stats(inst)
        assert a.C.tolist() == C.tolist() and a.G.tolist() == G.tolist(), ("opt", it)
        assert nd == nodes, ("nodes", it)
        thr = None if it % 2 else float(rng.integers(0, 5))
        C, G = P.static_threshold(w, res, cap, thr)
        a = dali.static_threshold_assign(inst, thr)
        assert a.C.tolist() == C.tolist() and a.G.tolist() == G.tolist(), ("static", it)


def test_lru_lookup_and_force_insert(dali):
    st = dali.init_cache(0, 6, 2, 4, 1, policy="lru", seed=0)
    oc = P.new_cache(0, 6, 2, 4, 1, 0, policy="lru")
    for e in [0, 1, 2, 0, 3, 3, 4, 1, 0, 5]:
        assert dali.lookup(st, e) == P.lookup(oc, e)[0]
        assert st.on_gpu.tolist() == oc.on_gpu.tolist()
    for e in [2, 4, 5]:
        assert dali.force_insert(st, e) == P.force_insert(oc, e)
        assert st.on_gpu.tolist() == oc.on_gpu.tolist()
    ws = dali.init_cache(1, 8, 3, 2, 1, policy="workload", seed=2)
    ow = P.new_cache(1, 8, 3, 2, 1, 2)
    ws.scores = np.array([3.0, 1.0, 1.0, 0.0, 2.0, 5.0, 0.0, 4.0])
    ow.scores = ws.scores.copy()
    for e in range(8):
        assert dali.force_insert(ws, e) == P.force_insert(ow, e)
        assert ws.on_gpu.tolist() == ow.on_gpu.tolist()


def test_statistical_and_random_predictors(dali, traces):
    tr = traces["tiny_decode"]
    cfg = dali.ModelConfig(tr.L, tr.N, 0, tr.k, tr.d)
    t = dali.Trace(cfg, 1, "decode", [dali.TokenStep(s.token_index, s.tokens, s.workloads,
                                                     s.hidden, s.eos) for s in tr.steps])
    sp = dali.statistical_predictor(t)
    table = P.frequency_table([s.workloads for s in tr.steps])
    assert np.array_equal(sp.frequency_table, table)
    for l in range(tr.L - 1):
        d = dali.predict_next_layer(sp, None, None, tr.k, 3, l)
        assert d.prefetch_set.tolist() == P.stable_topk(table[l + 1].astype(float), 3).tolist()
    rp = dali.random_predictor(seed=9, n_experts=tr.N)
    rng = np.random.default_rng(9)
    for l in range(5):
        d = dali.predict_next_layer(rp, None, None, tr.k, 2, 0)
        perm = rng.permutation(tr.N)
        assert d.predicted_workloads.tolist() == perm.tolist()
        assert d.prefetch_set.tolist() == P.stable_topk(perm.astype(float), 2).tolist()
