"""Reference-format artifacts: trace / gates / residual sidecars written by the
B200 package round-trip through its own loader and -- when the reference is
present in this (build) container -- load in ``moesim`` and replay to the same
report as the oracle driver."""

import os
import sys

import numpy as np
import pytest

from oracle import driver as D
from oracle import policy as P
from paper_2602_03495_b200 import trace as T


def _trace():
    tr = P.synth_trace(3, 8, 2, 32, 2, 10, locality=0.9, drift_scale=0.4, noise_scale=0.08,
                       seed=4)
    cfg = T.ModelConfig(3, 8, 0, 2, 32)
    steps = [T.TokenStep(s.token_index, s.tokens, s.workloads, s.hidden, s.eos) for s in tr.steps]
    return tr, T.Trace(cfg, 2, "decode", steps, generator_seed=4,
                       gate_params=T.GateParams(tr.gates))


def test_trace_roundtrip(tmp_path):
    _, tr = _trace()
    p = tmp_path / "t.jsonl"
    T.save_trace(tr, p)
    back = T.load_trace(p)
    assert back.model_config == tr.model_config and back.num_steps == tr.num_steps
    for a, b in zip(tr.steps, back.steps):
        assert np.array_equal(a.workloads, b.workloads) and np.array_equal(a.hidden, b.hidden)
        assert a.eos == b.eos and a.token_index == b.token_index
    bad = tmp_path / "bad.jsonl"
    bad.write_text('{"format": "nope"}\n')
    with pytest.raises(T.TraceError):
        T.load_trace(bad)


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"),
                    reason="reference only present in the build container")
def test_reference_replays_our_artifacts(tmp_path):
    sys.path.insert(0, "/root/reference/pkg/src")
    import moesim
    from moesim.trace import load_gate_params
    raw, tr = _trace()
    T.save_trace(tr, tmp_path / "t.jsonl")
    T.save_gate_params(tr.gate_params, tmp_path / "t.gates")
    res = P.calibrate([s.hidden for s in raw.steps])
    T.save_residuals(T.ResidualVectors(res), tmp_path / "t.res")
    mt = moesim.load_trace(tmp_path / "t.jsonl")
    mt.gate_params = load_gate_params(tmp_path / "t.gates")
    mres = moesim.trace.load_residuals(tmp_path / "t.res")
    cfg = moesim.SimConfig(cost_model=moesim.default_cost_model(non_moe_layer_time=3.0),
                           prefetch_kind="residual", prefetch_size=1, residuals=mres,
                           cache_policy="workload", cache_capacity=2, w_size=4, seed=3)
    ref = moesim.simulate_run(mt, cfg).to_dict()
    dcfg = D.DriverConfig(tables=P.default_tables(non_moe_layer_time=3.0), prefetch_size=1,
                          residuals=res, cache_capacity=2, w_size=4, seed=3)
    ours, _ = D.run([D.StepInput(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                     for s in raw.steps], raw.gates, dcfg, 3, 8, 2)
    for k in ours:
        assert ref[k] == ours[k], k
