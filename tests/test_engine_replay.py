"""Engine -> reference replay.

``tests/golden/make_engine_replay.py`` ran real requests through the B200
offloaded engine (from its seeded initial cache) and froze what the engine's
exporter wrote -- the ``moesim-trace-v1`` trace of the routed workloads and
captured gate inputs, the router and residual sidecars and the cost model the
engine decided with -- together with the engine's own RunReport-shaped report
and per-(step, layer) decisions.  Here the reference itself,
``moesim.simulate_run`` (simulator.py:318-522), replays those artifacts and
must reproduce the engine: the same initial residency, the same GPU expert
set in every layer of every step (from the reference's per-layer timelines,
simulator.py:456-468), the same virtual-clock latencies, and an equal report
(hit rates, prefetch accuracy, replacement events, PCIe accounting).

CPU only; needs the reference package (present in the build container at
/root/reference, or installed under baseline/_ref); skipped otherwise.
"""

import gzip
import json
import os
import shutil
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
FIX = os.path.join(HERE, "golden", "engine_replay")
CASES = ["tiny", "mixtral_L3", "qwen_L4_b2"]


def _moesim():
    for p in ("/root/reference/pkg/src", os.path.join(ROOT, "baseline", "_ref")):
        if os.path.isdir(os.path.join(p, "moesim")) and p not in sys.path:
            sys.path.insert(0, p)
    try:
        import moesim
        return moesim
    except ImportError:
        return None


moesim = _moesim()
pytestmark = pytest.mark.skipif(moesim is None, reason="reference moesim not importable here")


def _gunzip(src, dst):
    with gzip.open(src, "rb") as fi, open(dst, "wb") as fo:
        shutil.copyfileobj(fi, fo)
    return dst


def _replay(case, tmp_path):
    from moesim.cache import init_cache
    from moesim.cost_model import load_cost_model
    from moesim.simulator import SimConfig, simulate_run
    from moesim.trace import load_gate_params, load_residuals, load_trace
    base = os.path.join(FIX, case)
    eng = json.load(open(base + ".engine.json"))
    tr = load_trace(_gunzip(base + ".trace.jsonl.gz", tmp_path / "t.jsonl"))
    tr.gate_params = load_gate_params(_gunzip(base + ".gates.gz", tmp_path / "t.gates"))
    res = load_residuals(_gunzip(base + ".res.gz", tmp_path / "t.res"))
    sc = eng["sim_config"]
    cfg = SimConfig(cost_model=load_cost_model(base + ".cost.json"),
                    prefetch_kind=sc["prefetch_kind"], prefetch_size=sc["prefetch_size"],
                    residuals=res, cache_policy=sc["cache_policy"],
                    cache_capacity=sc["cache_capacity"], w_size=sc["w_size"],
                    u_size=sc["u_size"], seed=sc["seed"], keep_timelines=True)
    rep = simulate_run(tr, cfg).to_dict()
    return eng, tr, cfg, rep, init_cache


@pytest.mark.parametrize("case", CASES)
def test_reference_replays_engine_request(case, tmp_path):
    eng, tr, cfg, rep, init_cache = _replay(case, tmp_path)
    L, N = tr.model_config.num_layers, tr.model_config.num_routed_experts
    # 1. the engine started from the reference's seeded residency (cache.py:67-101)
    u = cfg.u_size if cfg.u_size is not None else \
        moesim.simulator.default_u_size(N, cfg.cache_capacity)
    for l in range(L):
        st = init_cache(l, N, cfg.cache_capacity, cfg.w_size, u, seed=cfg.seed)
        assert np.array_equal(np.asarray(st.on_gpu, dtype=int), eng["initial_on_gpu"][l]), l
    # 2. every (step, layer): GPU expert set and layer latency from the
    #    reference's timelines equal the engine's device decision records
    tl = rep["timelines"]
    dec = eng["decisions"]
    assert len(tl) == len(dec) == tr.num_steps * L
    for t, g in zip(tl, dec):
        assert t["layer"] == g["layer"]
        assert sorted(int(iv[2]) for iv in t["gpu_compute_intervals"]) == g["gpu"], g
        assert t["layer_latency"] == g["latency"], g
    # 3. the whole report (virtual clock, hit rates, prefetch accuracy,
    #    replacement log, PCIe accounting) -- exact equality
    ours = eng["report"]
    for key in rep:
        if key in ("spec", "timelines"):
            continue
        assert rep[key] == ours[key], key
    # the request exercised the DALI path: CPU and GPU experts, hits and swaps
    assert eng["cpu_expert_calls"] > 0 and eng["gpu_expert_calls"] > 0
    assert rep["replacement_events"], "no cache swap in the request"


def test_fixture_recipe_is_committed():
    assert os.path.exists(os.path.join(HERE, "golden", "make_engine_replay.py"))
    for c in CASES:
        for ext in (".trace.jsonl.gz", ".gates.gz", ".res.gz", ".cost.json", ".engine.json"):
            assert os.path.exists(os.path.join(FIX, c + ext)), c + ext
