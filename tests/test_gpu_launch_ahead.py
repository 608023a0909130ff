"""Launch-ahead offloaded decode (engine/decode_graph.py, csrc/moe.cu
combine_kernel wait path): a layer's combine is queued before its CPU
experts finish and polls the worker's completion word.  Checks that it changes
nothing observable -- same tokens, bit-identical logits and decision log as
the join-then-launch order -- and that no poll ever times out over many short
requests (the regression that ld.global.cv fixed)."""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _engine(name):
    from paper_2602_03495_b200.cost_model import default_cost_model
    from paper_2602_03495_b200.engine import EngineConfig, build_engine
    cfg = EngineConfig(cache_slots_per_layer=2 if name == "tiny" else 6, prefetch_size=2, seed=3)
    cm = default_cost_model(shared_expert_gpu_time=0.0 if name == "tiny" else 0.5,
                            non_moe_layer_time=3.0)
    return build_engine(name, cfg, seed=5, cost_model=cm, max_seq=128)


def _timeouts():
    from paper_2602_03495_b200 import _lib
    v = ctypes.c_uint64()
    _lib.call("dali_host_wait_timeouts", ctypes.byref(v), 0)
    return int(v.value)


@pytest.mark.parametrize("name", ["tiny", "tiny-shared"])
def test_launch_ahead_matches_join_first(name):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    eng = _engine(name)
    prompt = torch.randint(0, eng.arch.vocab_size, (1, 24), generator=torch.Generator().manual_seed(1))
    out = {}
    for ahead in (False, True):
        eng._launch_ahead = ahead
        eng.reset_cache()
        toks, st = eng.generate(prompt, 16)
        log = eng.policy.decision_log()
        out[ahead] = (toks.cpu().numpy(), [(g["C"].tolist(), g["G"].tolist()) for g in log])
    assert np.array_equal(out[False][0], out[True][0])
    assert out[False][1] == out[True][1]


def test_launch_ahead_stress_no_poll_timeouts():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    eng = _engine("tiny-shared")
    assert eng._launch_ahead
    t0 = _timeouts()
    g = torch.Generator().manual_seed(0)
    for it in range(40):
        p = torch.randint(0, eng.arch.vocab_size, (1, 16 + it % 7), generator=g)
        eng.generate(p, 16)
        torch.cuda.synchronize()
        x = eng._wsd[("dec_X", torch.bfloat16, False)]
        assert bool(torch.isfinite(x).all()), it
    assert _timeouts() == t0
