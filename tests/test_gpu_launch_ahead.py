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


def test_sm_driven_h2d_copy_and_engine_option():
    """Opt-in SM-driven expert copies (EngineConfig.h2d_sm_ctas > 0,
    dali_copy_h2d_sm): byte-exact against the source for several CTA / unroll
    settings, and an engine using them for replacements and prefetches makes
    the same decisions and tokens as the copy-engine default."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2602_03495_b200 import _lib
    from paper_2602_03495_b200.cost_model import default_cost_model
    from paper_2602_03495_b200.engine import EngineConfig, build_engine
    src = torch.randint(0, 256, (3 << 20,), dtype=torch.uint8).pin_memory()
    st = torch.cuda.current_stream()
    for nctas in (1, 4, 8 + 64, 16 + 192):
        dst = torch.zeros(src.numel(), dtype=torch.uint8, device="cuda")
        _lib.call("dali_copy_h2d_sm", dst.data_ptr(), src.data_ptr(), src.numel(), nctas,
                  st.cuda_stream)
        torch.cuda.synchronize()
        assert torch.equal(dst.cpu(), src), nctas
    cm = default_cost_model(non_moe_layer_time=3.0)
    prompt = torch.randint(0, 512, (1, 20), generator=torch.Generator().manual_seed(3))
    outs = []
    for n in (0, 4):
        eng = build_engine("tiny", EngineConfig(cache_slots_per_layer=2, prefetch_size=2, seed=3,
                                                h2d_sm_ctas=n), seed=5, cost_model=cm, max_seq=96)
        toks, _ = eng.generate(prompt, 24)
        outs.append((toks.cpu(), [(r["C"].tolist(), r["G"].tolist(), r["event"])
                                  for r in eng.policy.decision_log()]))
    assert torch.equal(outs[0][0], outs[1][0])
    assert outs[0][1] == outs[1][1]
