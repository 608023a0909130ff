"""Deferred window replacements (EngineConfig.lazy_replace).

The workload-aware cache's window swaps are recorded, not copied at once: a
copy is issued when a later decision hits the slot (on the demand stream) or
in the background in next-use order, and a pending admission evicted again
before any read is never copied.  Execution only -- the decisions and the
bytes every FFN reads are the same -- so tokens, decision records and every
MoE layer output must be identical with the option on and off, and every
replacement the policy made is either copied or superseded.
"""
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("model,slots,pf,w,inflight", [("tiny", 2, 2, 2, 2),
                                                       ("tiny-shared", 3, 1, 2, 2),
                                                       ("tiny", 3, 1, 1, 0),
                                                       ("tiny-shared", 2, 2, 2, 0)])
def test_lazy_replace_identical(model, slots, pf, w, inflight):
    """inflight = 0 disables the background copies, so every replacement a
    hit needs is issued by the hit (the urgent path) and the rest are
    superseded or stay pending."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2602_03495_b200.cost_model import default_cost_model
    from paper_2602_03495_b200.engine import EngineConfig, build_engine
    cm = default_cost_model(non_moe_layer_time=3.0)
    g = torch.Generator().manual_seed(11)
    prompts = [torch.randint(0, 512, (1, 24), generator=g) for _ in range(2)]
    res = {}
    for lazy in (False, True):
        eng = build_engine(model, EngineConfig(cache_slots_per_layer=slots, prefetch_size=pf,
                                               w_size=w, seed=3, lazy_replace=lazy,
                                               repl_inflight=inflight, capture_moe_io=True),
                           seed=5, cost_model=cm, max_seq=128)
        out = []
        for p in prompts:                       # two requests: pending copies carry over
            toks, st = eng.generate(p, 40)
            torch.cuda.synchronize()
            out.append(dict(toks=toks.cpu(), st=st,
                            log=[(r["C"].tolist(), r["G"].tolist(), r["event"])
                                 for r in eng.policy.decision_log()],
                            io=[(s_, l_, xo.clone()) for (s_, l_, _, xo) in st.moe_io]))
        pending = sum(len(d) for d in eng._repl_pend)
        res[lazy] = (out, pending)
    (off, _), (on, pending) = res[False], res[True]
    n_off = n_on = n_urgent = 0
    for a, b in zip(off, on):
        assert torch.equal(a["toks"], b["toks"])
        assert a["log"] == b["log"]
        assert len(a["io"]) == len(b["io"])
        for x, y in zip(a["io"], b["io"]):
            assert x[:2] == y[:2] and torch.equal(x[2], y[2]), x[:2]
        n_off += a["st"].replace_copies
        n_on += b["st"].replace_copies + b["st"].replace_dropped
        n_urgent += b["st"].replace_urgent
    assert n_off > 0
    # stats are per request: every replacement copied, superseded or still pending
    assert n_on + pending == n_off, (n_on, pending, n_off)
    if inflight == 0:
        assert n_urgent > 0
