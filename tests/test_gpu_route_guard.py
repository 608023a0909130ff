"""GPU parity of the certified-margin bf16 routing kernel (csrc/route_guard.cu).

The kernel ranks fp32 logits and recomputes in fp64 every row whose k+1
leading logits are not separated by the rigorous summation-error bound.  The
bar is the reference's: top-k indices and workloads bit-exact against fp64
gating (reference trace.py:236-265, restated in oracle/policy.py:route) on
the same bf16-representable values, including near-ties, exact ties, the
residual-shifted prediction input (prefetch.py:127-136) and ragged token
counts around the decode/prefill switch (T = 16 / 17).
"""

import numpy as np
import pytest

from oracle import policy as P

pytestmark = pytest.mark.gpu

SHAPES = [(256, 8, 2), (4096, 8, 2), (2048, 60, 4), (2048, 64, 6), (6144, 8, 2), (256, 16, 4)]
TOKENS = [1, 2, 3, 5, 8, 16, 17, 33, 100, 512]


@pytest.fixture(scope="module")
def lib():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2602_03495_b200 import _lib
    _lib.load()
    yield _lib
    _lib.call("dali_route_guard_scale", 1.0)


def _inputs(T, d, N, seed):
    import torch
    g = torch.Generator().manual_seed(seed)
    h = torch.randn(T, d, generator=g).to(torch.bfloat16)
    w = (torch.randn(d, N, generator=g) * 0.4 / d ** 0.5 *
         torch.linspace(0.15, 1.85, N)[torch.randperm(N, generator=g)]).to(torch.bfloat16)
    return h, w


def _route(h, w, k, res=None, renorm=True):
    from paper_2602_03495_b200.trace import route_device
    r = None if res is None else __import__("torch").from_numpy(res).cuda()
    idx, wts, wl = route_device(h.cuda(), w.cuda(), k, residual=r, renorm=renorm)
    return idx.cpu().numpy(), wts.cpu().numpy(), wl.cpu().numpy()


def _oracle(h, w, k, res=None):
    x = h.double().numpy()
    if res is not None:
        x = x + res[None, :]
    return P.route(x, w.double().numpy(), k)


@pytest.mark.parametrize("d,N,k", SHAPES)
def test_guarded_route_matches_fp64_oracle(lib, d, N, k):
    for T in TOKENS:
        h, w = _inputs(T, d, N, seed=T * 7 + N)
        idx, wts, wl = _route(h, w, k)
        o_idx, o_sc, o_wl = _oracle(h, w, k)
        assert np.array_equal(idx, o_idx), (T, d, N)
        assert np.array_equal(wl, o_wl), (T, d, N)
        ref_w = o_sc / o_sc.sum(axis=1, keepdims=True)
        np.testing.assert_allclose(wts, ref_w, rtol=2e-6, atol=1e-7)


@pytest.mark.parametrize("d,N,k", [(4096, 8, 2), (2048, 64, 6), (2048, 60, 4)])
def test_guarded_route_residual_shift(lib, d, N, k):
    """Prediction input: hidden + residual in fp64 (not bf16-representable)."""
    rng = np.random.default_rng(d + N)
    res = rng.normal(size=d) * 0.1
    for T in (1, 4, 16, 64, 512):
        h, w = _inputs(T, d, N, seed=T + 3)
        _, _, wl = _route(h, w, k, res=res)
        _, _, o_wl = _oracle(h, w, k, res=res)
        assert np.array_equal(wl, o_wl), (T, d, N)


def test_forced_fp64_recompute_equals_certified_path(lib):
    """scale < 0: every row takes the fp64 recompute; indices, workloads and
    (to fp32 rounding) weights are unchanged and every row counts as a fire."""
    for (d, N, k) in [(4096, 8, 2), (2048, 64, 6)]:
        for T in (1, 16, 300):
            h, w = _inputs(T, d, N, seed=11 * T)
            a = _route(h, w, k)
            lib.route_fire_count(reset=True)
            lib.call("dali_route_guard_scale", -1.0)
            try:
                b = _route(h, w, k)
            finally:
                lib.call("dali_route_guard_scale", 1.0)
            fires, rows = lib.route_fire_count(reset=True)
            assert fires == rows == T
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])
            np.testing.assert_allclose(a[1], b[1], rtol=2e-6)


def test_near_ties_fire_and_match_fp64(lib):
    """Adversarial rows: the top two experts' logits differ by far less than
    the fp32 error bound (one bf16 ulp of one weight times a tiny input), or
    tie exactly.  The guard must fire on them and the fp64 recompute must
    reproduce the reference ranks (ties to the lower index)."""
    import torch
    for (d, N, k) in [(4096, 8, 2), (2048, 64, 6), (2048, 60, 4)]:
        T = 40
        h, w = _inputs(T, d, N, seed=5)
        w = w.clone()
        # experts 3 and 4 dominate; 4 = 3 except one weight nudged by 1 ulp
        base = w[:, 3].float() + 0.5 / d ** 0.5
        w[:, 3] = base.to(torch.bfloat16)
        w[:, 4] = w[:, 3]
        w[7, 4] = torch.tensor(w[7, 4].float().item() * (1 + 2 ** -7)).to(torch.bfloat16)
        h = (h.float().abs() + 0.01).to(torch.bfloat16)             # dominant pair on top
        h[:, 7] = torch.tensor(2.0 ** -20).to(torch.bfloat16)       # tiny gap
        h[::2, 7] = torch.tensor(0.0).to(torch.bfloat16)            # exact tie on even rows
        lib.route_fire_count(reset=True)
        idx, _, wl = _route(h, w, k)
        fires, rows = lib.route_fire_count(reset=True)
        o_idx, _, o_wl = _oracle(h, w, k)
        assert np.array_equal(idx, o_idx), (d, N)
        assert np.array_equal(wl, o_wl)
        assert rows == T and fires >= T // 2, (fires, rows)
        # even rows tie exactly -> the lower index leads; odd rows differ by ~1e-8
        assert (o_idx[::2, 0] == 3).all() and (o_idx[::2, 1] == 4).all()
        assert set(o_idx[1::2, :2].ravel().tolist()) == {3, 4}


def test_fire_rate_on_realistic_inputs(lib):
    """On skewed routers (the reference generator's style) the certified
    margin leaves few rows to the fp64 recompute."""
    for (d, N, k) in [(4096, 8, 2), (2048, 64, 6), (2048, 60, 4)]:
        h, w = _inputs(2048, d, N, seed=9)
        lib.route_fire_count(reset=True)
        _route(h, w, k)
        fires, rows = lib.route_fire_count(reset=True)
        assert rows == 2048
        assert fires < 0.05 * rows, (d, N, fires)


@pytest.mark.parametrize("d,N,k", [(4096, 8, 2), (2048, 64, 6), (2048, 60, 4), (256, 8, 2)])
@pytest.mark.parametrize("force", [False, True])
def test_route_plan_fused_matches_separate(lib, d, N, k, force):
    """dali_route_plan_bf16 (routing, plan and permute in one launch for
    decode batches) == dali_route_bf16 + dali_moe_plan_permute, every output
    bit for bit, for T = 1..16 and the separate-launch fallback (T = 17, 33);
    force=True sends every row through the fp64 recompute first."""
    import torch
    from paper_2602_03495_b200.trace import gate_norm2
    lib.call("dali_route_guard_scale", -1.0 if force else 1.0)
    try:
        for T in (1, 2, 3, 5, 8, 16, 17, 33):
            h, w = _inputs(T, d, N, seed=T * 13 + N)
            h, w = h.cuda(), w.cuda()
            n2 = gate_norm2(w)
            sp = torch.cuda.current_stream().cuda_stream

            def outs():
                return (torch.full((T, k), -7, dtype=torch.int32, device="cuda"),
                        torch.zeros((T, k), dtype=torch.float32, device="cuda"),
                        torch.zeros((N,), dtype=torch.int64, device="cuda"),
                        torch.full((N + 1,), -7, dtype=torch.int32, device="cuda"),
                        torch.full((T * k,), -7, dtype=torch.int32, device="cuda"),
                        torch.full((T, k), -7, dtype=torch.int32, device="cuda"),
                        torch.zeros((T * k, d), dtype=torch.bfloat16, device="cuda"))
            a = outs()
            lib.call("dali_route_bf16", h.data_ptr(), None, w.data_ptr(), n2.data_ptr(), T, d, N,
                     k, 1, a[0].data_ptr(), a[1].data_ptr(), a[2].data_ptr(), sp)
            lib.call("dali_moe_plan_permute", a[0].data_ptr(), T, k, N, h.data_ptr(), d,
                     a[3].data_ptr(), a[4].data_ptr(), a[5].data_ptr(), a[6].data_ptr(), sp)
            b = outs()
            lib.call("dali_route_plan_bf16", h.data_ptr(), w.data_ptr(), n2.data_ptr(), T, d, N,
                     k, 1, *[t.data_ptr() for t in b], sp)
            torch.cuda.synchronize()
            for x_, y_ in zip(a, b):
                assert torch.equal(x_, y_), (T, d, N, k)
    finally:
        lib.call("dali_route_guard_scale", 1.0)


@pytest.mark.parametrize("d,N,k", [(4096, 8, 2), (2048, 64, 6), (2048, 60, 4), (6144, 8, 2),
                                   (256, 16, 4), (1024, 32, 4)])
def test_prefill_kernel_matches_chunked_kernel_and_oracle(lib, d, N, k):
    """T > 16 with N <= 64: the fixed-geometry prefill kernel (4..32 tokens
    per CTA, fp32 operand tiles; dali_route_prefill_variant(2) forces it at
    every T) against the round-1 d-chunked kernel (variant 1).  Indices and workloads equal each other
    and the fp64 oracle, weights to fp32 rounding, at every token-tile size;
    the forced-fp64 path too."""
    import torch
    for T in (17, 100, 300, 700, 1300, 2100, 4096):
        h, w = _inputs(T, d, N, seed=T * 3 + d + N)
        res = None
        if T == 700:
            res = np.random.default_rng(T).normal(size=d) * 0.1
        lib.call("dali_route_prefill_variant", 2)
        try:
            new = _route(h, w, k, res=res)
            lib.call("dali_route_prefill_variant", 1)
            old = _route(h, w, k, res=res)
        finally:
            lib.call("dali_route_prefill_variant", 0)
        o_idx, o_sc, o_wl = _oracle(h, w, k, res=res)
        assert np.array_equal(new[0], o_idx), (T, d, N)
        assert np.array_equal(new[2], o_wl), (T, d, N)
        assert np.array_equal(new[0], old[0]) and np.array_equal(new[2], old[2])
        np.testing.assert_allclose(new[1], old[1], rtol=2e-6, atol=1e-7)
        if T in (100, 1300):
            lib.route_fire_count(reset=True)
            lib.call("dali_route_guard_scale", -1.0)
            lib.call("dali_route_prefill_variant", 2)
            try:
                f = _route(h, w, k, res=res)
            finally:
                lib.call("dali_route_guard_scale", 1.0)
                lib.call("dali_route_prefill_variant", 0)
            fires, rows = lib.route_fire_count(reset=True)
            assert fires == rows == T
            assert np.array_equal(f[0], o_idx) and np.array_equal(f[2], o_wl)
            np.testing.assert_allclose(f[1], new[1], rtol=2e-6, atol=1e-7)
    torch.cuda.synchronize()
