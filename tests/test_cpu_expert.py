"""Native CPU expert worker (AVX-512 BF16) vs a torch fp32 reference -- runs on
the host, no GPU needed."""

import pytest
import torch

from oracle import model_cpu as M
from paper_2602_03495_b200 import _lib


def _has_bf16():
    try:
        return "avx512_bf16" in open("/proc/cpuinfo").read()
    except OSError:
        return False


@pytest.mark.skipif(not _has_bf16(), reason="host CPU lacks AVX512-BF16")
@pytest.mark.parametrize("d,f,R", [(256, 512, 1), (512, 1408, 3), (1024, 2048, 16),
                                   (256, 512, 21), (512, 1408, 64), (256, 512, 100),
                                   (1024, 2048, 130),
                                   # wide f: the AMX down projection runs in 2 / 7 k chunks
                                   (256, 14336, 40), (256, 14336, 130)])
def test_cpu_expert_matches_fp32_reference(d, f, R):
    g = torch.Generator().manual_seed(d + R)
    block = (torch.randn(3 * f * d, generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(R, d, generator=g).to(torch.bfloat16)
    y = torch.empty(R, d, dtype=torch.float32)
    _lib.call("dali_cpu_expert", block.data_ptr(), d, f, x.data_ptr(), R, y.data_ptr(), 4)
    ref = M.expert_forward(x.float(), block, d, f)
    torch.testing.assert_close(y, ref, rtol=2e-2, atol=2e-2 * ref.abs().max().item())


@pytest.mark.skipif(not _has_bf16(), reason="host CPU lacks AVX512-BF16")
@pytest.mark.parametrize("late_ms", [0.0, 5.0])
def test_cpu_expert_submit_wait_matches_sync(late_ms):
    """Asynchronous submission (workers start, the caller joins late and takes
    the remaining units) gives bit-identical rows to the synchronous call, for
    a layer's worth of experts with different row counts; a synchronous call
    while a job is in flight is refused."""
    import time

    import numpy as np
    d, f = 512, 1408
    g = torch.Generator().manual_seed(11)
    rows = [1, 3, 0, 16, 2]
    blocks = [(torch.randn(3 * f * d, generator=g) * 0.05).to(torch.bfloat16) for _ in rows]
    xs = [torch.randn(max(r, 1), d, generator=g).to(torch.bfloat16) for r in rows]
    ys = [torch.full((max(r, 1), d), float("nan")) for r in rows]
    refs = []
    for b, x, r in zip(blocks, xs, rows):
        y = torch.zeros(max(r, 1), d)
        _lib.call("dali_cpu_expert", b.data_ptr(), d, f, x.data_ptr(), r, y.data_ptr(), 4)
        refs.append(y)
    for _ in range(3):
        p = lambda ts: np.array([t.data_ptr() for t in ts], np.uint64)  # noqa: E731
        bp, xp, yp = p(blocks), p(xs), p(ys)
        rp = np.array(rows, np.int32)
        _lib.call("dali_cpu_expert_submit", len(rows), bp.ctypes.data, xp.ctypes.data,
                  rp.ctypes.data, yp.ctypes.data, d, f, 4)
        y1 = torch.empty(1, d)
        rc = _lib.load().dali_cpu_expert(blocks[0].data_ptr(), d, f, xs[0].data_ptr(), 1,
                                         y1.data_ptr(), 4)
        assert rc != 0                       # pool busy: refused, not corrupted
        time.sleep(late_ms / 1e3)
        _lib.call("dali_cpu_expert_wait")
        for r, y, ref in zip(rows, ys, refs):
            if r:
                assert torch.equal(y[:r], ref[:r])


@pytest.mark.skipif(not _has_bf16(), reason="host CPU lacks AVX512-BF16")
@pytest.mark.parametrize("d,f,R", [(256, 512, 17), (512, 1408, 40), (1024, 2048, 130),
                                   (4096, 1408, 64)])
def test_cpu_expert_prefill_rows_keep_fp32_outputs(d, f, R):
    """Prefill-sized batches (R > 16, the AMX-BF16 path when the host has it)
    have the decode kernel's rounding points: fp32 gate/up and down outputs,
    only the SwiGLU intermediate rounded to bf16 (the oneDNN path
    rounded all three).  Each row must equal the single-row AVX-512 result up
    to fp32 summation order and rare 1-ulp flips of the bf16 intermediate --
    far below one bf16 rounding of the output (2^-9 relative)."""
    g = torch.Generator().manual_seed(7 * d + R)
    block = (torch.randn(3 * f * d, generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(R, d, generator=g).to(torch.bfloat16)
    y = torch.empty(R, d, dtype=torch.float32)
    _lib.call("dali_cpu_expert", block.data_ptr(), d, f, x.data_ptr(), R, y.data_ptr(), 4)
    ref = torch.empty(R, d, dtype=torch.float32)
    for r in range(R):
        _lib.call("dali_cpu_expert", block.data_ptr(), d, f, x[r:r + 1].data_ptr(), 1,
                  ref[r:r + 1].data_ptr(), 4)
    err = (y - ref).abs()
    scale = ref.pow(2).mean(dim=1, keepdim=True).sqrt()
    assert float((err / scale).max()) < 2e-3, float((err / scale).max())
    # and the outputs are not bf16-rounded: most values carry more mantissa bits
    assert float((y != y.to(torch.bfloat16).float()).float().mean()) > 0.9


@pytest.mark.skipif(not _has_bf16(), reason="host CPU lacks AVX512-BF16")
def test_cpu_submit_layer_from_record_and_completion_word():
    """dali_cpu_submit_layer (launch-ahead decode): the experts the C vector
    marks, with rows from the offsets, run on the pool and give the rows
    dali_cpu_expert gives; the completion word receives the sequence number
    when the last unit ends (at once when no expert has rows); a prefill-sized
    expert starts nothing and leaves the word alone."""
    import ctypes as C

    import numpy as np

    d, f, N = 256, 512, 8
    g = torch.Generator().manual_seed(11)
    blocks = [(torch.randn(3 * f * d, generator=g) * 0.05).to(torch.bfloat16) for _ in range(N)]
    tab = np.array([b.data_ptr() for b in blocks], dtype=np.uint64)
    counts = np.array([1, 0, 2, 1, 0, 3, 1, 0], dtype=np.int32)
    offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    R = int(offs[-1])
    x = torch.randn(R, d, generator=g).to(torch.bfloat16)
    cmask = np.array([1, 1, 0, 1, 0, 1, 0, 0], dtype=np.int8)      # expert 1 has no rows
    flag = np.zeros(2, dtype=np.uint64)
    out = torch.full((R, d), 7.0, dtype=torch.float32)
    n = C.c_int32()
    _lib.call("dali_cpu_submit_layer", cmask.ctypes.data, offs.ctypes.data, N, tab.ctypes.data,
              x.data_ptr(), out.data_ptr(), d, f, 4, flag.ctypes.data, 41, C.byref(n))
    assert n.value == 3                                               # experts 0, 3, 5
    _lib.call("dali_cpu_expert_wait")
    assert int(flag[0]) == 41
    for e in range(N):
        r0, r1 = int(offs[e]), int(offs[e + 1])
        if r1 == r0:
            continue
        if cmask[e]:
            ref = torch.empty(r1 - r0, d, dtype=torch.float32)
            _lib.call("dali_cpu_expert", blocks[e].data_ptr(), d, f, x[r0:r1].data_ptr(),
                      r1 - r0, ref.data_ptr(), 4)
            assert torch.equal(out[r0:r1], ref), e
        else:
            assert bool((out[r0:r1] == 7.0).all()), e                # GPU experts' rows untouched
    # no CPU expert with rows: the word is stored at once, nothing to join
    zero = np.zeros(N, dtype=np.int8)
    _lib.call("dali_cpu_submit_layer", zero.ctypes.data, offs.ctypes.data, N, tab.ctypes.data,
              x.data_ptr(), out.data_ptr(), d, f, 4, flag.ctypes.data, 42, C.byref(n))
    assert n.value == 0 and int(flag[0]) == 42
    _lib.call("dali_cpu_expert_wait")
    # a prefill-sized expert (> 16 rows): nothing started, the word untouched
    big = np.array([0, 17] + [17] * (N - 1), dtype=np.int32)
    xb = torch.randn(int(big[-1]), d, generator=g).to(torch.bfloat16)
    outb = torch.empty(int(big[-1]), d, dtype=torch.float32)
    one = np.zeros(N, dtype=np.int8)
    one[0] = 1
    _lib.call("dali_cpu_submit_layer", one.ctypes.data, big.ctypes.data, N, tab.ctypes.data,
              xb.data_ptr(), outb.data_ptr(), d, f, 4, flag.ctypes.data, 43, C.byref(n))
    assert n.value == -1 and int(flag[0]) == 42
