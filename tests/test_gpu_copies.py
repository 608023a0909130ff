"""Engine copy plumbing through the C-ABI: dali_copy_mapped (kernel copy
over UVA), dali_copy_mapped2 (two ranges in one launch) and
dali_memcpy_async (copy-engine expert-block transfers) move exactly the
bytes asked for, tails included, in both directions."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def _needs_gpu():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("n0,n1", [(136, 32768), (1088, 16384), (16, 0), (0, 48), (4096 + 9, 7),
                                   (100_000, 300_000)])
def test_copy_mapped2_matches_two_copies(n0, n1):
    _needs_gpu()
    from paper_2602_03495_b200 import _lib
    g = torch.Generator().manual_seed(n0 + n1)
    s0 = torch.randint(0, 256, (max(n0, 1),), dtype=torch.uint8, generator=g).cuda()
    s1 = torch.randint(0, 256, (max(n1, 1),), dtype=torch.uint8, generator=g).cuda()
    d0 = torch.zeros(max(n0, 1) + 32, dtype=torch.uint8, pin_memory=True)
    d1 = torch.zeros(max(n1, 1) + 32, dtype=torch.uint8, pin_memory=True)
    st = torch.cuda.current_stream().cuda_stream
    _lib.call("dali_copy_mapped2", d0.data_ptr(), s0.data_ptr(), n0, d1.data_ptr(), s1.data_ptr(),
              n1, st)
    torch.cuda.synchronize()
    assert torch.equal(d0[:n0], s0[:n0].cpu()) and int(d0[n0:].sum()) == 0
    assert torch.equal(d1[:n1], s1[:n1].cpu()) and int(d1[n1:].sum()) == 0


def test_copy_mapped2_rejects_unaligned():
    _needs_gpu()
    from paper_2602_03495_b200 import _lib
    from paper_2602_03495_b200._lib import DaliCudaError
    s = torch.zeros(64, dtype=torch.uint8, device="cuda")
    d = torch.zeros(64, dtype=torch.uint8, pin_memory=True)
    with pytest.raises(DaliCudaError):
        _lib.call("dali_copy_mapped2", d.data_ptr() + 1, s.data_ptr(), 8, d.data_ptr(),
                  s.data_ptr(), 8, None)


@pytest.mark.parametrize("nbytes", [1, 4096, 8 * 1024 * 1024 + 3])
def test_memcpy_async_h2d_and_d2d(nbytes):
    _needs_gpu()
    from paper_2602_03495_b200 import _lib
    src = torch.randint(0, 256, (nbytes,), dtype=torch.uint8,
                        generator=torch.Generator().manual_seed(nbytes)).pin_memory()
    dst = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    dst2 = torch.zeros(nbytes, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    _lib.call("dali_memcpy_async", dst.data_ptr(), src.data_ptr(), nbytes, st.cuda_stream)
    _lib.call("dali_memcpy_async", dst2.data_ptr(), dst.data_ptr(), nbytes, st.cuda_stream)
    st.synchronize()
    assert torch.equal(dst.cpu(), src) and torch.equal(dst2.cpu(), src)
    _lib.call("dali_memcpy_async", dst.data_ptr(), src.data_ptr(), 0, st.cuda_stream)   # no-op
