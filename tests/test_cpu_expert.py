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
                                   (1024, 2048, 130)])
def test_cpu_expert_matches_fp32_reference(d, f, R):
    g = torch.Generator().manual_seed(d + R)
    block = (torch.randn(3 * f * d, generator=g) * 0.05).to(torch.bfloat16)
    x = torch.randn(R, d, generator=g).to(torch.bfloat16)
    y = torch.empty(R, d, dtype=torch.float32)
    _lib.call("dali_cpu_expert", block.data_ptr(), d, f, x.data_ptr(), R, y.data_ptr(), 4)
    ref = M.expert_forward(x.float(), block, d, f)
    torch.testing.assert_close(y, ref, rtol=2e-2, atol=2e-2 * ref.abs().max().item())
