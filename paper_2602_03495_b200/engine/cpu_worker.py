"""Host worker for CPU-assigned experts (DALI hybrid execution, PAPER.md
section 4: experts the greedy assignment places on the CPU run there).

Every batch goes to the native worker in libdali (``dali_cpu_expert``):
decode-sized batches (<= NATIVE_MAX_ROWS tokens per expert) to the AVX-512
BF16 weight-streaming kernel, which reads the pinned expert block once at
host-DRAM bandwidth; prefill-sized batches to the AMX-BF16 tile kernel (on a
host without AMX, to the AVX-512 kernel 16 rows at a time).

Rounding points.  All of them, like the GPU tcgen05 kernel, keep the gate/up
and down projections in fp32 accumulators, round only the SwiGLU
intermediate to bf16, and return fp32 rows -- so a row's numerics do not
depend on whether the policy placed its expert on the CPU or the GPU.
(Round 1 sent prefill batches to torch's oneDNN bf16 GEMM, which also
rounds the gate/up and down outputs to bf16; the AMX kernel replaced it and
is faster on the GPU boxes' hosts, tools/cpu_prefill_ab.py.)
"""

from __future__ import annotations

import torch

from .. import _lib

NATIVE_MAX_ROWS = 16


def cpu_expert_rows(block: torch.Tensor, x: torch.Tensor, d: int, f: int, threads: int,
                    out: torch.Tensor | None = None) -> torch.Tensor:
    """SwiGLU of rows x (n, d) bf16 with expert block (bf16, W13|W2 layout)
    -> (n, d) f32 (written into ``out`` when given)."""
    n = x.shape[0]
    if out is None:
        out = torch.empty((n, d), dtype=torch.float32)
    xc = x.contiguous()
    _lib.call("dali_cpu_expert", block.data_ptr(), d, f, xc.data_ptr(), n, out.data_ptr(),
              threads)
    return out
