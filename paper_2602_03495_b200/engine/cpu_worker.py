"""Host worker for CPU-assigned experts (DALI hybrid execution, PAPER.md
section 4: experts the greedy assignment places on the CPU run there).

Decode-sized batches (<= NATIVE_MAX_ROWS tokens per expert) use the native
AVX-512 BF16 weight-streaming kernel in libdali (``dali_cpu_expert``), which
reads the pinned expert block once at host-DRAM bandwidth; larger batches
(prefill) are compute-heavy and go to oneDNN's AMX-BF16 GEMM through torch.

Rounding points.  The native kernel, like the GPU tcgen05 kernel, keeps the
gate/up and down projections in fp32 accumulators and rounds only the SwiGLU
intermediate to bf16.  torch's CPU bf16 GEMM has no fp32-output variant
(``mm(..., out_dtype=float32)`` is CUDA-only in this torch), so on the
oneDNN path the gate/up outputs and the down-projection output are also
rounded to bf16 (two extra roundings, each <= 2^-9 relative per element).
A prefill row therefore differs at bf16-rounding level depending on whether
the policy puts its expert on the CPU or the GPU; the engine's numeric parity
tests (tolerance rtol 2e-2 per element, tests/test_gpu_engine.py) cover both
placements.  Decode (<= 16 rows per expert) always takes the native path.
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
    if n <= NATIVE_MAX_ROWS:
        xc = x.contiguous()
        _lib.call("dali_cpu_expert", block.data_ptr(), d, f, xc.data_ptr(), n, out.data_ptr(),
                  threads)
        return out
    W13 = block[:2 * f * d].view(2 * f, d)
    W2 = block[2 * f * d:].view(d, f)
    gu = (x @ W13.t()).view(n, f // 64, 2, 64)
    g = gu[:, :, 0, :].reshape(n, f).float()
    u = gu[:, :, 1, :].reshape(n, f).float()
    act = (torch.nn.functional.silu(g) * u).to(torch.bfloat16)
    out.copy_((act @ W2.t()).float())
    return out
