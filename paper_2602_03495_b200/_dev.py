"""Device plumbing for the drop-in API: numpy <-> CUDA tensors, stream handle.

torch is used only for device memory and streams.  Every function that
launches a kernel calls ``require_cuda`` first: there is no CPU path.
"""

from __future__ import annotations

import numpy as np
import torch

from .errors import MoesimError


class NoDeviceError(MoesimError):
    module = "cuda"


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise NoDeviceError("a CUDA device (B200, sm_100a) is required; the DALI hot path "
                            "has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def to_dev(a, dtype: torch.dtype) -> torch.Tensor:
    """numpy / tensor -> contiguous CUDA tensor of ``dtype``."""
    dev = require_cuda()
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    return torch.from_numpy(arr).to(device=dev, dtype=dtype).contiguous()


def ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else int(t.data_ptr())


def empty(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.empty(shape, dtype=dtype, device=require_cuda())


def zeros(shape, dtype: torch.dtype) -> torch.Tensor:
    return torch.zeros(shape, dtype=dtype, device=require_cuda())


def bf16_bits(t: torch.Tensor) -> torch.Tensor:
    """View a bf16 CUDA tensor as its raw uint16 bits (int16 storage)."""
    assert t.dtype == torch.bfloat16
    return t.contiguous().view(torch.int16)
