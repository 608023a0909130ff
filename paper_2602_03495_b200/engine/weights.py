"""Random-init weights for the inference engine.

Dense weights (embeddings, attention, norms, routers, LM head) live in HBM.
Routed experts live in one page-locked host store (``dali_host_alloc``),
one contiguous block per (layer, expert) -- the unit the H2D copy stream
moves into an HBM slot and the CPU worker computes on:

    block(l, e) = [ W13 (2f, d) | W2 (d, f) ]  bf16
    W13 rows [128b, 128b+64) = gate rows [64b, 64b+64); next 64 = up rows

In ``resident`` mode (the all-resident roofline reference) the same blocks
are kept in HBM instead.  All tensors are produced on the GPU by the
counter-hash init kernel (``dali_init_uniform_bf16``), so any tensor can be
regenerated bit-identically from (seed, name); routers follow the
reference generator's skew (normal * 0.4/sqrt(d) * permuted column scales
linspace(0.15, 1.85, N), trace.py:308-311).
"""

from __future__ import annotations

import ctypes as C
import math
import os

import numpy as np
import torch

from .. import _lib
from .arch import MoEArch

KIND_EMBED, KIND_LMHEAD, KIND_QKV, KIND_O, KIND_W13, KIND_W2 = 1, 2, 3, 4, 5, 6
KIND_SH13, KIND_SH2, KIND_SHGATE = 7, 8, 9


def tensor_seed(seed: int, kind: int, layer: int, index: int) -> int:
    return ((seed * 1000003 + kind) * 4099 + layer) * 65537 + index


def init_uniform_(t: torch.Tensor, seed: int, std: float, stream=None) -> torch.Tensor:
    """Fill a bf16 CUDA tensor with the counter-hash uniform init."""
    assert t.dtype == torch.bfloat16 and t.is_cuda and t.is_contiguous()
    s = stream if stream is not None else torch.cuda.current_stream()
    _lib.call("dali_init_uniform_bf16", t.data_ptr(), t.numel(), seed & (2 ** 64 - 1), 0,
              float(std), int(s.cuda_stream))
    return t


def router_weights(arch: MoEArch, seed: int, layer: int) -> np.ndarray:
    """Skewed router (d, N) in the reference generator's style, as fp64."""
    rng = np.random.default_rng([seed, 17, layer])
    d, N = arch.hidden_dim, arch.num_experts
    base = rng.normal(size=(d, N)) * (0.4 / math.sqrt(d))
    scale = rng.permutation(np.linspace(0.15, 1.85, N))
    return base * scale[None, :]


H2D_SM_CTAS = int(os.environ.get("DALI_H2D_SM_CTAS", "0"))


def h2d_block(dst: torch.Tensor, src: torch.Tensor, stream: torch.cuda.Stream,
              nctas: int = H2D_SM_CTAS) -> None:
    """Expert-block host->device copy from the pinned store on ``stream``.
    nctas = 0 (default): copy engine.  nctas > 0: a few SMs read the mapped
    pinned block (dali_copy_h2d_sm) with a bounded number of bytes in flight
    and pause in the decode chain's PCIe quiet window, so the decode path's
    small PCIe transfers (decision mirrors, pointer tables, CPU-expert rows)
    are not queued behind the copy engine's deep read queue: +40-50 us each
    under copy-engine DMA, ~0 with the SM copy (tools/pcie_latency_probe.py,
    profiles/r02_pcie_latency_probe.log).  End to end it lost: the SM copy
    moves 45-49 instead of 54 GB/s, the replacement queue backs up and cache
    hits wait on in-flight copies ("Tried and rejected")."""
    nbytes = src.numel() * src.element_size()
    if nctas > 0 and not (src.data_ptr() | dst.data_ptr() | nbytes) & 15:
        _lib.call("dali_copy_h2d_sm", dst.data_ptr(), src.data_ptr(), nbytes, int(nctas),
                  stream.cuda_stream)
    else:
        # copy engine, straight through the C-ABI: a torch.cuda.stream context
        # around Tensor.copy_ costs ~40 us of host time per block
        _lib.call("dali_memcpy_async", dst.data_ptr(), src.data_ptr(), nbytes, stream.cuda_stream)


class HostStore:
    """Page-locked expert store (exact size, huge pages, parallel first touch)."""

    def __init__(self, nbytes: int, nthreads: int = 16, shared: str | None = None,
                 fd: int = -1, owner_pid: int = 0):
        """shared=None: private store; "create": node-shared memfd store (its
        fd/pid go to the other local ranks); "open": map the owner's store."""
        self.nbytes = int(nbytes)
        p = C.c_void_p()
        self.fd, self.owner_pid = fd, owner_pid
        if shared is None:
            _lib.call("dali_host_alloc", self.nbytes, int(nthreads), C.byref(p))
        else:
            cfd = C.c_int32(fd)
            _lib.call("dali_host_alloc_shared", self.nbytes, int(nthreads),
                      int(shared == "create"), C.byref(cfd), int(owner_pid), C.byref(p))
            self.fd = int(cfd.value)
            if shared == "create":
                self.owner_pid = os.getpid()
        self.ptr = int(p.value)
        arr = np.ctypeslib.as_array((C.c_uint8 * self.nbytes).from_address(self.ptr))
        self.bytes = torch.from_numpy(arr)           # uint8 CPU view (pinned)

    def close(self):
        if self.ptr:
            _lib.load().dali_host_free(self.ptr, self.nbytes)
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ModelWeights:
    def __init__(self, arch: MoEArch, seed: int = 0, device="cuda", resident: bool = False,
                 host_threads: int = 16, host_store: "HostStore | None" = None,
                 fill_experts: bool = True, experts: list | None = None):
        """experts: the routed experts this process holds (expert-parallel
        shard); default all.  Block (l, j) of the store is expert experts[j];
        values depend only on (seed, layer, global expert id)."""
        self.arch, self.seed = arch, seed
        a = arch
        dev = torch.device(device)
        d, H, KV, hd = a.hidden_dim, a.num_heads, a.num_kv_heads, a.head_dim
        bf = torch.bfloat16

        def w(shape, kind, layer, idx, std):
            t = torch.empty(shape, dtype=bf, device=dev)
            return init_uniform_(t, tensor_seed(seed, kind, layer, idx), std)

        self.embed = w((a.vocab_size, d), KIND_EMBED, 0, 0, 1.0)
        self.lm_head = w((a.vocab_size, d), KIND_LMHEAD, 0, 0, 1.0 / math.sqrt(d))
        self.final_norm = torch.ones(d, dtype=bf, device=dev)
        self.attn_norm = [torch.ones(d, dtype=bf, device=dev) for _ in range(a.num_layers)]
        self.moe_norm = [torch.ones(d, dtype=bf, device=dev) for _ in range(a.num_layers)]
        self.wqkv = [w(((H + 2 * KV) * hd, d), KIND_QKV, l, 0, 1.0 / math.sqrt(d))
                     for l in range(a.num_layers)]
        self.wo = [w((d, H * hd), KIND_O, l, 0, 1.0 / math.sqrt(H * hd))
                   for l in range(a.num_layers)]
        self.router64 = [router_weights(a, seed, l) for l in range(a.num_layers)]
        # shared expert(s): one dense SwiGLU block per layer, always resident in HBM
        self.shared = []
        self.shared_gate = []
        if a.num_shared_experts > 0:
            fs = a.shared_ffn_dim
            for l in range(a.num_layers):
                blk = torch.empty((3 * fs * d,), dtype=bf, device=dev)
                init_uniform_(blk[:2 * fs * d], tensor_seed(seed, KIND_SH13, l, 0), 1.0 / math.sqrt(d))
                init_uniform_(blk[2 * fs * d:], tensor_seed(seed, KIND_SH2, l, 0), 1.0 / math.sqrt(fs))
                self.shared.append(blk)
                if a.shared_gate:
                    self.shared_gate.append(w((1, d), KIND_SHGATE, l, 0, 1.0 / math.sqrt(d)))
        self.router = torch.stack([torch.from_numpy(r).to(bf) for r in self.router64]).to(dev)
        # squared router column norms (L, N) f32: the certified routing kernel's
        # error bound (csrc/route_guard.cu), computed once
        self.router_norm2 = self.router.float().square().sum(dim=1).contiguous()

        # routed experts
        self.resident = resident
        self.experts = list(range(a.num_experts)) if experts is None else list(experts)
        self.n_local = len(self.experts)
        L, N, E = a.num_layers, self.n_local, a.expert_elems
        self.expert_bytes = a.expert_bytes
        if resident:
            self.dev_store = torch.empty((L * N * E,), dtype=bf, device=dev)
            self.host = None
        else:
            self.dev_store = None
            self.host = host_store or HostStore(L * N * a.expert_bytes, host_threads)
            if self.host.nbytes != L * N * a.expert_bytes:
                raise ValueError("host store size does not match the architecture")
        if resident or fill_experts:
            stage = torch.empty((E,), dtype=bf, device=dev)
            for l in range(L):
                for e in range(N):
                    dst = self.expert_dev(l, e) if resident else stage
                    self.init_expert(l, e, dst)
                    if not resident:
                        self.expert_host(l, e).copy_(stage)   # D2H into the pinned store
        torch.cuda.synchronize()

    def init_expert(self, l: int, e: int, out: torch.Tensor) -> torch.Tensor:
        a = self.arch
        n13 = 2 * a.ffn_dim * a.hidden_dim
        ge = self.experts[e]              # global expert id -> seed
        init_uniform_(out[:n13], tensor_seed(self.seed, KIND_W13, l, ge), 1.0 / math.sqrt(a.hidden_dim))
        init_uniform_(out[n13:], tensor_seed(self.seed, KIND_W2, l, ge), 1.0 / math.sqrt(a.ffn_dim))
        return out

    def expert_index(self, l: int, e: int) -> int:
        return l * self.n_local + e

    def expert_host(self, l: int, e: int) -> torch.Tensor:
        """bf16 CPU view of block (l, e) in the pinned store."""
        off = self.expert_index(l, e) * self.expert_bytes
        return self.host.bytes[off:off + self.expert_bytes].view(torch.bfloat16)

    def expert_host_ptr(self, l: int, e: int) -> int:
        return self.host.ptr + self.expert_index(l, e) * self.expert_bytes

    def expert_dev(self, l: int, e: int) -> torch.Tensor:
        E = self.arch.expert_elems
        i = self.expert_index(l, e)
        return self.dev_store[i * E:(i + 1) * E]

    def split_expert(self, block: torch.Tensor):
        """(W13 (2f, d), W2 (d, f)) views of one block."""
        a = self.arch
        n13 = 2 * a.ffn_dim * a.hidden_dim
        return (block[:n13].view(2 * a.ffn_dim, a.hidden_dim),
                block[n13:].view(a.hidden_dim, a.ffn_dim))
