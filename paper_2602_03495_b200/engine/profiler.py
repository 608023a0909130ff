"""Warm-up profiler: measure this box's cost model.

Greedy decisions are only as good as t_cpu / t_gpu / trans_time measured on
the machine that runs them ("warm-up profiling").  The
profile samples power-of-two workloads and quantises every time to the
2^-12 ms grid, which makes all interpolated times and lane sums exact in
fp64 (cost_model.quantize_ms) -- so the device policy kernel, the host
report and the CPU oracle agree bit-for-bit regardless of summation order.
Output is a reference-format cost-model JSON (cost_model.py:158-179).
"""

from __future__ import annotations

import os
import statistics
import time

import numpy as np
import torch

from .. import _lib
from ..cost_model import CostModel, fit_cost_model, quantize_ms
from .arch import MoEArch
from .cpu_worker import NATIVE_MAX_ROWS, cpu_expert_rows
from .offload import ffn_splits
from .weights import h2d_block


def _cpu_expert(h: torch.Tensor, blk: torch.Tensor, d: int, f: int, threads: int):
    return cpu_expert_rows(blk, h, d, f, threads)


def _monotone(samples):
    out, best = [], 0.0
    for w, ms in samples:
        best = max(best, ms)
        out.append((w, best))
    return out


def profile_cost_model(arch: MoEArch, weights, max_w: int = 1024, reps: int = 3,
                       non_moe_ms: float | None = None, log=None, tc: bool = True,
                       threads: int | None = None,
                       contended_from_rows: int | None = None,
                       warmup_s: float = 0.6, h2d_ctas: int = 0) -> CostModel:
    dev = torch.device("cuda", torch.cuda.current_device())
    d, f, N = arch.hidden_dim, arch.ffn_dim, arch.num_experts
    ws = [1 << i for i in range(0, 32) if (1 << i) <= max_w]
    # CPU lane: SwiGLU of w tokens on the host worker over the pinned store
    # cycle over distinct expert blocks (as the engine does: every call streams
    # a block that is not in any cache level) and take the median
    n_blk = min(N, 8)
    if weights.host is not None:
        blks = [weights.expert_host(0, e) for e in range(n_blk)]
    else:
        blks = [weights.expert_dev(0, 0).cpu()]
    threads = threads or torch.get_num_threads()
    torch.set_num_threads(threads)
    # Prefill-sized CPU experts run while the GPU lane's demand copies stream
    # over PCIe (host DRAM is shared), so those sizes are timed with H2D
    # expert copies in flight on a side stream; decode sizes are timed alone
    # (the copy engines are mostly idle during a decode layer's CPU experts).
    contended = contended_from_rows if contended_from_rows is not None else NATIVE_MAX_ROWS + 1
    if os.environ.get("DALI_PROFILE_CONTENDED", "1") == "0":      # A/B switch
        contended = max_w + 1
    n_dma = min(6, arch.num_layers * N)
    side = dma_dst = None
    if weights.host is not None and contended <= max_w:
        side = torch.cuda.Stream(dev)
        dma_dst = torch.empty((weights.expert_bytes,), dtype=torch.uint8, device=dev)
    # Sustained warm-up first: on the GPU boxes (KVM guests) an idle host
    # streams experts at ~60% of its loaded bandwidth for the first ~0.3 s of
    # work (tools/cpu_expert_drift.py: 2.9-3.0 ms -> 1.75-1.8 ms per Mixtral
    # expert at w=1), which would overstate t_cpu and skew every decision.
    h1 = torch.randn(1, d).to(torch.bfloat16)
    t_end, i = time.perf_counter() + warmup_s, 0
    while time.perf_counter() < t_end:
        _cpu_expert(h1, blks[i % len(blks)], d, f, threads)
        i += 1
    cpu = []
    for w in ws:
        h = torch.randn(w, d).to(torch.bfloat16)
        for blk in blks[:2]:
            _cpu_expert(h, blk, d, f, threads)          # warm the pool and the clocks
        ts = []
        for i in range(max(reps + 2, 2 * len(blks) if w <= 16 else reps + 2)):
            blk = blks[(i + 1) % len(blks)]
            busy = side is not None and w >= contended
            if busy:
                with torch.cuda.stream(side):
                    for j in range(n_dma):               # ~6 x trans_time of DMA
                        h2d_block(dma_dst, weights.host.bytes[weights.expert_bytes * j:
                                                              weights.expert_bytes * (j + 1)],
                                  side, h2d_ctas)
                time.sleep(0.001)                        # let the first copy start
            t0 = time.perf_counter()
            _cpu_expert(h, blk, d, f, threads)
            ts.append((time.perf_counter() - t0) * 1e3)
            if busy:
                side.synchronize()
        # best of the runs: the steady-state streaming cost (transient host
        # hiccups during start-up otherwise bias every later decision)
        cpu.append((w, quantize_ms(min(ts))))
    del dma_dst
    # GPU compute: grouped FFN kernel, one expert resident, w tokens
    block = torch.empty((arch.expert_elems,), dtype=torch.bfloat16, device=dev)
    weights.init_expert(0, 0, block)
    ptrs = torch.zeros((N,), dtype=torch.int64, device=dev)
    ptrs[0] = block.data_ptr()
    mp = np.zeros(256, dtype=np.uint8)
    _lib.call("dali_expert_maps", block.data_ptr(), d, f, mp.ctypes.data)
    maps_dev = torch.from_numpy(mp).to(dev)
    maps = torch.zeros((N,), dtype=torch.int64, device=dev)
    maps[0] = maps_dev.data_ptr()
    gpu = []
    cs = torch.cuda.current_stream()
    for w in ws:
        xp = torch.randn(w, d, device=dev).to(torch.bfloat16)
        offs = torch.tensor([0] + [w] * N, dtype=torch.int32, device=dev)
        hbuf = torch.empty((w, f), dtype=torch.bfloat16, device=dev)
        tiles = ((w + 15) // 16 if w <= 16 else 1) * (d // 128)
        splits = ffn_splits(w, tiles, f // 64,
                            torch.cuda.get_device_properties(dev).multi_processor_count)
        yp = torch.empty((splits, w, d), dtype=torch.float32, device=dev)

        def run():
            if tc:
                _lib.call("dali_expert_ffn_tc", xp.data_ptr(), offs.data_ptr(), N,
                          maps.data_ptr(), d, f, w, w, 1, hbuf.data_ptr(), yp.data_ptr(), splits,
                          cs.cuda_stream)
            else:
                _lib.call("dali_expert_ffn", xp.data_ptr(), offs.data_ptr(), N, ptrs.data_ptr(),
                          d, f, w, w, hbuf.data_ptr(), yp.data_ptr(), cs.cuda_stream)
        run()
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            run()
            e1.record(cs)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        gpu.append((w, quantize_ms(statistics.median(ts))))
    # transfer: one expert block H2D from the pinned store
    if weights.host is not None:
        src = weights.host.bytes[:weights.expert_bytes]
        dst = torch.empty((weights.expert_bytes,), dtype=torch.uint8, device=dev)
        h2d_block(dst, src, cs, h2d_ctas)         # demand copies: copy engine
        ts = []
        for _ in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            h2d_block(dst, src, cs, h2d_ctas)
            e1.record(cs)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        trans = quantize_ms(statistics.median(ts))
        del dst
    else:
        trans = 0.0
    nm = quantize_ms(non_moe_ms) if non_moe_ms is not None else 0.0
    shared_ms = 0.0
    if arch.num_shared_experts > 0:
        # shared expert(s) at a decode-sized batch: always on the GPU (resident)
        fs = arch.shared_ffn_dim
        smp = np.zeros(256, dtype=np.uint8)
        _lib.call("dali_expert_maps", weights.shared[0].data_ptr(), d, fs, smp.ctypes.data)
        smd = torch.from_numpy(smp).to(dev)
        sptr = torch.tensor([smd.data_ptr()], dtype=torch.int64, device=dev)
        w = 1
        xs = torch.randn(w, d, device=dev).to(torch.bfloat16)
        offs = torch.tensor([0, w], dtype=torch.int32, device=dev)
        hs = torch.empty((w, fs), dtype=torch.bfloat16, device=dev)
        ys = torch.empty((1, w, d), dtype=torch.float32, device=dev)
        ts = []
        for _ in range(reps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cs)
            _lib.call("dali_expert_ffn_tc", xs.data_ptr(), offs.data_ptr(), 1, sptr.data_ptr(),
                      d, fs, w, w, 1, hs.data_ptr(), ys.data_ptr(), 1, cs.cuda_stream)
            e1.record(cs)
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        shared_ms = quantize_ms(statistics.median(ts[1:]))
    cpu = [(w, max(ms, 2.0 ** -12)) for w, ms in _monotone(cpu)]
    gpu = [(w, max(ms, 2.0 ** -12)) for w, ms in _monotone(gpu)]
    if log:
        log(f"cost model: cpu {cpu} gpu {gpu} trans {trans} non_moe {nm} shared {shared_ms}")
    return fit_cost_model(cpu, gpu, trans, shared_ms, nm)
