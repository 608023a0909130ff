"""DALI offloading inference engine: prefill / decode / generate.

Per MoE layer (the reference driver's order, simulator.py:354-444):

  compute stream: attention -> RMSNorm -> route kernel (top-k, combine
      weights, workload histogram) -> [residual prediction for layer+1] ->
      fused policy kernel (greedy C/G, lookups, prefetch window, cache
      update; record -> pinned host memory) -> plan -> permute -> D2H of
      the gate input + routing for the CPU worker -> event
  host:  wait for the decision record, then
      * GPU experts: weights from the HBM cache slot, the prefetch staging
        slot, or a demand H2D copy (copy stream) into a staging slot;
        pointer table + G mask H2D; grouped SwiGLU FFN kernel
      * prefetch: H2D of the experts the virtual clock says arrive for
        layer+1 (copy stream, behind the demand copies)
      * replacement: admitted experts copied into the victims' HBM slots
        once this layer's FFN has read them (copy stream)
      * CPU experts: SwiGLU on the host worker (torch CPU, AMX bf16) over the
        pinned expert store, weighted partial output H2D
  compute stream: combine (Eq. 2) fused with the residual add.

Decisions are a pure function of (gate inputs, cost model, config, initial
residency): physical execution obeys them, so a CPU oracle replaying the
captured gate inputs reproduces every decision bit-for-bit.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _lib
from ..cost_model import CostModel
from ..errors import SimulationError
from ..policy_engine import PolicyEngine
from ..trace import route_device
from .arch import MoEArch
from .cpu_worker import NATIVE_MAX_ROWS, cpu_expert_rows
from .layers import KVCache, Rope, attention, rms_norm
from .weights import ModelWeights


@dataclass
class EngineConfig:
    cache_slots_per_layer: int = 0          # 0 = no cache (every GPU expert demand-fetched)
    cache_gb: float | None = None           # alternative: HBM budget -> slots per layer
    prefetch_size: int = 0
    w_size: int = 4
    u_size: int | None = None
    seed: int = 0
    assignment: str = "greedy"              # or a reference baseline solver: beam | optimal |
    #                                         static-threshold | all-cpu | all-gpu
    gpu_capacity: int | None = None
    beam_width: int = 2
    threshold: float | None = None
    exact_solver_limit: int = 24
    cache_policy: str = "workload"          # or the lru / score baselines
    insert_demand_fetched: bool = False     # reference insert toggles (cache.py:13-15)
    insert_prefetched: bool = False
    prefetch_kind: str = "residual"         # or feature | statistical | random
    frequency_table: np.ndarray | None = None   # statistical predictor (L, N)
    cpu_threads: int | None = None
    staging_slots: int | None = None
    capture: bool = False                   # keep gate inputs for oracle replay
    max_records: int = 16384
    time_ffn: bool = False                  # CUDA events around every expert-FFN launch
    ffn_kernel: str = "tc"                  # "tc" (tcgen05 + TMA) | "simt" (weight streaming)
    resident_fast: bool = True              # all-resident: no per-layer host wait
    use_graph: bool = True                  # all-resident decode steps replay one CUDA graph
    trace_layers: bool = False              # per-layer host/device timeline (tools/decode_timeline.py)


@dataclass
class RunStats:
    prefill_ms: float = 0.0
    decode_ms: float = 0.0
    prefill_tokens: int = 0
    decode_tokens: int = 0
    h2d_bytes: int = 0
    demand_copies: int = 0
    prefetch_copies: int = 0
    replace_copies: int = 0
    insert_copies: int = 0                 # D2D staging -> slot (baseline cache policies)
    cpu_expert_calls: int = 0
    gpu_expert_calls: int = 0
    dali_launches: int = 0
    initial_on_gpu: np.ndarray | None = None
    captured: list = field(default_factory=list)    # (step, layer, h (T,d) bf16 cpu)
    workloads: dict = field(default_factory=dict)   # (step, layer) -> realised workloads
    topk: dict = field(default_factory=dict)        # (step, layer) -> (T, k) experts (capture)
    logits: list = field(default_factory=list)      # per step (B, V) fp32 (capture)
    ffn_events: list = field(default_factory=list)  # (start, end, algorithmic bytes, rows)
    host_ms: dict = field(default_factory=dict)     # host-side time breakdown of _moe
    steps_meta: list = field(default_factory=list)  # (token_index, tokens, eos)
    layer_trace: list = field(default_factory=list)  # per-layer timeline (cfg.trace_layers)


def ffn_splits(max_rows: int, tiles: int, kb: int, n_sm: int) -> int:
    """Split-K planes of the down projection for dali_expert_ffn_tc: the
    smallest factor dividing f/64 that gives >= 2 CTAs per SM (``max_rows``
    is kept for the signature: every token-tile width uses the same rule)."""
    best = 1
    for s in range(1, 17):
        if kb % s == 0:
            best = s
            if tiles * s >= 2 * n_sm:
                break
    return best


class _Staging:
    """Ring of HBM staging slots for demand / prefetch copies."""

    def __init__(self, n: int, nbytes: int, device):
        self.buf = torch.empty((n, nbytes), dtype=torch.uint8, device=device)
        self.free = list(range(n))
        self.free_after = [None] * n      # event after which the slot may be overwritten

    def get(self) -> int:
        if not self.free:
            raise SimulationError("staging slots exhausted; raise EngineConfig.staging_slots")
        return self.free.pop(0)

    def release(self, i: int, ev) -> None:
        self.free_after[i] = ev
        self.free.append(i)

    def ptr(self, i: int) -> int:
        return self.buf[i].data_ptr()


class OffloadEngine:
    def __init__(self, arch: MoEArch, weights: ModelWeights, cost_model: CostModel,
                 cfg: EngineConfig, residuals: np.ndarray | None = None,
                 max_batch: int = 1, max_seq: int = 1024, ep=None):
        self.arch, self.w, self.cm, self.cfg = arch, weights, cost_model, cfg
        self.ep = ep                        # EPGroup or None (see ep.py)
        self.NL = weights.n_local           # routed experts held by this rank
        self.dev = torch.device("cuda", torch.cuda.current_device())
        a = arch
        L, k, d, f = a.num_layers, a.top_k, a.hidden_dim, a.ffn_dim
        N = self.NL
        if ep is not None and weights.experts != ep.local_experts:
            raise SimulationError("weights must hold this rank's expert shard")
        if ep is None and self.NL != a.num_experts:
            raise SimulationError("an expert shard needs an EPGroup")
        self.resident_mode = weights.resident
        slots = cfg.cache_slots_per_layer
        if cfg.cache_gb is not None:
            slots = int(cfg.cache_gb * 1e9 // weights.expert_bytes) // L
        if self.resident_mode:
            slots = 0
        slots = min(slots, N - 1)
        self.slots_per_layer = slots
        self.residuals_np = residuals
        res_dev = torch.from_numpy(np.ascontiguousarray(residuals)).to(self.dev) \
            if residuals is not None else None
        # all-resident mode is the roofline reference: every expert on the GPU
        assignment = "all-gpu" if self.resident_mode else cfg.assignment
        self.policy = PolicyEngine(
            L, N, k, cost_model, assignment=assignment, gpu_capacity=cfg.gpu_capacity,
            prefetch_size=cfg.prefetch_size if not self.resident_mode else 0,
            residuals=res_dev, cache_capacity=slots, w_size=cfg.w_size, u_size=cfg.u_size,
            seed=cfg.seed, max_records=cfg.max_records, all_resident=self.resident_mode,
            num_shared_experts=a.num_shared_experts, beam_width=cfg.beam_width,
            threshold=cfg.threshold, exact_solver_limit=cfg.exact_solver_limit,
            cache_policy=cfg.cache_policy, insert_demand_fetched=cfg.insert_demand_fetched,
            insert_prefetched=cfg.insert_prefetched, prefetch_kind=cfg.prefetch_kind,
            frequency_table=cfg.frequency_table)
        self.copy_stream = torch.cuda.Stream()       # demand + prefetch expert copies
        self.repl_stream = torch.cuda.Stream()       # cache replacement copies (off the
        #                                              demand path: never delays a demand copy)
        # HBM expert cache slots: layer l owns slots [l*slots, (l+1)*slots)
        self.cache_buf = (torch.empty((L * slots, weights.expert_bytes), dtype=torch.uint8,
                                      device=self.dev) if slots else None)
        self.host_slot = self.policy.slot_of.cpu().numpy().copy()
        self.slot_ready = [None] * (L * slots)   # per cache slot: last replacement copy
        n_stage = cfg.staging_slots or (0 if self.resident_mode else
                                        max(2 * k, N) + 2 * max(cfg.prefetch_size, 1) + 2)
        self.staging = _Staging(n_stage, weights.expert_bytes, self.dev) if n_stage else None
        self.prefetched: dict = {}          # (layer, expert) -> (staging idx, event)
        self.cpu_threads = cfg.cpu_threads or len(os.sched_getaffinity(0))
        # asynchronous CPU experts (dispatcher thread) measured ~12% slower per
        # decode token on the 16-vCPU boxes: the Python thread's GPU dispatch
        # preempts a pool thread and the pool's phase barrier waits for it.
        # Off by default; DALI_CPU_ASYNC=1 enables it.
        self._cpu_async = os.environ.get("DALI_CPU_ASYNC", "0") == "1"
        torch.set_num_threads(self.cpu_threads)
        # per-layer pinned scratch for pointer table + G mask
        row = (N * 17 + 63) // 64 * 64        # ptrs | maps | G mask, 64-B aligned rows
        self.ptr_host = torch.zeros((L, row), dtype=torch.uint8, pin_memory=True)
        self._ptr_host_np = self.ptr_host.numpy()    # same pinned memory
        self.ptr_dev = torch.zeros((L, row), dtype=torch.uint8, device=self.dev)
        self.rope = Rope(a, max_seq, self.dev)
        self.max_batch, self.max_seq = max_batch, max_seq
        self.kv = None
        self.stats = RunStats()
        self.use_tc = cfg.ffn_kernel == "tc"
        self.n_cache_slots = L * slots
        self._build_maps()
        # shared expert(s): resident dense SwiGLU blocks, one tensor-map pair per layer
        self.shared_map_ptr = None
        if a.num_shared_experts > 0:
            sm = np.zeros((L, 256), dtype=np.uint8)
            for l in range(L):
                _lib.call("dali_expert_maps", weights.shared[l].data_ptr(), d, a.shared_ffn_dim,
                          sm[l].ctypes.data)
            self.shared_maps_dev = torch.from_numpy(sm).to(self.dev)
            self.shared_map_ptr = torch.tensor(
                [self.shared_maps_dev[l].data_ptr() for l in range(L)], dtype=torch.int64,
                device=self.dev)
        self._offs_cache: dict = {}
        self._wsd: dict = {}
        self._res_maps = None
        self._wl_log = None
        self.desc_dev = torch.zeros((8,), dtype=torch.int32, device=self.dev)
        self.desc_host = torch.zeros((8,), dtype=torch.int32, pin_memory=True)
        self.desc_step_host = torch.zeros((8,), dtype=torch.int32, pin_memory=True)
        self._graph = None
        self._heads: dict = {}              # offloaded decode: layer -> (graph, h, views)
        self._heads_warm = False
        self._in_capture = False
        self._capturing = False
        self._cs_cached = None
        self._eos_at = -1
        self._pending_ffn, self._pending_cap = [], []
        self._used_fast = False
        self.n_sm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self._load_initial_cache()

    # ------------------------------------------------------------------ setup
    def _build_maps(self):
        """One (W13, W2) tensor-map pair per physical expert location: cache
        slots, then staging slots (offload mode) or every expert (resident)."""
        a = self.arch
        if self.resident_mode:
            addrs = [self.w.expert_dev(l, e).data_ptr() for l in range(a.num_layers)
                     for e in range(self.NL)]
        else:
            addrs = [self.cache_buf[s].data_ptr() for s in range(self.n_cache_slots)]
            addrs += [self.staging.ptr(i) for i in range(len(self.staging.free))]
        buf = np.zeros((max(len(addrs), 1), 256), dtype=np.uint8)
        if self.use_tc:
            for i, ad in enumerate(addrs):
                _lib.call("dali_expert_maps", ad, a.hidden_dim, a.ffn_dim,
                          buf[i].ctypes.data)
        self.maps_dev = torch.from_numpy(buf).to(self.dev)

    def _shared_ffn(self, l: int, h: torch.Tensor) -> torch.Tensor:
        """Shared expert(s) of layer l over all T tokens -> (T, d) f32."""
        a = self.arch
        T, d, fs = h.shape[0], a.hidden_dim, a.shared_ffn_dim
        offs = self._offs_cache.get(T)
        if offs is None:
            offs = torch.tensor([0, T], dtype=torch.int32, device=self.dev)
            self._offs_cache[T] = offs
        bn = 16 if T <= 16 else 32 if T <= 32 else 64 if T <= 64 else 128 if T <= 128 else 256
        kb = fs // 64
        tiles = ((T + bn - 1) // bn) * (d // 128)
        sp = ffn_splits(T, tiles, kb, self.n_sm)
        hs = self._ws("sh_h", (T, fs), torch.bfloat16)
        ys = self._ws("sh_y", (sp, T, d), torch.float32)
        cs = self._cur()
        _lib.call("dali_expert_ffn_tc", h.data_ptr(), offs.data_ptr(), 1,
                  self.shared_map_ptr.data_ptr() + 8 * l, d, fs, T, T, 1, hs.data_ptr(),
                  ys.data_ptr(), sp, cs.cuda_stream)
        y = self._ws("sh_out", (T, d), torch.float32)
        _lib.call("dali_shared_finish", ys.data_ptr(), sp, T, d, h.data_ptr(),
                  self.w.shared_gate[l].data_ptr() if a.shared_gate else None, y.data_ptr(),
                  cs.cuda_stream)
        return y

    def _cur(self):
        """The compute stream.  torch.cuda.current_stream() costs ~15 us of
        Python per call, so it is looked up once per prefill / decode step and
        cached; during graph capture the (capture) stream is read live."""
        if self._capturing or self._cs_cached is None:
            return torch.cuda.current_stream()
        return self._cs_cached

    def _ws(self, name: str, shape: tuple, dtype, pinned: bool = False) -> torch.Tensor:
        """Per-engine workspace reused across layers/steps (stream-ordered on
        the compute stream; pinned ones are rewritten only after the event
        wait that follows their previous consumer)."""
        key = (name, shape, dtype)
        t = self._wsd.get(key)
        if t is None:
            t = (torch.empty(shape, dtype=dtype, pin_memory=True) if pinned
                 else torch.empty(shape, dtype=dtype, device=self.dev))
            self._wsd[key] = t
        return t

    def _map_addr(self, phys: int) -> int:
        return self.maps_dev.data_ptr() + int(phys) * 256

    def _splits_for(self, tiles: int, max_rows: int, ffn_dim: int | None = None) -> int:
        return ffn_splits(max_rows, tiles, (ffn_dim or self.arch.ffn_dim) // 64, self.n_sm)

    def _load_initial_cache(self):
        if not self.slots_per_layer:
            return
        with torch.cuda.stream(self.copy_stream):
            for l in range(self.arch.num_layers):
                for e in range(self.NL):
                    s = self.host_slot[l, e]
                    if s >= 0:
                        self.cache_buf[s].copy_(self.w.host.bytes[
                            self.w.expert_index(l, e) * self.w.expert_bytes:
                            (self.w.expert_index(l, e) + 1) * self.w.expert_bytes],
                            non_blocking=True)
        self.copy_stream.synchronize()

    def reset_cache(self) -> None:
        """Return the HBM expert cache to its seeded initial residency (the
        state after construction): policy residency + slot table, host slot
        mirror and slot contents.  Used to start measurement passes from the
        same state so their decision sequences are identical."""
        torch.cuda.synchronize()
        pol = self.policy
        L, N, cap = self.arch.num_layers, self.NL, self.slots_per_layer
        on = pol.initial_on_gpu.astype(np.uint8)
        slot = np.full((L, N), -1, np.int32)
        if cap:
            for l in range(L):
                slot[l, np.flatnonzero(on[l])] = np.arange(cap) + l * cap
        pol.on_gpu.copy_(torch.from_numpy(on))
        pol.slot_of.copy_(torch.from_numpy(slot))
        self.host_slot = slot.copy()
        self.slot_ready = [None] * (L * cap)
        for key in list(self.prefetched):
            i, ev = self.prefetched.pop(key)
            self.staging.release(i, ev)
        self._load_initial_cache()

    def _host_block(self, l: int, e: int) -> torch.Tensor:
        off = self.w.expert_index(l, e) * self.w.expert_bytes
        return self.w.host.bytes[off:off + self.w.expert_bytes]

    # ------------------------------------------------------------- copies
    def _copy_into_staging(self, l: int, e: int) -> tuple[int, torch.cuda.Event]:
        i = self.staging.get()
        ev_prev = self.staging.free_after[i]
        with torch.cuda.stream(self.copy_stream):
            if ev_prev is not None:
                self.copy_stream.wait_event(ev_prev)
            self.staging.buf[i].copy_(self._host_block(l, e), non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(self.copy_stream)
        self.stats.h2d_bytes += self.w.expert_bytes
        return i, ev

    # ------------------------------------------------------------- MoE layer
    def _route(self, l: int, h: torch.Tensor):
        """Route kernel + plan + permute for this rank's T tokens.  Outputs live
        in one device block [wl (N i64) | offsets (N+1 i32, padded) | idx | wts]
        mirrored to pinned host memory by one D2H after the decision."""
        a = self.arch
        N, k, d = a.num_experts, a.top_k, a.hidden_dim
        T = h.shape[0]
        cs = self._cur()
        o_off = N * 8
        o_idx = o_off + ((N + 1) * 4 + 7) // 8 * 8
        o_w = o_idx + T * k * 4
        nb = o_w + T * k * 4
        rblk = self._ws("route", (nb,), torch.uint8)
        v = {
            "wl": rblk[:o_off].view(torch.int64),
            "offsets": rblk[o_off:o_off + (N + 1) * 4].view(torch.int32),
            "idx": rblk[o_idx:o_w].view(torch.int32).view(T, k),
            "wts": rblk[o_w:nb].view(torch.float32).view(T, k),
        }
        route_device(h, self.w.router[l], k, renorm=a.norm_topk_prob,
                     out=(v["idx"], v["wts"], v["wl"]))
        perm = self._ws("perm", (T * k,), torch.int32)
        v["pos"] = self._ws("pos", (T, k), torch.int32)
        v["xp"] = self._ws("xp", (T * k, d), torch.bfloat16)
        _lib.call("dali_moe_plan_permute", v["idx"].data_ptr(), T, k, N, h.data_ptr(), d,
                  v["offsets"].data_ptr(), perm.data_ptr(), v["pos"].data_ptr(),
                  v["xp"].data_ptr(), cs.cuda_stream)
        v["blk"], v["layout"] = rblk, (o_off, o_idx, o_w, nb)
        return v

    def _host_view(self, v, T: int):
        """Pinned host mirror of the routing block (valid after the event wait)."""
        N, k = self.arch.num_experts, self.arch.top_k
        o_off, o_idx, o_w, nb = v["layout"]
        hb = self._ws("route_h", (nb,), torch.uint8, pinned=True)
        hb.copy_(v["blk"], non_blocking=True)
        return {
            "wl": hb[:o_off].view(torch.int64),
            "offsets": hb[o_off:o_off + (N + 1) * 4].view(torch.int32),
            "idx": hb[o_idx:o_w].view(torch.int32).view(T, k),
            "wts": hb[o_w:nb].view(torch.float32).view(T, k),
        }

    def _exec_local(self, l: int, xrows: torch.Tensor, offsets: torch.Tensor,
                    wl_np: np.ndarray, rec, R: int):
        """GPU side of the local experts' decision: locate (cache slot /
        prefetch staging) or demand-fetch each GPU expert's weights, run the
        grouped FFN over ``xrows`` grouped by ``offsets``; issue the layer+1
        prefetch copies and the cache replacement copies.  Returns
        (yp planes, splits, G mask device pointer)."""
        a = self.arch
        NL, d, f = self.NL, a.hidden_dim, a.ffn_dim
        cs = self._cur()
        g_np = np.frombuffer(rec.G, dtype=np.int8, count=NL)
        G = np.flatnonzero(g_np).tolist()
        # numpy views of this layer's pinned row: ptrs | maps | G mask
        ph = self.ptr_host[l]
        row = self._ptr_host_np[l]
        ptrs = row[:NL * 8].view(np.uint64)
        maps = row[NL * 8:NL * 16].view(np.uint64)
        ptrs[:] = 0
        maps[:] = 0
        row[NL * 16:NL * 17] = g_np.view(np.uint8)
        waits = []
        used_staging = []
        n_hit = n_pf = n_dem = 0
        stage_of = {}                      # expert -> staging slot holding its weights
        t0_ev = None
        for e in G:
            if self.resident_mode:
                ptrs[e] = self.w.expert_dev(l, e).data_ptr()
                maps[e] = self._map_addr(self.w.expert_index(l, e))
                continue
            s = self.host_slot[l, e]
            if s >= 0:
                ptrs[e] = self.cache_buf[s].data_ptr()
                maps[e] = self._map_addr(s)
                if self.slot_ready[s] is not None:
                    waits.append(self.slot_ready[s])
                n_hit += 1
                continue
            if (l, e) in self.prefetched:
                i, ev = self.prefetched.pop((l, e))
                n_pf += 1
            else:
                i, ev = self._copy_into_staging(l, e)
                self.stats.demand_copies += 1
                n_dem += 1
            ptrs[e] = self.staging.ptr(i)
            maps[e] = self._map_addr(self.n_cache_slots + i)
            waits.append(ev)
            used_staging.append(i)
            stage_of[e] = i
        pd = self.ptr_dev[l]
        # kernel copy from mapped pinned memory: never queues behind expert DMA
        _lib.call("dali_copy_mapped", pd.data_ptr(), ph.data_ptr(), ph.numel(), cs.cuda_stream)
        splits = 1
        max_rows = 0
        if G and self.use_tc:
            wg = wl_np[G]
            max_rows = int(wg.max())
            bn = 16 if max_rows <= 16 else 32 if max_rows <= 32 else 64 if max_rows <= 64 \
                else 128 if max_rows <= 128 else 256
            tiles = int(((wg + bn - 1) // bn).sum()) * (d // 128)
            splits = self._splits_for(tiles, max_rows)
        yp = self._ws("yp", (splits, max(R, 1), d), torch.float32)
        if G and R > 0:
            for ev in waits:
                cs.wait_event(ev)
            hbuf = self._ws("hbuf", (R, f), torch.bfloat16)
            if self.cfg.time_ffn or self.cfg.trace_layers:
                t0 = t0_ev = torch.cuda.Event(enable_timing=True)
                t0.record(cs)
            if self.use_tc:
                _lib.call("dali_expert_ffn_tc", xrows.data_ptr(), offsets.data_ptr(), NL,
                          pd.data_ptr() + NL * 8, d, f, R, max_rows, len(G),
                          hbuf.data_ptr(), yp.data_ptr(), splits, cs.cuda_stream)
            else:
                _lib.call("dali_expert_ffn", xrows.data_ptr(), offsets.data_ptr(), NL,
                          pd.data_ptr(), d, f, R, R, hbuf.data_ptr(), yp.data_ptr(),
                          cs.cuda_stream)
            if self.cfg.time_ffn:
                t1 = torch.cuda.Event(enable_timing=True)
                t1.record(cs)
                n_rows = int(sum(int(wl_np[e]) for e in G))
                # algorithmic bytes: each GPU expert's weights once + activations
                byts = len(G) * self.w.expert_bytes + n_rows * (d * 2 + 2 * f * 2 + d * 4)
                self.stats.ffn_events.append((t0, t1, byts, n_rows))
            self.stats.gpu_expert_calls += len(G)
        ffn_done = torch.cuda.Event()
        ffn_done.record(cs)
        if rec.err:
            self.policy.check_errors()
        kept = self._apply_inserts(l, rec, stage_of, ffn_done, now=True)
        for i in used_staging:
            if i not in kept:
                self.staging.release(i, ffn_done)
        for key in [kk for kk in self.prefetched if kk[0] == l]:   # granted but unused
            i, ev = self.prefetched.pop(key)
            self.staging.release(i, ev)
        if not self.resident_mode:
            # prefetch for layer+1: the arrivals the virtual clock granted
            for j in range(rec.n_done):
                e = int(rec.cand[j])
                i, ev = self._copy_into_staging(l + 1, e)
                self.prefetched[(l + 1, e)] = (i, ev)
                self.stats.prefetch_copies += 1
            self._apply_inserts(l, rec, None, None, now=False)
            # replacement: admitted experts into the victims' slots once read
            if rec.ev_valid and rec.ev_n:
                with torch.cuda.stream(self.repl_stream):
                    self.repl_stream.wait_event(ffn_done)
                    for j in range(rec.ev_n):
                        v_, c_ = int(rec.evicted[j]), int(rec.admitted[j])
                        s = self.host_slot[l, v_]
                        self.cache_buf[s].copy_(self._host_block(l, c_), non_blocking=True)
                        self.host_slot[l, c_], self.host_slot[l, v_] = s, -1
                        self.stats.h2d_bytes += self.w.expert_bytes
                        self.stats.replace_copies += 1
                        ev = torch.cuda.Event()
                        ev.record(self.repl_stream)
                        self.slot_ready[s] = ev
        self._last_exec = dict(hit=n_hit, pf=n_pf, dem=n_dem, t0=t0_ev,
                               rep=int(rec.ev_n) if (rec.ev_valid and not self.resident_mode) else 0,
                               done=int(rec.n_done) if not self.resident_mode else 0)
        return yp, splits, pd.data_ptr() + NL * 16

    def _apply_inserts(self, l: int, rec, stage_of, ffn_done, now: bool) -> set:
        """Execute the cache insertions the policy kernel made outside the
        window (LRU miss inserts, insert toggles; simulator.py:372-379,
        421-423): the inserted expert's weights already sit in a staging slot
        (demand copy or prefetch), so they move into the victim's HBM slot by
        a device-to-device copy once the layer's FFN stopped reading the
        victim.  now=True handles this layer's inserts (returns the staging
        slots it keeps alive), now=False the prefetch inserts into layer+1."""
        kept = set()
        if self.resident_mode or not rec.n_ins:
            return kept
        if now:
            # An LRU lookup can evict an expert this layer used from its slot and
            # re-insert it later in the same lookup pass.  Such an expert's
            # weights live in a cache slot that an earlier insert of this pass
            # overwrites, so they are saved to staging before any insert copy.
            with torch.cuda.stream(self.repl_stream):
                self.repl_stream.wait_event(ffn_done)
                for j in range(rec.n_ins):
                    x = int(rec.ins_expert[j])
                    if int(rec.ins_kind[j]) == 2 or x in stage_of:
                        continue
                    i = self.staging.get()
                    if self.staging.free_after[i] is not None:
                        self.repl_stream.wait_event(self.staging.free_after[i])
                    self.staging.buf[i].copy_(self.cache_buf[int(self.host_slot[l, x])],
                                              non_blocking=True)
                    stage_of[x] = i
        for j in range(rec.n_ins):
            kind = int(rec.ins_kind[j])
            if (kind == 2) == now:
                continue
            ll = l + 1 if kind == 2 else l
            v, x = int(rec.ins_victim[j]), int(rec.ins_expert[j])
            s = int(self.host_slot[ll, v])
            with torch.cuda.stream(self.repl_stream):
                if kind == 2:
                    i, ev_src = self.prefetched.pop((ll, x))
                    self.repl_stream.wait_event(ev_src)
                else:
                    i = stage_of.pop(x)
                    self.repl_stream.wait_event(ffn_done)
                self.cache_buf[s].copy_(self.staging.buf[i], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.repl_stream)
            self.slot_ready[s] = ev
            self.staging.release(i, ev)
            kept.add(i)
            self.host_slot[ll, x], self.host_slot[ll, v] = s, -1
            self.stats.insert_copies += 1
        return kept

    def _cpu_submit(self, l: int, rows_host: torch.Tensor, offs_np: np.ndarray, rec, R: int):
        """Start the CPU-assigned experts on the host worker: decode-sized
        experts (<= NATIVE_MAX_ROWS rows) go to the native pool asynchronously
        (``dali_cpu_expert_submit``) so the caller dispatches the GPU side of
        the layer meanwhile; prefill-sized ones are returned for the oneDNN
        path.  Returns the job description for ``_cpu_finish``."""
        Cx = np.flatnonzero(np.frombuffer(rec.C, dtype=np.int8, count=self.NL)).tolist()
        if not Cx or R == 0:
            return None
        d = self.arch.hidden_dim
        out = self._ws("cpu_rows_h", (R, d), torch.float32, pinned=True)
        native, big = [], []
        lo, hi = R, 0
        for e in Cx:
            r0, r1 = int(offs_np[e]), int(offs_np[e + 1])
            if r1 <= r0:
                continue
            (native if r1 - r0 <= NATIVE_MAX_ROWS else big).append((e, r0, r1))
            self.stats.cpu_expert_calls += 1
            lo, hi = min(lo, r0), max(hi, r1)
        if native and not self._cpu_async:          # synchronous (A/B switch)
            for e, r0, r1 in native:
                cpu_expert_rows(self._host_block(l, e).view(torch.bfloat16),
                                rows_host[r0:r1], d, self.arch.ffn_dim, self.cpu_threads,
                                out=out[r0:r1])
            native = []
        if native:
            n = len(native)
            blocks = np.array([self.w.expert_host_ptr(l, e) for e, _, _ in native], np.uint64)
            xs = np.array([rows_host[r0].data_ptr() for _, r0, _ in native], np.uint64)
            rows = np.array([r1 - r0 for _, r0, r1 in native], np.int32)
            ys = np.array([out[r0].data_ptr() for _, r0, _ in native], np.uint64)
            _lib.call("dali_cpu_expert_submit", n, blocks.ctypes.data, xs.ctypes.data,
                      rows.ctypes.data, ys.ctypes.data, d, self.arch.ffn_dim, self.cpu_threads)
        return dict(out=out, native=bool(native), big=big, lo=lo, hi=hi, l=l, rows=rows_host)

    def _cpu_finish(self, job, R: int) -> torch.Tensor | None:
        """Run the prefill-sized CPU experts, join the asynchronous ones and
        move the CPU rows to the device (kernel copy: no copy-engine queueing)."""
        if job is None:
            return None
        a = self.arch
        d, f = a.hidden_dim, a.ffn_dim
        out = job["out"]
        for e, r0, r1 in job["big"]:
            cpu_expert_rows(self._host_block(job["l"], e).view(torch.bfloat16),
                            job["rows"][r0:r1], d, f, self.cpu_threads, out=out[r0:r1])
        if job["native"]:
            _lib.call("dali_cpu_expert_wait")
        dev_rows = self._ws("cpu_rows_d", (R, d), torch.float32)
        lo, hi = job["lo"], job["hi"]
        if hi > lo:
            _lib.call("dali_copy_mapped", dev_rows[lo].data_ptr(), out[lo].data_ptr(),
                      (hi - lo) * d * 4, self._cur().cuda_stream)
        return dev_rows

    def _cpu_rows(self, l: int, rows_host: torch.Tensor, offs_np: np.ndarray, rec,
                  R: int) -> torch.Tensor | None:
        """CPU-assigned experts on the host worker, synchronously -> (R, d)
        f32 on the device (rows of GPU experts are left unused)."""
        return self._cpu_finish(self._cpu_submit(l, rows_host, offs_np, rec, R), R)

    def _moe(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int, token_index: int,
             is_eos: bool) -> torch.Tensor:
        if self.ep is not None:
            return self._moe_ep(l, x, h, step, token_index, is_eos)
        if self.resident_mode and self.use_tc and self.cfg.resident_fast:
            return self._moe_resident(l, x, h, step, token_index, is_eos)
        cs = self._cur()
        ev_r = None
        if self.cfg.trace_layers:
            ev_r = torch.cuda.Event(enable_timing=True)
            ev_r.record(cs)
        tp0 = time.perf_counter()
        views = self._moe_head(l, h, step, token_index, is_eos, use_desc=False)
        return self._moe_tail(l, x, h, step, views, tp0, ev_r, torch.empty_like(x))

    def _moe_head(self, l: int, h: torch.Tensor, step: int, token_index: int, is_eos: bool,
                  use_desc: bool):
        """Device half of a MoE layer up to the decision: route + plan +
        permute, residual prediction for layer+1, fused policy kernel, and the
        D2H mirrors the host needs.  No host synchronisation inside, so the
        decode variant (``use_desc``: step scalars from the device descriptor,
        record at desc[3] + l) is captured into one CUDA graph per layer."""
        a = self.arch
        d, k = a.hidden_dim, a.top_k
        T = h.shape[0]
        R = T * k
        cs = self._cur()
        v = self._route(l, h)
        gate_next = self.w.router[l + 1] if l + 1 < a.num_layers else None
        if use_desc:
            pol = self.policy
            pred_p = pol.predicted_ptr(l, h, gate_next, rec_index=pol.n_records + l)
            probs_p, n_tok = pol.gate_probs_ptr(h, self.w.router[l])
            _lib.call("dali_policy_layer_desc", C.addressof(pol.cfg), C.addressof(pol.cm_c), l,
                      self.desc_dev.data_ptr(), v["wl"].data_ptr(), pred_p,
                      pol.on_gpu.data_ptr(), pol.scores.data_ptr(), pol.counters.data_ptr(),
                      pol.arrived.data_ptr(), pol.slot_of.data_ptr(), pol.lru_state.data_ptr(),
                      probs_p, n_tok, pol.record_ptr(0), cs.cuda_stream)
            ri = None
        else:
            ri = self.policy.layer_step(step, l, token_index, is_eos, v["wl"], h, gate_next,
                                        gate_this=self.w.router[l])
        hv = self._host_view(v, T)
        xp_host = self._ws("xp_h", (R, d), torch.bfloat16, pinned=True)
        xp_host.copy_(v["xp"], non_blocking=True)
        h_host = None
        if self.cfg.capture:
            h_host = self._ws("h_h", (T, d), torch.bfloat16, pinned=True)
            h_host.copy_(h, non_blocking=True)
        return dict(v=v, hv=hv, xp_host=xp_host, h_host=h_host, ri=ri, T=T)

    def _moe_tail(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int, views: dict,
                  tp0: float, ev_r, out: torch.Tensor) -> torch.Tensor:
        """Host half: wait for the decision record, execute it (GPU experts
        from cache / staging / demand copy, prefetch + replacement copies, CPU
        experts on the host worker) and queue the Eq. (2) combine into ``out``."""
        a = self.arch
        N, k, d = a.num_experts, a.top_k, a.hidden_dim
        v, hv, xp_host, T = views["v"], views["hv"], views["xp_host"], views["T"]
        R = T * k
        cs = self._cur()
        tr = self.cfg.trace_layers
        ri = views["ri"] if views["ri"] is not None else self.policy.n_records + l
        ev_dec = torch.cuda.Event(enable_timing=tr)
        ev_dec.record(cs)
        tp1 = time.perf_counter()
        ev_dec.synchronize()
        tp2 = time.perf_counter()
        rec = self.policy.record(ri)
        wl_np = hv["wl"].numpy().copy()
        self.stats.workloads[(step, l)] = wl_np
        if self.cfg.capture:
            self.stats.captured.append((step, l, views["h_host"].clone()))
            self.stats.topk[(step, l)] = hv["idx"].numpy().astype(np.int64).copy()
        offs_np = hv["offsets"].numpy()
        if self._cpu_async:
            # the CPU experts start first and run on the pool while this thread
            # dispatches the GPU experts and copies of the same layer
            job = self._cpu_submit(l, xp_host, offs_np, rec, R)
            try:
                yp, splits, gmask_p = self._exec_local(l, v["xp"], v["offsets"], wl_np, rec, R)
                y_shared = self._shared_ffn(l, h) if self.shared_map_ptr is not None else None
            except BaseException:
                if job is not None and job["native"]:
                    _lib.load().dali_cpu_expert_wait()     # never leave a job in flight
                raise
            tp3 = time.perf_counter()
        else:
            # GPU work is queued first (it runs during the CPU experts), then the
            # CPU experts run on this thread's pool
            yp, splits, gmask_p = self._exec_local(l, v["xp"], v["offsets"], wl_np, rec, R)
            y_shared = self._shared_ffn(l, h) if self.shared_map_ptr is not None else None
            tp3 = time.perf_counter()
            job = self._cpu_submit(l, xp_host, offs_np, rec, R)
        cpu_rows = self._cpu_finish(job, R)
        tp4 = time.perf_counter()
        self._acct(tp0, tp1, tp2, tp3, tp4)
        _lib.call("dali_unpermute_combine", x.data_ptr(), yp.data_ptr(), v["idx"].data_ptr(),
                  v["pos"].data_ptr(), v["wts"].data_ptr(), gmask_p,
                  cpu_rows.data_ptr() if cpu_rows is not None else None,
                  y_shared.data_ptr() if y_shared is not None else None, T, k, d, splits,
                  R, out.data_ptr(), cs.cuda_stream)
        if tr:
            ev_c = torch.cuda.Event(enable_timing=True)
            ev_c.record(cs)
            le = self._last_exec
            self.stats.layer_trace.append(dict(
                step=step, layer=l, T=T, nC=int(sum(1 for e in range(N) if rec.C[e] and wl_np[e])),
                hit=le["hit"], pf=le["pf"], dem=le["dem"], rep=le["rep"], done=le["done"],
                host=(tp0, tp1, tp2, tp3, tp4, time.perf_counter()),
                ev=(ev_r if ev_r is not None else ev_dec, ev_dec, le["t0"], ev_c)))
        return out

    def _moe_resident(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int,
                      token_index: int, is_eos: bool) -> torch.Tensor:
        """All-resident fast path (roofline reference): every expert lives in
        HBM, so the decision needs no host action -- route, policy, plan,
        permute, grouped FFN over the static per-layer map table and combine
        are enqueued back to back with no host wait.  Records and workloads
        are read after the step (``_finish_resident``): a CPU assignment
        there would be a contract violation and raises."""
        a = self.arch
        N, k, d, f = a.num_experts, a.top_k, a.hidden_dim, a.ffn_dim
        T = h.shape[0]
        R = T * k
        cs = self._cur()
        tp0 = time.perf_counter()
        v = self._route(l, h)
        if T == self.kv.k.shape[1] and self.stats.steps_meta:     # decode: device descriptor
            ri = self.policy.n_records + l
            _lib.call("dali_policy_layer_desc", C.addressof(self.policy.cfg),
                      C.addressof(self.policy.cm_c), l, self.desc_dev.data_ptr(),
                      v["wl"].data_ptr(), None, self.policy.on_gpu.data_ptr(),
                      self.policy.scores.data_ptr(), self.policy.counters.data_ptr(),
                      self.policy.arrived.data_ptr(), self.policy.slot_of.data_ptr(),
                      self.policy.lru_state.data_ptr(), None, 0, self.policy.record_ptr(0),
                      cs.cuda_stream)
            if l == a.num_layers - 1 and not self._in_capture:
                self.policy.n_records += a.num_layers
        else:
            ri = self.policy.layer_step(step, l, token_index, is_eos, v["wl"], None, None)
        self._used_fast = True
        if self._res_maps is None:
            tab = np.array([[self._map_addr(self.w.expert_index(ll, e)) for e in range(N)]
                            for ll in range(a.num_layers)], dtype=np.int64)
            self._res_maps = torch.from_numpy(tab).to(self.dev)
        mr = min(T, R)                 # an expert sees each token at most once
        bn = 16 if mr <= 16 else 32 if mr <= 32 else 64 if mr <= 64 else 128 if mr <= 128 else 256
        tiles = min(N, R) * ((mr + bn - 1) // bn) * (d // 128)
        splits = self._splits_for(tiles, mr)
        yp = self._ws("yp", (splits, R, d), torch.float32)
        hbuf = self._ws("hbuf", (R, f), torch.bfloat16)
        if self.cfg.time_ffn:
            t0 = torch.cuda.Event(enable_timing=True)
            t0.record(cs)
        _lib.call("dali_expert_ffn_tc", v["xp"].data_ptr(), v["offsets"].data_ptr(), N,
                  self._res_maps[l].data_ptr(), d, f, R, mr, min(N, R), hbuf.data_ptr(),
                  yp.data_ptr(), splits, cs.cuda_stream)
        if self.cfg.time_ffn:
            t1 = torch.cuda.Event(enable_timing=True)
            t1.record(cs)
            self._pending_ffn.append((t0, t1, step, l))
        y_shared = self._shared_ffn(l, h) if self.shared_map_ptr is not None else None
        out = torch.empty_like(x)
        _lib.call("dali_unpermute_combine", x.data_ptr(), yp.data_ptr(), v["idx"].data_ptr(),
                  v["pos"].data_ptr(), v["wts"].data_ptr(), None, None,
                  y_shared.data_ptr() if y_shared is not None else None, T, k, d, splits, R,
                  out.data_ptr(), cs.cuda_stream)
        if self.cfg.capture:
            hh = torch.empty((T, d), dtype=torch.bfloat16, pin_memory=True)
            hh.copy_(h, non_blocking=True)
            ih = torch.empty((T, k), dtype=torch.int32, pin_memory=True)
            ih.copy_(v["idx"], non_blocking=True)
            self._pending_cap.append((step, l, hh, ih))
        tp1 = time.perf_counter()
        self._acct(tp0, tp1, tp1, tp1, tp1)
        return out

    def _finish_resident(self):
        """Deferred bookkeeping of the resident fast path / graph replays (after
        a sync): workloads and assignments come from the decision records."""
        a = self.arch
        d, f, NL = a.hidden_dim, a.ffn_dim, self.NL
        for i in range(self.policy.n_records):
            rec = self.policy.record(i)
            key = (rec.step, rec.layer)
            self.stats.workloads[key] = np.array(rec.workload[:NL], dtype=np.int64)
            if any(rec.C[e] for e in range(NL)):
                raise SimulationError("all-resident mode: the policy assigned an expert to the "
                                      "CPU (cost model contract violated)")
            self.stats.gpu_expert_calls += int(sum(1 for e in range(NL) if rec.G[e]))
        for (t0, t1, step, l) in self._pending_ffn:
            wl = self.stats.workloads[(step, l)]
            n_rows = int(wl.sum())
            ng = int((wl > 0).sum())
            byts = ng * self.w.expert_bytes + n_rows * (d * 2 + 2 * f * 2 + d * 4)
            self.stats.ffn_events.append((t0, t1, byts, n_rows))
        for (step, l, hh, ih) in self._pending_cap:
            self.stats.captured.append((step, l, hh))
            self.stats.topk[(step, l)] = ih.numpy().astype(np.int64).copy()
        self._pending_ffn, self._pending_cap = [], []
        self._used_fast = False

    def _acct(self, tp0, tp1, tp2, tp3, tp4):
        pr = self.stats.host_ms
        for key, val in (("launch_pre", tp1 - tp0), ("wait_decision", tp2 - tp1),
                         ("dispatch_gpu", tp3 - tp2), ("cpu_experts", tp4 - tp3)):
            pr[key] = pr.get(key, 0.0) + val * 1e3

    def _moe_ep(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int, token_index: int,
                is_eos: bool) -> torch.Tensor:
        """Expert-parallel MoE layer (see ep.py): dispatch all-to-all, DALI
        policy + execution on this rank's NL experts with global workloads,
        return all-to-all, Eq. (2) combine on the source rank."""
        from .ep import plan_regroup, send_sizes
        a, ep = self.arch, self.ep
        N, k, d, NL = a.num_experts, a.top_k, a.hidden_dim, self.NL
        T = h.shape[0]
        cs = self._cur()
        tp0 = time.perf_counter()
        v = self._route(l, h)
        recv_counts = ep.exchange_counts(v["wl"])                  # (G*NL,) int64
        wl_glob = recv_counts.view(ep.world, NL).sum(0)
        pred = None
        if self.policy.prefetch_size > 0 and l + 1 < a.num_layers:
            _, _, pw = route_device(h, self.w.router[l + 1], k, residual=self.policy.residuals[l],
                                    want_idx=False, want_weights=False)
            pred = ep.all_reduce_sum_(pw)[ep.rank * NL:(ep.rank + 1) * NL].contiguous()
        ri = self.policy.layer_step(step, l, token_index, is_eos, wl_glob, None, None,
                                    predicted=pred)
        hv = self._host_view(v, T)
        rc_host = self._ws("rc_h", (ep.world * NL,), torch.int64, pinned=True)
        rc_host.copy_(recv_counts, non_blocking=True)
        if self.cfg.capture:
            h_host = self._ws("h_h", (T, d), torch.bfloat16, pinned=True)
            h_host.copy_(h, non_blocking=True)
        ev_dec = torch.cuda.Event()
        ev_dec.record(cs)
        tp1 = time.perf_counter()
        ev_dec.synchronize()
        tp2 = time.perf_counter()
        rec = self.policy.record(ri)
        rc = rc_host.numpy().reshape(ep.world, NL).copy()
        wl_np = rc.sum(axis=0)
        self.stats.workloads[(step, l)] = wl_np
        if self.cfg.capture:
            self.stats.captured.append((step, l, h_host.clone()))
            self.stats.topk[(step, l)] = hv["idx"].numpy().astype(np.int64).copy()
        perm2, offs_l, recv_sz = plan_regroup(rc)
        snd_sz = send_sizes(hv["wl"].numpy(), ep.world)
        recv_x = ep.exchange_rows(v["xp"], snd_sz, recv_sz)        # (R, d) bf16
        R = int(recv_x.shape[0])
        perm2_d = torch.from_numpy(perm2).to(self.dev, non_blocking=True)
        offs_d = torch.from_numpy(offs_l).to(self.dev, non_blocking=True)
        xl = self._ws("xl", (max(R, 1), d), torch.bfloat16)
        if R:
            _lib.call("dali_permute", recv_x.data_ptr(), perm2_d.data_ptr(), R, d, xl.data_ptr(),
                      cs.cuda_stream)
        yp, splits, _ = self._exec_local(l, xl, offs_d, wl_np, rec, R)
        y_shared = self._shared_ffn(l, h) if self.shared_map_ptr is not None else None
        tp3 = time.perf_counter()
        cpu_rows = None
        if any(rec.C[e] for e in range(NL)) and R:
            xl_host = self._ws("xl_h", (R, d), torch.bfloat16, pinned=True)
            xl_host.copy_(xl[:R])
            cpu_rows = self._cpu_rows(l, xl_host, offs_l, rec, R)
        tp4 = time.perf_counter()
        self._acct(tp0, tp1, tp2, tp3, tp4)
        # per-row expert outputs in grouped order -> received order -> sources
        # split-K planes summed in plane order, exactly as the combine kernel
        # does (fp32 adds in the same order: bit-identical to the 1-GPU engine)
        y_l = yp[0, :R].clone()
        for s_ in range(1, splits):
            y_l += yp[s_, :R]
        if cpu_rows is not None:
            for e in range(NL):
                if rec.C[e] and offs_l[e + 1] > offs_l[e]:
                    y_l[offs_l[e]:offs_l[e + 1]] = cpu_rows[offs_l[e]:offs_l[e + 1]]
        y_recv = torch.empty_like(y_l)
        if R:
            y_recv.index_copy_(0, perm2_d.long(), y_l)
        y_back = ep.exchange_rows(y_recv, recv_sz, snd_sz)          # (T*k, d) f32
        out = torch.empty_like(x)
        _lib.call("dali_unpermute_combine", x.data_ptr(), y_back.data_ptr(), v["idx"].data_ptr(),
                  v["pos"].data_ptr(), v["wts"].data_ptr(), None, None,
                  y_shared.data_ptr() if y_shared is not None else None, T, k, d, 1, T * k,
                  out.data_ptr(), cs.cuda_stream)
        return out

    # ------------------------------------------------------------- forward
    def _attn_decode(self, l: int, hn: torch.Tensor, B: int) -> torch.Tensor:
        """One-token GQA attention: qkv GEMM, fused RoPE + KV append and
        split-K decode attention reading pos / len from the device step
        descriptor (graph-capturable), o-proj GEMM."""
        a, W = self.arch, self.w
        H, KV, hd = a.num_heads, a.num_kv_heads, a.head_dim
        sp = self._cur().cuda_stream
        nqkv = (H + 2 * KV) * hd
        if B <= 8:          # weight-streaming GEMV kernel (decode batches)
            qkv = self._ws("qkv_dec", (B, nqkv), torch.bfloat16)
            _lib.call("dali_gemv_bf16", hn.data_ptr(), W.wqkv[l].data_ptr(), B, nqkv,
                      a.hidden_dim, qkv.data_ptr(), sp)
        else:
            qkv = hn @ W.wqkv[l].t()
        q = self._ws("q_dec", (B, H, hd), torch.bfloat16)
        kc, vc = self.kv.k[l], self.kv.v[l]
        _lib.call("dali_rope_append", qkv.data_ptr(), self.rope.cos.data_ptr(),
                  self.rope.sin.data_ptr(), self.desc_dev.data_ptr() + 16, B, H, KV, hd,
                  self.max_seq, q.data_ptr(), kc.data_ptr(), vc.data_ptr(), sp)
        splits = 16
        ws = self._ws("attn_ws", (B * H * splits * (hd + 2),), torch.float32)
        o = self._ws("o_dec", (B, H * hd), torch.bfloat16)
        _lib.call("dali_decode_attention", q.data_ptr(), kc.data_ptr(), vc.data_ptr(),
                  self.desc_dev.data_ptr() + 20, B, H, KV, hd, self.max_seq, splits,
                  1.0 / math.sqrt(hd), ws.data_ptr(), o.data_ptr(), sp)
        if B <= 8:
            att = self._ws("att_dec", (B, a.hidden_dim), torch.bfloat16)
            _lib.call("dali_gemv_bf16", o.data_ptr(), W.wo[l].data_ptr(), B, a.hidden_dim,
                      H * hd, att.data_ptr(), sp)
            return att
        return o @ W.wo[l].t()

    def _forward(self, tokens_dev: torch.Tensor, B: int, S: int, pos0: int, step: int,
                 token_index: int, is_eos: bool) -> torch.Tensor:
        a, W = self.arch, self.w
        x = W.embed[tokens_dev.reshape(-1)]
        T, d = x.shape
        sp = self._cur().cuda_stream
        hn = self._ws("hn", (T, d), torch.bfloat16)
        h = self._ws("h", (T, d), torch.bfloat16)
        dev_attn = S == 1 and a.head_dim in (64, 128)
        for l in range(a.num_layers):
            _lib.call("dali_add_rmsnorm", x.data_ptr(), None, W.attn_norm[l].data_ptr(),
                      a.rms_eps, T, d, None, hn.data_ptr(), sp)
            if dev_attn:
                att = self._attn_decode(l, hn, B)
            else:
                att = attention(a, hn, W.wqkv[l], W.wo[l], self.rope, self.kv, l, B, S, pos0)
            x2 = torch.empty_like(x)
            _lib.call("dali_add_rmsnorm", x.data_ptr(), att.data_ptr(), W.moe_norm[l].data_ptr(),
                      a.rms_eps, T, d, x2.data_ptr(), h.data_ptr(), sp)
            x = self._moe(l, x2, h, step, token_index, is_eos)
        last = x.view(B, S, -1)[:, -1]
        return rms_norm(last, W.final_norm, a.rms_eps) @ W.lm_head.t()

    # ------------------------------------------------- offloaded decode (graphs)
    def _offload_graphable(self) -> bool:
        # the random predictor draws on the host every step: not graph-capturable
        return (not self.resident_mode and self.ep is None and self.cfg.use_graph and
                self.arch.head_dim in (64, 128) and self.policy.prefetch_kind != "random")

    def _decode_head(self, l: int, X: torch.Tensor, X2: torch.Tensor, B: int):
        """Layer l of a decode step up to the MoE decision: attention block
        (norm, qkv, fused RoPE/KV append, split-K attention, o-proj, add +
        norm) and the MoE head.  Step scalars come from the device descriptor,
        so the same launch sequence is valid for every step (graph body)."""
        a, W = self.arch, self.w
        d = a.hidden_dim
        sp = self._cur().cuda_stream
        hn = self._ws("hn", (B, d), torch.bfloat16)
        h = self._ws("h", (B, d), torch.bfloat16)
        _lib.call("dali_add_rmsnorm", X.data_ptr(), None, W.attn_norm[l].data_ptr(), a.rms_eps,
                  B, d, None, hn.data_ptr(), sp)
        att = self._attn_decode(l, hn, B)
        _lib.call("dali_add_rmsnorm", X.data_ptr(), att.data_ptr(), W.moe_norm[l].data_ptr(),
                  a.rms_eps, B, d, X2.data_ptr(), h.data_ptr(), sp)
        return h, self._moe_head(l, h, 0, 0, False, use_desc=True)

    def _decode_offload(self, tok_dev: torch.Tensor, B: int, is_eos: bool) -> torch.Tensor:
        """One offloaded decode step.  Per layer, the device half (attention +
        routing + policy + D2H mirrors) replays a CUDA graph captured on the
        second decode step (the first runs eagerly and warms workspaces); the
        host half executes the decision.  The step descriptor is written from
        pinned memory by a kernel copy before the layers run."""
        a, W = self.arch, self.w
        L, d = a.num_layers, a.hidden_dim
        cs = self._cur()
        step, pos = self._step, self.kv.len
        base = self.policy.n_records
        if base + L > self.policy.max_records:
            raise SimulationError("decision log full")
        dh = self.desc_step_host
        dh.copy_(torch.tensor([step, step, step if is_eos else -1, base, pos, pos + 1, L, 0],
                              dtype=torch.int32))
        _lib.call("dali_copy_mapped", self.desc_dev.data_ptr(), dh.data_ptr(), 32, cs.cuda_stream)
        X = self._ws("dec_X", (B, d), torch.bfloat16)
        X2 = self._ws("dec_X2", (B, d), torch.bfloat16)
        torch.index_select(W.embed, 0, tok_dev.reshape(-1), out=X)
        heads = self._heads
        capture = self._heads_warm and not heads
        for l in range(L):
            ev_r = None
            if self.cfg.trace_layers:
                ev_r = torch.cuda.Event(enable_timing=True)
                ev_r.record(cs)
            tp0 = time.perf_counter()
            if l in heads:
                g, h, views = heads[l]
                g.replay()
            elif capture:
                g = torch.cuda.CUDAGraph()
                self._capturing = True
                try:
                    with torch.cuda.graph(g):
                        h, views = self._decode_head(l, X, X2, B)
                finally:
                    self._capturing = False
                g.replay()
                heads[l] = (g, h, views)
            else:
                h, views = self._decode_head(l, X, X2, B)
            self._moe_tail(l, X2, h, step, views, tp0, ev_r, X)
        self._heads_warm = True
        self.policy.n_records = base + L
        return rms_norm(X, W.final_norm, a.rms_eps) @ W.lm_head.t()

    def _set_desc(self, step: int, token_index: int, eos_at: int, rec_index: int, pos: int):
        """Write the device step descriptor (stream-ordered kernel copy from
        pinned memory: never queued behind expert DMA on a copy engine)."""
        dh = self.desc_host
        dh.copy_(torch.tensor([step, token_index, eos_at, rec_index, pos, pos + 1,
                               self.arch.num_layers, 0], dtype=torch.int32))
        _lib.call("dali_copy_mapped", self.desc_dev.data_ptr(), dh.data_ptr(), 32,
                  self._cur().cuda_stream)

    def start_request(self, batch: int) -> np.ndarray:
        """New policy run for one request; cache residency carries over."""
        if self.kv is None or self.kv.k.shape[1] != batch:
            self.kv = KVCache(self.arch, batch, self.max_seq, self.dev)
            self._graph = None
            self._heads, self._heads_warm = {}, False
        self.kv.len = 0
        for key in list(self.prefetched):
            i, ev = self.prefetched.pop(key)
            self.staging.release(i, ev)
        init = self.policy.new_run()
        self.stats = RunStats(initial_on_gpu=init)
        self._step = 0
        self._eos_at = -1
        return init

    def prefill(self, prompt_dev: torch.Tensor, is_eos: bool = False) -> torch.Tensor:
        self._cs_cached = torch.cuda.current_stream()
        B, S = prompt_dev.shape
        logits = self._forward(prompt_dev, B, S, 0, self._step, 0, is_eos)
        self.stats.steps_meta.append((0, B * S, is_eos))
        self._step += 1
        self.kv.len = S
        # device descriptor of the first decode step (pos = S)
        self._set_desc(self._step, self._step, self._eos_at, self.policy.n_records, S)
        return logits

    def _graphable(self) -> bool:
        return (self.resident_mode and self.use_tc and self.cfg.resident_fast and
                self.cfg.use_graph and self.arch.head_dim == 128 and self.ep is None and
                not self.cfg.capture)

    def decode(self, tok_dev: torch.Tensor, is_eos: bool = False) -> torch.Tensor:
        self._cs_cached = torch.cuda.current_stream()
        B = tok_dev.shape[0]
        pos = self.kv.len
        ti = self._step
        if self._graphable():
            logits = self._decode_graph(tok_dev)
        elif self._offload_graphable():
            logits = self._decode_offload(tok_dev, B, is_eos)
        else:
            logits = self._forward(tok_dev.view(B, 1), B, 1, pos, self._step, ti, is_eos)
            _lib.call("dali_step_advance", self.desc_dev.data_ptr(),
                      self._cur().cuda_stream)
        self.stats.steps_meta.append((ti, B, is_eos))
        self._step += 1
        self.kv.len = pos + 1
        return logits

    def _decode_graph(self, tok_dev: torch.Tensor) -> torch.Tensor:
        """All-resident decode step as one CUDA graph: every per-step scalar
        (step, token index, record slot, KV position) lives in the device
        descriptor, which the graph advances itself, so a replay needs no
        host input.  The first decode step runs eagerly (warms workspaces)
        and the graph is captured on the second."""
        B = tok_dev.shape[0]
        L = self.arch.num_layers
        if self._graph is not None:
            self._graph_in.copy_(tok_dev.view(B))
            self._graph.replay()
            self.policy.n_records += L
            return self._graph_logits
        if not getattr(self, "_graph_warm", False):
            logits = self._forward(tok_dev.view(B, 1), B, 1, self.kv.len, self._step, self._step,
                                   False)
            _lib.call("dali_step_advance", self.desc_dev.data_ptr(),
                      self._cur().cuda_stream)
            self._graph_warm = True
            return logits
        self._graph_in = torch.zeros((B,), dtype=torch.int64, device=self.dev)
        self._graph_in.copy_(tok_dev.view(B))
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        saved = self.cfg.time_ffn
        self.cfg.time_ffn = False                 # no timing events inside the graph
        self._in_capture = True
        n0 = self.policy.n_records
        self._capturing = True
        with torch.cuda.graph(g):
            out = self._forward(self._graph_in.view(B, 1), B, 1, 0, 0, 0, False)
            _lib.call("dali_step_advance", self.desc_dev.data_ptr(),
                      self._cur().cuda_stream)
        self._in_capture = False
        self._capturing = False
        self.cfg.time_ffn = saved
        self.policy.n_records = n0
        self._graph, self._graph_logits = g, out
        g.replay()
        self.policy.n_records += L
        return out

    def generate(self, prompt: torch.Tensor, max_new_tokens: int, host_io: bool = True):
        """Greedy generation for one request.

        host_io=True (the end-to-end path a user sees): ``prompt`` (B, S)
        int64 on the HOST, copied in inside the timed region, and every
        generated token is read back to the host as it is produced.
        host_io=False: ``prompt`` already in HBM and tokens stay on device.
        Returns (tokens (B, n) int64, stats)."""
        B, S = prompt.shape
        self._cs_cached = torch.cuda.current_stream()
        self.start_request(B)
        l0 = _lib.launch_count()
        cs = self._cur()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(cs)
        if host_io:
            # host I/O through pinned staging + kernel copies (UVA): neither the
            # prompt upload nor the per-token read can queue behind expert DMA
            # on a copy engine
            p_pin = self._ws("prompt_h", (B, S), torch.int64, pinned=True)
            p_pin.copy_(prompt)
            p_dev = self._ws("prompt_d", (B, S), torch.int64)
            _lib.call("dali_copy_mapped", p_dev.data_ptr(), p_pin.data_ptr(), B * S * 8,
                      cs.cuda_stream)
            toks_h = self._ws("tokens_h", (max(max_new_tokens, 1), B), torch.int64, pinned=True)

            def fetch(t, i):
                _lib.call("dali_copy_mapped", toks_h[i].data_ptr(), t.data_ptr(), B * 8,
                          self._cur().cuda_stream)
                ev = torch.cuda.Event()
                ev.record()
                ev.synchronize()
                return toks_h[i].clone()
        else:
            p_dev = prompt

            def fetch(t, i):
                return t
        logits = self.prefill(p_dev, is_eos=(max_new_tokens <= 1))
        nxt = logits.argmax(-1)
        out = [fetch(nxt, 0)]
        if self.cfg.capture:
            self.stats.logits.append(logits.float().cpu())
        e1.record(cs)
        for i in range(max_new_tokens - 1):
            logits = self.decode(nxt, is_eos=(i == max_new_tokens - 2))
            nxt = logits.argmax(-1)
            out.append(fetch(nxt, i + 1))
            if self.cfg.capture:
                self.stats.logits.append(logits.float().cpu())
        e2.record(cs)
        e2.synchronize()
        if self._used_fast:
            self._finish_resident()
        st = self.stats
        st.prefill_ms = e0.elapsed_time(e1)
        st.decode_ms = e1.elapsed_time(e2)
        st.prefill_tokens = B * S
        st.decode_tokens = B * max(max_new_tokens - 1, 0)
        st.dali_launches = _lib.launch_count() - l0
        return torch.stack(out, dim=1), st

    # ------------------------------------------------------------- reporting
    def policy_report(self) -> dict:
        """RunReport-shaped dict of the current request's decisions (virtual
        clock, hit rates, prefetch accuracy, replacement log)."""
        toks = [m[1] for m in self.stats.steps_meta]
        return self.policy.build_report(toks, self.stats.workloads, {})


def export_trace(engine: "OffloadEngine", trace_path: str, gates_path: str | None = None,
                 residuals_path: str | None = None, batch_size: int = 1):
    """Write the last request as reference-format artifacts (SURVEY section 8f
    rank 3): the per-step x per-layer workloads (plus gate inputs when the
    engine captured them), the router sidecar and the residual sidecar, so
    ``moesim`` can replay exactly the routing the B200 engine executed."""
    from ..trace import (GateParams, ResidualVectors, Trace, TokenStep, save_gate_params,
                         save_residuals, save_trace)
    a, st = engine.arch, engine.stats
    L = a.num_layers
    hid = {}
    for (s, l, h) in st.captured:
        hid.setdefault(s, {})[l] = h.double().numpy()
    steps = []
    for s, (ti, ntok, eos) in enumerate(st.steps_meta):
        wl = np.stack([st.workloads[(s, l)] for l in range(L)])
        h = np.stack([hid[s][l] for l in range(L)]) if s in hid and len(hid[s]) == L else None
        steps.append(TokenStep(ti, ntok, wl, h, eos))
    cfg = a.routing
    tr = Trace(cfg, batch_size, "decode", steps,
               generator_params={"source": "paper_2602_03495_b200 engine", "arch": a.name})
    save_trace(tr, trace_path)
    if gates_path is not None:
        save_gate_params(GateParams(np.stack([engine.w.router[l].double().cpu().numpy()
                                              for l in range(L)])), gates_path)
    if residuals_path is not None and engine.residuals_np is not None:
        save_residuals(ResidualVectors(engine.residuals_np), residuals_path)
    return tr
