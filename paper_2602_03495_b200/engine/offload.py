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
    assignment: str = "greedy"
    gpu_capacity: int | None = None
    cpu_threads: int | None = None
    staging_slots: int | None = None
    capture: bool = False                   # keep gate inputs for oracle replay
    max_records: int = 16384
    time_ffn: bool = False                  # CUDA events around every expert-FFN launch
    ffn_kernel: str = "tc"                  # "tc" (tcgen05 + TMA) | "simt" (weight streaming)


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
                 max_batch: int = 1, max_seq: int = 1024):
        self.arch, self.w, self.cm, self.cfg = arch, weights, cost_model, cfg
        self.dev = torch.device("cuda", torch.cuda.current_device())
        a = arch
        L, N, k, d, f = a.num_layers, a.num_experts, a.top_k, a.hidden_dim, a.ffn_dim
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
        self.policy = PolicyEngine(
            L, N, k, cost_model, assignment=cfg.assignment, gpu_capacity=cfg.gpu_capacity,
            prefetch_size=cfg.prefetch_size if not self.resident_mode else 0,
            residuals=res_dev, cache_capacity=slots, w_size=cfg.w_size, u_size=cfg.u_size,
            seed=cfg.seed, max_records=cfg.max_records, all_resident=self.resident_mode,
            num_shared_experts=a.num_shared_experts)
        self.copy_stream = torch.cuda.Stream()
        # HBM expert cache slots: layer l owns slots [l*slots, (l+1)*slots)
        self.cache_buf = (torch.empty((L * slots, weights.expert_bytes), dtype=torch.uint8,
                                      device=self.dev) if slots else None)
        self.host_slot = self.policy.slot_of.cpu().numpy().copy()
        self.slot_ready = [None] * L
        n_stage = cfg.staging_slots or (0 if self.resident_mode else
                                        max(2 * k, N) + 2 * max(cfg.prefetch_size, 1) + 2)
        self.staging = _Staging(n_stage, weights.expert_bytes, self.dev) if n_stage else None
        self.prefetched: dict = {}          # (layer, expert) -> (staging idx, event)
        self.cpu_threads = cfg.cpu_threads or len(os.sched_getaffinity(0))
        torch.set_num_threads(self.cpu_threads)
        # per-layer pinned scratch for pointer table + G mask
        row = (N * 17 + 63) // 64 * 64        # ptrs | maps | G mask, 64-B aligned rows
        self.ptr_host = torch.zeros((L, row), dtype=torch.uint8, pin_memory=True)
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
        self.n_sm = torch.cuda.get_device_properties(self.dev).multi_processor_count
        self._load_initial_cache()

    # ------------------------------------------------------------------ setup
    def _build_maps(self):
        """One (W13, W2) tensor-map pair per physical expert location: cache
        slots, then staging slots (offload mode) or every expert (resident)."""
        a = self.arch
        if self.resident_mode:
            addrs = [self.w.expert_dev(l, e).data_ptr() for l in range(a.num_layers)
                     for e in range(a.num_experts)]
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
        sp = 1
        for s in range(1, 17):
            if kb % s == 0:
                sp = s
                if tiles * s >= 2 * self.n_sm:
                    break
        hs = self._ws("sh_h", (T, fs), torch.bfloat16)
        ys = self._ws("sh_y", (sp, T, d), torch.float32)
        cs = torch.cuda.current_stream()
        _lib.call("dali_expert_ffn_tc", h.data_ptr(), offs.data_ptr(), 1,
                  self.shared_map_ptr.data_ptr() + 8 * l, d, fs, T, T, 1, hs.data_ptr(),
                  ys.data_ptr(), sp, cs.cuda_stream)
        y = ys.sum(0) if sp > 1 else ys[0]
        if a.shared_gate:
            y = y * torch.sigmoid(h.float() @ self.w.shared_gate[l].float().t())
        return y

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

    def _splits_for(self, tiles: int) -> int:
        """Split-K factor of the down projection so decode fills the SMs."""
        kb = self.arch.ffn_dim // 64
        best = 1
        for s in range(1, 17):
            if kb % s == 0:
                best = s
                if tiles * s >= 2 * self.n_sm:
                    break
        return best

    def _load_initial_cache(self):
        if not self.slots_per_layer:
            return
        with torch.cuda.stream(self.copy_stream):
            for l in range(self.arch.num_layers):
                for e in range(self.arch.num_experts):
                    s = self.host_slot[l, e]
                    if s >= 0:
                        self.cache_buf[s].copy_(self.w.host.bytes[
                            self.w.expert_index(l, e) * self.w.expert_bytes:
                            (self.w.expert_index(l, e) + 1) * self.w.expert_bytes],
                            non_blocking=True)
        self.copy_stream.synchronize()

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
    def _moe(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int, token_index: int,
             is_eos: bool) -> torch.Tensor:
        a = self.arch
        N, k, d, f = a.num_experts, a.top_k, a.hidden_dim, a.ffn_dim
        T = h.shape[0]
        cs = torch.cuda.current_stream()
        tp0 = time.perf_counter()
        # routing outputs live in one device block [wl | idx | wts] so a single
        # D2H moves them to the host worker's pinned mirror
        nb = N * 8 + T * k * 8
        rblk = self._ws("route", (nb,), torch.uint8)
        wl = rblk[:N * 8].view(torch.int64)
        idx = rblk[N * 8:N * 8 + T * k * 4].view(torch.int32).view(T, k)
        wts = rblk[N * 8 + T * k * 4:].view(torch.float32).view(T, k)
        route_device(h, self.w.router[l], k, renorm=a.norm_topk_prob, out=(idx, wts, wl))
        gate_next = self.w.router[l + 1] if l + 1 < a.num_layers else None
        ri = self.policy.layer_step(step, l, token_index, is_eos, wl, h, gate_next)
        offsets = self._ws("offsets", (N + 1,), torch.int32)
        perm = self._ws("perm", (T * k,), torch.int32)
        pos = self._ws("pos", (T, k), torch.int32)
        _lib.call("dali_moe_plan", idx.data_ptr(), T, k, N, offsets.data_ptr(), perm.data_ptr(),
                  pos.data_ptr(), cs.cuda_stream)
        xp = self._ws("xp", (T * k, d), torch.bfloat16)
        _lib.call("dali_permute", h.data_ptr(), perm.data_ptr(), T * k, d, xp.data_ptr(),
                  cs.cuda_stream)
        # host copies for the CPU worker (small; needed before the decision is known)
        rblk_host = self._ws("route_h", (nb,), torch.uint8, pinned=True)
        h_host = self._ws("h_h", (T, d), torch.bfloat16, pinned=True)
        rblk_host.copy_(rblk, non_blocking=True)
        h_host.copy_(h, non_blocking=True)
        wl_host = rblk_host[:N * 8].view(torch.int64)
        idx_host = rblk_host[N * 8:N * 8 + T * k * 4].view(torch.int32).view(T, k)
        w_host = rblk_host[N * 8 + T * k * 4:].view(torch.float32).view(T, k)
        ev_dec = torch.cuda.Event()
        ev_dec.record(cs)
        tp1 = time.perf_counter()
        ev_dec.synchronize()
        tp2 = time.perf_counter()
        rec = self.policy.record(ri)
        self.stats.workloads[(step, l)] = wl_host.numpy().copy()
        if self.cfg.capture:
            self.stats.captured.append((step, l, h_host.clone()))
            self.stats.topk[(step, l)] = idx_host.numpy().astype(np.int64).copy()

        G = [e for e in range(N) if rec.G[e]]
        Cx = [e for e in range(N) if rec.C[e]]
        # ---- GPU experts: locate or fetch weights (raw block pointer + the
        # physical slot's tensor-map pair for the tcgen05 path)
        ptrs = np.zeros(N, dtype=np.uint64)
        maps = np.zeros(N, dtype=np.uint64)
        waits = []
        used_staging = []
        for e in G:
            if self.resident_mode:
                ptrs[e] = self.w.expert_dev(l, e).data_ptr()
                maps[e] = self._map_addr(self.w.expert_index(l, e))
                continue
            s = self.host_slot[l, e]
            if s >= 0:
                ptrs[e] = self.cache_buf[s].data_ptr()
                maps[e] = self._map_addr(s)
                if self.slot_ready[l] is not None:
                    waits.append(self.slot_ready[l])
                continue
            if (l, e) in self.prefetched:
                i, ev = self.prefetched.pop((l, e))
            else:
                i, ev = self._copy_into_staging(l, e)
                self.stats.demand_copies += 1
            ptrs[e] = self.staging.ptr(i)
            maps[e] = self._map_addr(self.n_cache_slots + i)
            waits.append(ev)
            used_staging.append(i)
        ph = self.ptr_host[l]
        ph[:N * 8].view(torch.int64).copy_(torch.from_numpy(ptrs.view(np.int64)))
        ph[N * 8:N * 16].view(torch.int64).copy_(torch.from_numpy(maps.view(np.int64)))
        gm = np.array(rec.G[:N], dtype=np.int8)
        ph[N * 16:N * 17].copy_(torch.from_numpy(gm.view(np.uint8)))
        pd = self.ptr_dev[l]
        pd.copy_(ph, non_blocking=True)
        wl_np = self.stats.workloads[(step, l)]
        splits = 1
        if G and self.use_tc:
            max_rows = int(max(wl_np[e] for e in G))
            bn = 16 if max_rows <= 16 else 32 if max_rows <= 32 else 64 if max_rows <= 64 \
                else 128 if max_rows <= 128 else 256
            tiles = sum((int(wl_np[e]) + bn - 1) // bn for e in G) * (d // 128)
            splits = self._splits_for(tiles)
        yp = self._ws("yp", (splits, T * k, d), torch.float32)
        if G:
            for ev in waits:
                cs.wait_event(ev)
            hbuf = self._ws("hbuf", (T * k, f), torch.bfloat16)
            if self.cfg.time_ffn:
                t0 = torch.cuda.Event(enable_timing=True)
                t0.record(cs)
            if self.use_tc:
                _lib.call("dali_expert_ffn_tc", xp.data_ptr(), offsets.data_ptr(), N,
                          pd.data_ptr() + N * 8, d, f, T * k, max_rows, len(G),
                          hbuf.data_ptr(), yp.data_ptr(), splits, cs.cuda_stream)
            else:
                _lib.call("dali_expert_ffn", xp.data_ptr(), offsets.data_ptr(), N, pd.data_ptr(),
                          d, f, T * k, T, hbuf.data_ptr(), yp.data_ptr(), cs.cuda_stream)
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
        for i in used_staging:
            self.staging.release(i, ffn_done)
        # prefetched-but-unused entries for this layer are dropped
        for key in [kk for kk in self.prefetched if kk[0] == l]:
            i, ev = self.prefetched.pop(key)
            self.staging.release(i, ev)

        # ---- prefetch for layer+1: the arrivals the virtual clock granted
        if not self.resident_mode:
            for j in range(rec.n_done):
                e = int(rec.cand[j])
                i, ev = self._copy_into_staging(l + 1, e)
                self.prefetched[(l + 1, e)] = (i, ev)
                self.stats.prefetch_copies += 1

        # ---- replacement: admitted experts into the victims' slots
        if rec.ev_valid and rec.ev_n and not self.resident_mode:
            with torch.cuda.stream(self.copy_stream):
                self.copy_stream.wait_event(ffn_done)
                for j in range(rec.ev_n):
                    v, c = int(rec.evicted[j]), int(rec.admitted[j])
                    s = self.host_slot[l, v]
                    self.cache_buf[s].copy_(self._host_block(l, c), non_blocking=True)
                    self.host_slot[l, c], self.host_slot[l, v] = s, -1
                    self.stats.h2d_bytes += self.w.expert_bytes
                    self.stats.replace_copies += 1
                ev = torch.cuda.Event()
                ev.record(self.copy_stream)
            self.slot_ready[l] = ev

        # ---- shared expert(s): dense SwiGLU over every token on the tensor cores,
        # queued before the host starts the CPU experts so the two overlap
        y_shared = None
        if self.shared_map_ptr is not None:
            y_shared = self._shared_ffn(l, h)

        # ---- CPU experts on the host worker
        tp3 = time.perf_counter()
        extra_dev = None
        if Cx:
            extra = self._ws("extra_h", (T, d), torch.float32, pinned=True)
            extra.zero_()
            idx_np = idx_host.numpy()
            w_np = w_host.numpy()
            for e in Cx:
                tok, slot = np.nonzero(idx_np == e)
                W13, W2 = self.w.split_expert(self._host_block(l, e).view(torch.bfloat16))
                xr = h_host[torch.from_numpy(tok)]
                gu = (xr @ W13.t()).view(len(tok), f // 64, 2, 64)
                g = gu[:, :, 0, :].reshape(len(tok), f).float()
                u = gu[:, :, 1, :].reshape(len(tok), f).float()
                act = (torch.nn.functional.silu(g) * u).to(torch.bfloat16)
                y = (act @ W2.t()).float()
                extra.index_add_(0, torch.from_numpy(tok),
                                 y * torch.from_numpy(w_np[tok, slot])[:, None])
                self.stats.cpu_expert_calls += 1
            extra_dev = extra.to(self.dev, non_blocking=True)
        if y_shared is not None:
            extra_dev = y_shared if extra_dev is None else extra_dev + y_shared
        tp4 = time.perf_counter()
        pr = self.stats.host_ms
        for key, v in (("launch_pre", tp1 - tp0), ("wait_decision", tp2 - tp1),
                       ("dispatch_gpu", tp3 - tp2), ("cpu_experts", tp4 - tp3)):
            pr[key] = pr.get(key, 0.0) + v * 1e3

        out = torch.empty_like(x)
        _lib.call("dali_unpermute_combine", x.data_ptr(), yp.data_ptr(), idx.data_ptr(),
                  pos.data_ptr(), wts.data_ptr(), pd[N * 16:].data_ptr(),
                  extra_dev.data_ptr() if extra_dev is not None else None, T, k, d, splits,
                  T * k, out.data_ptr(), cs.cuda_stream)
        return out

    # ------------------------------------------------------------- forward
    def _forward(self, tokens_dev: torch.Tensor, B: int, S: int, pos0: int, step: int,
                 token_index: int, is_eos: bool) -> torch.Tensor:
        a, W = self.arch, self.w
        x = W.embed[tokens_dev.reshape(-1)]
        T, d = x.shape
        sp = torch.cuda.current_stream().cuda_stream
        hn = self._ws("hn", (T, d), torch.bfloat16)
        h = self._ws("h", (T, d), torch.bfloat16)
        for l in range(a.num_layers):
            _lib.call("dali_add_rmsnorm", x.data_ptr(), None, W.attn_norm[l].data_ptr(),
                      a.rms_eps, T, d, None, hn.data_ptr(), sp)
            att = attention(a, hn, W.wqkv[l], W.wo[l], self.rope, self.kv, l, B, S, pos0)
            x2 = torch.empty_like(x)
            _lib.call("dali_add_rmsnorm", x.data_ptr(), att.data_ptr(), W.moe_norm[l].data_ptr(),
                      a.rms_eps, T, d, x2.data_ptr(), h.data_ptr(), sp)
            x = self._moe(l, x2, h, step, token_index, is_eos)
        last = x.view(B, S, -1)[:, -1]
        return rms_norm(last, W.final_norm, a.rms_eps) @ W.lm_head.t()

    def start_request(self, batch: int) -> np.ndarray:
        """New policy run for one request; cache residency carries over."""
        self.kv = KVCache(self.arch, batch, self.max_seq, self.dev)
        for key in list(self.prefetched):
            i, ev = self.prefetched.pop(key)
            self.staging.release(i, ev)
        init = self.policy.new_run()
        self.stats = RunStats(initial_on_gpu=init)
        self._step = 0
        return init

    def prefill(self, prompt_dev: torch.Tensor, is_eos: bool = False) -> torch.Tensor:
        B, S = prompt_dev.shape
        logits = self._forward(prompt_dev, B, S, 0, self._step, 0, is_eos)
        self.stats.steps_meta.append((0, B * S, is_eos))
        self._step += 1
        self.kv.len = S
        return logits

    def decode(self, tok_dev: torch.Tensor, is_eos: bool = False) -> torch.Tensor:
        B = tok_dev.shape[0]
        pos = self.kv.len
        ti = self._step
        logits = self._forward(tok_dev.view(B, 1), B, 1, pos, self._step, ti, is_eos)
        self.stats.steps_meta.append((ti, B, is_eos))
        self._step += 1
        self.kv.len = pos + 1
        return logits

    def generate(self, prompt: torch.Tensor, max_new_tokens: int, host_io: bool = True):
        """Greedy generation for one request.

        host_io=True (the end-to-end path a user sees): ``prompt`` (B, S)
        int64 on the HOST, copied in inside the timed region, and every
        generated token is read back to the host as it is produced.
        host_io=False: ``prompt`` already in HBM and tokens stay on device.
        Returns (tokens (B, n) int64, stats)."""
        B, S = prompt.shape
        self.start_request(B)
        l0 = _lib.launch_count()
        cs = torch.cuda.current_stream()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(cs)
        p_dev = prompt.to(self.dev, non_blocking=True) if host_io else prompt
        fetch = (lambda t: t.to("cpu")) if host_io else (lambda t: t)
        logits = self.prefill(p_dev, is_eos=(max_new_tokens <= 1))
        nxt = logits.argmax(-1)
        out = [fetch(nxt)]
        if self.cfg.capture:
            self.stats.logits.append(logits.float().cpu())
        e1.record(cs)
        for i in range(max_new_tokens - 1):
            logits = self.decode(nxt, is_eos=(i == max_new_tokens - 2))
            nxt = logits.argmax(-1)
            out.append(fetch(nxt))
            if self.cfg.capture:
                self.stats.logits.append(logits.float().cpu())
        e2.record(cs)
        e2.synchronize()
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
