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

This module holds the engine state, setup and the user-facing entry points;
the MoE layer lives in ``moe_exec.py``, the decode steps / CUDA graphs in
``decode_graph.py`` and the expert-parallel layer in ``ep.py`` (mixins).
"""

from __future__ import annotations

import collections
import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from .. import _lib
from ..cost_model import CostModel
from ..errors import SimulationError
from ..policy_engine import PolicyEngine
from .arch import MoEArch
from .decode_graph import DecodeGraphMixin
from .ep import EPMoEMixin
from .layers import KVCache, Rope, attention, rms_norm
from .moe_exec import MoEExecMixin, ffn_splits  # noqa: F401  (ffn_splits re-export)
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
    capture_moe_io: bool = False            # also keep every MoE layer's residual input and
    #                                         output (per-layer numeric parity tests)
    max_records: int = 16384
    time_ffn: bool = False                  # CUDA events around every expert-FFN launch
    ffn_kernel: str = "tc"                  # "tc" (tcgen05 + TMA) | "simt" (weight streaming)
    resident_fast: bool = True              # all-resident: no per-layer host wait
    use_graph: bool = True                  # all-resident decode steps replay one CUDA graph
    ep_transport: str = "p2p"               # expert parallelism: "p2p" (peer-memory kernels,
    #                                         csrc/ep.cu) or "nccl" (all_to_all baseline)
    trace_layers: bool = False              # per-layer host/device timeline (tools/decode_timeline.py)
    fused_route_plan: bool = os.environ.get("DALI_FUSED_ROUTE_PLAN", "1") != "0"
    #                                         decode (T <= 16): routing + plan + permute in
    #                                         one launch (dali_route_plan_bf16)
    shared_in_head: bool = os.environ.get("DALI_SHARED_HEAD", "1") != "0"
    #                                         the shared expert(s) run on a side stream
    #                                         beside routing + policy (offloaded: inside the
    #                                         per-layer decode graph, not after the host has
    #                                         read the decision; all-resident: beside routing
    #                                         and the routed FFN), joined before the combine
    fused_norm_gemv: bool = os.environ.get("DALI_FUSED_NORM", "1") != "0"
    #                                         decode (B <= 8): attention-block RMSNorms fused
    #                                         into the qkv / o projection GEMVs
    policy_side_stream: bool = os.environ.get("DALI_POLICY_SIDE", "1") != "0"
    #                                         all-resident decode: the policy kernel (records
    #                                         only, nothing downstream reads them) runs on a
    #                                         side stream off the layer's critical path
    h2d_sm_ctas: int = int(os.environ.get("DALI_H2D_SM_CTAS", "0"))
    #                                         replacement / prefetch H2D copies driven by this
    #                                         many SMs (bounded PCIe queue depth, paused in
    #                                         the decode chain's quiet window); 0 = copy
    #                                         engine (default: measured faster end to end)
    lazy_replace: bool = os.environ.get("DALI_LAZY_REPLACE", "1") != "0"
    #                                         window replacement copies deferred: issued when
    #                                         a hit needs the slot, else in the background in
    #                                         next-use order (MoEExecMixin._defer_repl)
    repl_inflight: int = int(os.environ.get("DALI_REPL_INFLIGHT", "-1"))
    #                                         deferred replacements copied in the background
    #                                         at a time (-1: 0 for blocks <= 64 MB, else 1)


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
    replace_urgent: int = 0                # deferred replacements issued by a hit
    replace_dropped: int = 0               # deferred replacements superseded before a read
    cpu_expert_calls: int = 0
    gpu_expert_calls: int = 0
    decode_host_bytes: int = 0             # expert bytes read from host DRAM while decoding
    decode_h2d_bytes: int = 0              # of which H2D expert copies (PCIe)
    dali_launches: int = 0
    initial_on_gpu: np.ndarray | None = None
    captured: list = field(default_factory=list)    # (step, layer, h (T,d) bf16 cpu)
    moe_io: list = field(default_factory=list)      # (step, layer, x_in, out) bf16 cpu pinned
    workloads: dict = field(default_factory=dict)   # (step, layer) -> realised workloads
    topk: dict = field(default_factory=dict)        # (step, layer) -> (T, k) experts (capture)
    logits: list = field(default_factory=list)      # per step (B, V) fp32 (capture)
    ffn_events: list = field(default_factory=list)  # (start, end, algorithmic bytes, rows)
    host_ms: dict = field(default_factory=dict)     # host-side time breakdown of _moe
    steps_meta: list = field(default_factory=list)  # (token_index, tokens, eos)
    layer_trace: list = field(default_factory=list)  # per-layer timeline (cfg.trace_layers)
    cpu_expert_ms: list = field(default_factory=list)  # (rows, ms, kind, t0) per CPU expert (trace_layers)


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


class OffloadEngine(MoEExecMixin, DecodeGraphMixin, EPMoEMixin):
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
        self._gemv_ctr = None                        # fused o-projection + norm counter
        self.shared_stream = torch.cuda.Stream()     # shared experts beside routing (head)
        self.policy_stream = torch.cuda.Stream()     # all-resident decode: policy records
        self._policy_side_used = False
        self.repl_stream = torch.cuda.Stream()       # cache replacement copies (off the
        #                                              demand path: never delays a demand copy)
        # HBM expert cache slots: layer l owns slots [l*slots, (l+1)*slots)
        self.cache_buf = (torch.empty((L * slots, weights.expert_bytes), dtype=torch.uint8,
                                      device=self.dev) if slots else None)
        self.host_slot = self.policy.slot_of.cpu().numpy().copy()
        self.slot_ready = [None] * (L * slots)   # per cache slot: last replacement copy
        self._slot_ptrs = ([self.cache_buf.data_ptr() + s * weights.expert_bytes
                            for s in range(L * slots)] if slots else [])
        self._repl_pend = [dict() for _ in range(L)]   # layer -> {slot: (expert, victim read)}
        self._repl_slot: dict = {}                      # slot -> layer of its pending copy
        self._repl_inflight = collections.deque()       # background copies in flight
        n_stage = cfg.staging_slots or (0 if self.resident_mode else
                                        max(2 * k, N) + 2 * max(cfg.prefetch_size, 1) + 2)
        self.staging = _Staging(n_stage, weights.expert_bytes, self.dev) if n_stage else None
        self.prefetched: dict = {}          # (layer, expert) -> (staging idx, event)
        self.cpu_threads = cfg.cpu_threads or len(os.sched_getaffinity(0))
        # asynchronous CPU experts (dispatcher thread) measured ~12% slower per
        # decode token on the 16-vCPU boxes: the Python thread's GPU dispatch
        # preempts a pool thread and the pool's phase barrier waits for it.
        # Off by default; DALI_CPU_ASYNC=1 enables it.
        # decode-sized CPU experts start on the pool's workers before the GPU
        # dispatch and the Python thread joins them afterwards (DALI_CPU_ASYNC=0:
        # dispatch first, then run them synchronously -- A/B switch)
        self._cpu_async = os.environ.get("DALI_CPU_ASYNC", "1") == "1"
        self._cpu_sub = None                  # preallocated submission arrays (_cpu_submit)
        # offloaded decode: a layer's combine is launched before its CPU experts
        # finish and polls this pinned word (dali_unpermute_combine_wait), which
        # the worker's last unit sets to the layer's sequence number; the join
        # is deferred past the next layer's head
        self._launch_ahead = os.environ.get("DALI_LAUNCH_AHEAD", "1") == "1"
        self._rows_flag = torch.zeros(2, dtype=torch.int64).pin_memory()
        self._rows_flag_p = self._rows_flag.data_ptr()
        self._rows_seq = self._rows_seq_checked = 0
        self._splits_memo: dict = {}
        self._pending_cpu = None              # deferred join of the previous layer
        self._blk_tab = None                  # (L, N) host block addresses (dali_cpu_submit_layer)
        self._sub_args = {}                   # layer -> prebuilt submission arguments
        self._ev_rows = None                  # trace: event before the CPU-row upload
        torch.set_num_threads(self.cpu_threads)
        # per-layer pinned scratch for pointer table + G mask
        row = (N * 17 + 63) // 64 * 64        # ptrs | maps | G mask, 64-B aligned rows
        self.ptr_host = torch.zeros((L, row), dtype=torch.uint8, pin_memory=True)
        self._ptr_host_np = self.ptr_host.numpy()    # same pinned memory
        self.ptr_dev = torch.zeros((L, row), dtype=torch.uint8, device=self.dev)
        # per layer: (device row address, pinned row address, row bytes) -- the
        # decode dispatch reads these instead of indexing the tensors per layer
        self._ptr_rows = [(self.ptr_dev.data_ptr() + l * row, self.ptr_host.data_ptr() + l * row,
                           row) for l in range(L)]
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
        self._wsv: dict = {}                    # (name, shape, dtype, pinned) -> view
        self._ws_retired: list = []             # outgrown workspaces, freed per request
        self._res_maps = None
        self._wl_log = None
        self.desc_dev = torch.zeros((8,), dtype=torch.int32, device=self.dev)
        self.desc_host = torch.zeros((8,), dtype=torch.int32, pin_memory=True)
        self.desc_step_host = torch.zeros((8,), dtype=torch.int32, pin_memory=True)
        self._graph = None
        self._heads: dict = {}              # offloaded decode: layer -> (graph, h, views, kernels)
        self.graph_kernels = 0              # our kernels launched by CUDA-graph replays
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
        wait that follows their previous consumer).

        One flat buffer per (name, dtype, pinned), grown to the largest size
        requested and handed out as a view of the requested shape, so serving
        varied prompt lengths and batches does not accumulate buffers.  A
        growth invalidates the captured CUDA graphs (they hold the old
        addresses; they are re-captured on the next decode step) and parks the
        old buffer until the next request starts, because queued kernels, the
        CPU worker and UVA kernel copies may still use it."""
        v = self._wsv.get((name, shape, dtype, pinned))
        if v is not None:                  # hot path: the same view as last time
            return v
        n = 1
        for x in shape:
            n *= int(x)
        key = (name, dtype, pinned)
        t = self._wsd.get(key)
        if t is None or t.numel() < n:
            if t is not None:
                if self._capturing:
                    raise SimulationError(f"workspace {name!r} grew during graph capture")
                self._ws_retired.append(t)
                self._wsv.clear()          # views of the outgrown buffer
                self._drop_graphs()
            t = (torch.empty((max(n, 1),), dtype=dtype, pin_memory=True) if pinned
                 else torch.empty((max(n, 1),), dtype=dtype, device=self.dev))
            self._wsd[key] = t
        v = t[:n].view(shape)
        self._wsv[(name, shape, dtype, pinned)] = v
        return v

    def _drop_graphs(self) -> None:
        """Forget the captured decode graphs (re-captured on demand)."""
        self._graph = None
        self._graph_warm = False
        self._heads, self._heads_warm = {}, False

    def _map_addr(self, phys: int) -> int:
        return self.maps_dev.data_ptr() + int(phys) * 256

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
        self._repl_pend = [dict() for _ in range(L)]
        self._repl_slot = {}
        self._repl_inflight = collections.deque()
        for key in list(self.prefetched):
            i, ev = self.prefetched.pop(key)
            self.staging.release(i, ev)
        self._load_initial_cache()

    def _host_block(self, l: int, e: int) -> torch.Tensor:
        off = self.w.expert_index(l, e) * self.w.expert_bytes
        return self.w.host.bytes[off:off + self.w.expert_bytes]

    # ------------------------------------------------------------- copies
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
            x2 = torch.empty_like(x)
            if dev_attn:
                self._attn_block(l, x, x2, h, B)
            else:
                _lib.call("dali_add_rmsnorm", x.data_ptr(), None, W.attn_norm[l].data_ptr(),
                          a.rms_eps, T, d, None, hn.data_ptr(), sp)
                att = attention(a, hn, W.wqkv[l], W.wo[l], self.rope, self.kv, l, B, S, pos0)
                _lib.call("dali_add_rmsnorm", x.data_ptr(), att.data_ptr(),
                          W.moe_norm[l].data_ptr(), a.rms_eps, T, d, x2.data_ptr(), h.data_ptr(),
                          sp)
            x = self._moe(l, x2, h, step, token_index, is_eos)
        if self._policy_side_used:              # join the side-stream policy kernels
            self._cur().wait_stream(self.policy_stream)
            self._policy_side_used = False
        last = x.view(B, S, -1)[:, -1]
        return rms_norm(last, W.final_norm, a.rms_eps) @ W.lm_head.t()

    # ------------------------------------------------- offloaded decode (graphs)
    def start_request(self, batch: int) -> np.ndarray:
        """New policy run for one request; cache residency carries over."""
        if self.kv is None or self.kv.k.shape[1] != batch:
            self.kv = KVCache(self.arch, batch, self.max_seq, self.dev)
            self._drop_graphs()
        if self._ws_retired:                    # the previous request has synchronised
            torch.cuda.synchronize()
            self._ws_retired.clear()
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

    def generate(self, prompt: torch.Tensor, max_new_tokens: int, host_io: bool = True,
                 forced: torch.Tensor | None = None):
        """Greedy generation for one request.

        host_io=True (the end-to-end path a user sees): ``prompt`` (B, S)
        int64 on the HOST, copied in inside the timed region, and every
        generated token is read back to the host as it is produced.
        host_io=False: ``prompt`` already in HBM and tokens stay on device.
        ``forced`` (B, max_new_tokens - 1) int64 on the host: teacher forcing --
        decode step i consumes forced[:, i] instead of the argmax (which is
        still computed and returned), so the routed workload does not depend
        on argmax near-ties of a random-weight model (the benchmark uses this
        for a workload that is identical on every box).
        Returns (tokens (B, n) int64, stats)."""
        B, S = prompt.shape
        self._cs_cached = torch.cuda.current_stream()
        self.start_request(B)
        l0, gk0 = _lib.launch_count(), self.graph_kernels
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
        f_pin = f_dev = None
        if forced is not None:
            assert forced.shape == (B, max(max_new_tokens - 1, 0)), "forced must be (B, n - 1)"
            n_f = max(max_new_tokens - 1, 1)
            f_pin = self._ws("forced_h", (n_f, B), torch.int64, pinned=True)
            f_dev = self._ws("forced_d", (n_f, B), torch.int64)
            if max_new_tokens > 1:
                f_pin[:max_new_tokens - 1].copy_(forced.t())
            if not host_io:                     # device-resident inputs: one upload
                f_dev.copy_(f_pin, non_blocking=True)
        logits = self.prefill(p_dev, is_eos=(max_new_tokens <= 1))
        nxt = logits.argmax(-1)
        out = [fetch(nxt, 0)]
        if self.cfg.capture:
            self.stats.logits.append(logits.float().cpu())
        e1.record(cs)
        st0 = self.stats
        copies0 = st0.demand_copies + st0.prefetch_copies + st0.replace_copies
        blocks0 = st0.cpu_expert_calls + copies0
        for i in range(max_new_tokens - 1):
            if f_dev is not None:
                if host_io:                     # this step's input ids: one H2D kernel copy
                    _lib.call("dali_copy_mapped", f_dev[i].data_ptr(), f_pin[i].data_ptr(),
                              B * 8, cs.cuda_stream)
                nxt = f_dev[i].view(nxt.shape)
            logits = self.decode(nxt, is_eos=(i == max_new_tokens - 2))
            nxt = logits.argmax(-1)
            out.append(fetch(nxt, i + 1))
            if self.cfg.capture:
                self.stats.logits.append(logits.float().cpu())
        e2.record(cs)
        e2.synchronize()
        if self._rows_seq != self._rows_seq_checked:
            # a launched-ahead combine that gave up waiting for its CPU rows
            # (4 s of device time) proceeded with whatever the rows held
            self._rows_seq_checked = self._rows_seq
            tmo = C.c_uint64()
            _lib.call("dali_host_wait_timeouts", C.byref(tmo), 1)
            if tmo.value:
                raise SimulationError(f"{tmo.value} decode combines timed out waiting for the "
                                      "host worker's CPU-expert rows")
        if self.ep is not None and self.ep.peer is not None:
            # a peer lost during the last layers' return exchange only sets the
            # mapped error flag; never hand back rows it left half-written
            self.ep.peer.check()
        if self._used_fast:
            self._finish_resident()
        st = self.stats
        st.prefill_ms = e0.elapsed_time(e1)
        st.decode_ms = e1.elapsed_time(e2)
        st.prefill_tokens = B * S
        st.decode_tokens = B * max(max_new_tokens - 1, 0)
        st.dali_launches = _lib.launch_count() - l0 + self.graph_kernels - gk0
        # expert blocks the decode phase streamed out of host DRAM (CPU experts
        # + H2D copies): the shared host-memory roofline of offloaded decode
        copies = st.demand_copies + st.prefetch_copies + st.replace_copies
        st.decode_host_bytes = (st.cpu_expert_calls + copies - blocks0) * self.arch.expert_bytes
        st.decode_h2d_bytes = (copies - copies0) * self.arch.expert_bytes
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
