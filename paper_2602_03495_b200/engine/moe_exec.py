"""MoE-layer execution of the offload engine (mixin of ``OffloadEngine``).

One MoE layer, in the reference driver's order (simulator.py:354-444):
``_moe_head`` queues the device half (route + plan/gather, residual
prediction, fused policy kernel, D2H mirrors); ``_moe_tail`` waits for the
decision record and executes it: GPU experts from an HBM slot, a prefetch
staging slot or a demand copy (``_exec_local``), cache insertions
(``_apply_inserts``), CPU experts on the host worker (``_cpu_submit`` /
``_cpu_finish``), then the Eq. (2) combine.  ``_moe_resident`` is the
all-resident fast path (no host wait).  Split out of ``offload.py``; the
state lives on the engine.
"""

from __future__ import annotations

import ctypes as C
import time

import numpy as np
import torch

from .. import _lib
from ..errors import SimulationError
from ..trace import route_device
from .cpu_worker import NATIVE_MAX_ROWS, cpu_expert_rows
from .weights import h2d_block

_REC_C_OFF = _lib.LayerRecordC.C.offset          # C vector inside dali_layer_record


def ffn_splits(max_rows: int, tiles: int, kb: int, n_sm: int) -> int:
    """Split-K planes of the down projection for dali_expert_ffn_tc: the
    smallest factor dividing f/64 that gives >= 1.5 CTAs per SM (``max_rows``
    is kept for the signature: every token-tile width uses the same rule).
    Measured at Mixtral shapes (tools/prof_ffn.py --splits): one expert runs
    best at 7 planes (224 CTAs), two at 4 (256 CTAs); a full second wave of
    short CTAs costs more in per-CTA prologue/epilogue than it hides."""
    best = 1
    for s in range(1, 17):
        if kb % s == 0:
            best = s
            if 2 * tiles * s >= 3 * n_sm:
                break
    return best



class MoEExecMixin:
    def _shared_ffn(self, l: int, h: torch.Tensor, stream=None) -> torch.Tensor:
        """Shared expert(s) of layer l over all T tokens -> (T, d) f32, on
        ``stream`` (default: the compute stream)."""
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
        cs = self._cur() if stream is None else stream
        _lib.call("dali_expert_ffn_tc", h.data_ptr(), offs.data_ptr(), 1,
                  self.shared_map_ptr.data_ptr() + 8 * l, d, fs, T, T, 1, hs.data_ptr(),
                  ys.data_ptr(), sp, cs.cuda_stream)
        if stream is not None:
            cs = stream
        y = self._ws("sh_out", (T, d), torch.float32)
        _lib.call("dali_shared_finish", ys.data_ptr(), sp, T, d, h.data_ptr(),
                  self.w.shared_gate[l].data_ptr() if a.shared_gate else None, y.data_ptr(),
                  cs.cuda_stream)
        return y

    def _splits_for(self, tiles: int, max_rows: int, ffn_dim: int | None = None) -> int:
        key = (tiles, max_rows, ffn_dim)
        sp = self._splits_memo.get(key)
        if sp is None:
            sp = self._splits_memo[key] = ffn_splits(max_rows, tiles,
                                                     (ffn_dim or self.arch.ffn_dim) // 64,
                                                     self.n_sm)
        return sp

    def _copy_into_staging(self, l: int, e: int, demand: bool = False
                           ) -> tuple[int, torch.cuda.Event]:
        """Expert block (l, e) -> a staging slot on the copy stream.  Demand
        copies (the GPU expert waits for them) always use the copy engine;
        prefetches, like replacements, follow ``EngineConfig.h2d_sm_ctas``
        (default 0 = copy engine; > 0 = the SM-driven copy of
        weights.h2d_block)."""
        i = self.staging.get()
        ev_prev = self.staging.free_after[i]
        if ev_prev is not None:
            self.copy_stream.wait_event(ev_prev)
        h2d_block(self.staging.buf[i], self._host_block(l, e), self.copy_stream,
                  0 if demand else self.cfg.h2d_sm_ctas)
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
        # the all-resident side-stream policy kernel reads this layer's
        # workloads after the next layer's route ran: one block per layer then
        side = self.resident_mode and self.cfg.policy_side_stream
        rblk = self._ws(f"route{l}" if side else "route", (nb,), torch.uint8)
        v = {
            "wl": rblk[:o_off].view(torch.int64),
            "offsets": rblk[o_off:o_off + (N + 1) * 4].view(torch.int32),
            "idx": rblk[o_idx:o_w].view(torch.int32).view(T, k),
            "wts": rblk[o_w:nb].view(torch.float32).view(T, k),
        }
        perm = self._ws("perm", (T * k,), torch.int32)
        v["pos"] = self._ws("pos", (T, k), torch.int32)
        v["xp"] = self._ws("xp", (T * k, d), torch.bfloat16)
        if T <= 16 and self.cfg.fused_route_plan:
            # decode: routing, plan and permute in one launch
            _lib.call("dali_route_plan_bf16", h.data_ptr(), self.w.router[l].data_ptr(),
                      self.w.router_norm2[l].data_ptr(), T, d, N, k, int(a.norm_topk_prob),
                      v["idx"].data_ptr(), v["wts"].data_ptr(), v["wl"].data_ptr(),
                      v["offsets"].data_ptr(), perm.data_ptr(), v["pos"].data_ptr(),
                      v["xp"].data_ptr(), cs.cuda_stream)
        else:
            route_device(h, self.w.router[l], k, renorm=a.norm_topk_prob,
                         out=(v["idx"], v["wts"], v["wl"]), norm2=self.w.router_norm2[l])
            _lib.call("dali_moe_plan_permute", v["idx"].data_ptr(), T, k, N, h.data_ptr(), d,
                      v["offsets"].data_ptr(), perm.data_ptr(), v["pos"].data_ptr(),
                      v["xp"].data_ptr(), cs.cuda_stream)
        v["blk"], v["layout"], v["perm"] = rblk, (o_off, o_idx, o_w, nb), perm
        return v

    def _d2h(self, dst: torch.Tensor, src: torch.Tensor) -> None:
        """Device -> pinned host mirror on the compute stream.  Decode-sized
        mirrors (<= 1 MiB) are kernel copies over UVA (no copy-engine launch
        latency on the decision path); prefill-sized ones use the copy engine."""
        nbytes = src.numel() * src.element_size()
        if nbytes <= (1 << 20):
            _lib.call("dali_copy_mapped", dst.data_ptr(), src.data_ptr(), nbytes,
                      self._cur().cuda_stream)
        else:
            dst.copy_(src, non_blocking=True)

    def _host_view(self, v, T: int, xp=None):
        """Pinned host mirror of the routing block (valid after the event wait).
        xp = (pinned dst, device src): the permuted rows, mirrored in the same
        kernel launch when both fit the kernel-copy path."""
        N, k = self.arch.num_experts, self.arch.top_k
        o_off, o_idx, o_w, nb = v["layout"]
        hb = self._ws("route_h", (nb,), torch.uint8, pinned=True)
        src = v["blk"]
        xd, xs = xp if xp is not None else (None, None)
        nx = xs.numel() * xs.element_size() if xs is not None else 0
        nr = src.numel() * src.element_size()
        if xs is not None and nx + nr <= (1 << 20) and not (
                (hb.data_ptr() | src.data_ptr() | xd.data_ptr() | xs.data_ptr()) & 15):
            _lib.call("dali_copy_mapped2", hb.data_ptr(), src.data_ptr(), nr, xd.data_ptr(),
                      xs.data_ptr(), nx, self._cur().cuda_stream)
        else:
            self._d2h(hb, src)
            if xs is not None:
                self._d2h(xd, xs)
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
        pd_addr, ph_addr, row_bytes = self._ptr_rows[l]
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
                if s in self._repl_slot:           # admitted, copy not issued yet
                    self._issue_repl(s, urgent=True)
                ptrs[e] = self._slot_ptrs[s]
                maps[e] = self._map_addr(s)
                if self.slot_ready[s] is not None:
                    waits.append(self.slot_ready[s])
                n_hit += 1
                continue
            if (l, e) in self.prefetched:
                i, ev = self.prefetched.pop((l, e))
                n_pf += 1
            else:
                i, ev = self._copy_into_staging(l, e, demand=True)
                self.stats.demand_copies += 1
                n_dem += 1
            ptrs[e] = self.staging.ptr(i)
            maps[e] = self._map_addr(self.n_cache_slots + i)
            waits.append(ev)
            used_staging.append(i)
            stage_of[e] = i
        # kernel copy from mapped pinned memory: never queues behind expert DMA
        _lib.call("dali_copy_mapped", pd_addr, ph_addr, row_bytes, cs.cuda_stream)
        splits = 1
        max_rows = 0
        if G and self.use_tc:
            wg = [int(wl_np[e]) for e in G]
            max_rows = max(wg)
            bn = 16 if max_rows <= 16 else 32 if max_rows <= 32 else 64 if max_rows <= 64 \
                else 128 if max_rows <= 128 else 256
            tiles = sum((w_ + bn - 1) // bn for w_ in wg) * (d // 128)
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
                          pd_addr + NL * 8, d, f, R, max_rows, len(G),
                          hbuf.data_ptr(), yp.data_ptr(), splits, cs.cuda_stream)
            else:
                _lib.call("dali_expert_ffn", xrows.data_ptr(), offsets.data_ptr(), NL,
                          pd_addr, d, f, R, R, hbuf.data_ptr(), yp.data_ptr(),
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
            if rec.ev_valid and rec.ev_n and self.cfg.lazy_replace:
                for j in range(rec.ev_n):
                    v_, c_ = int(rec.evicted[j]), int(rec.admitted[j])
                    s = int(self.host_slot[l, v_])
                    self._defer_repl(l, s, c_, ffn_done)
                    self.host_slot[l, c_], self.host_slot[l, v_] = s, -1
            elif rec.ev_valid and rec.ev_n:
                with torch.cuda.stream(self.repl_stream):
                    self.repl_stream.wait_event(ffn_done)
                    for j in range(rec.ev_n):
                        v_, c_ = int(rec.evicted[j]), int(rec.admitted[j])
                        s = self.host_slot[l, v_]
                        h2d_block(self.cache_buf[s], self._host_block(l, c_),
                                  self.repl_stream, self.cfg.h2d_sm_ctas)
                        self.host_slot[l, c_], self.host_slot[l, v_] = s, -1
                        self.stats.h2d_bytes += self.w.expert_bytes
                        self.stats.replace_copies += 1
                        ev = torch.cuda.Event()
                        ev.record(self.repl_stream)
                        self.slot_ready[s] = ev
        if self._repl_slot:
            self._pump_repl(l)
        self._last_exec = dict(hit=n_hit, pf=n_pf, dem=n_dem, t0=t0_ev,
                               rep=int(rec.ev_n) if (rec.ev_valid and not self.resident_mode) else 0,
                               done=int(rec.n_done) if not self.resident_mode else 0)
        return yp, splits, pd_addr + NL * 16

    # ------------------------------------------------ deferred replacements
    # EngineConfig.lazy_replace: a window replacement (the workload-aware
    # cache admitting expert c into the victim's slot, simulator.py window
    # swap) is recorded here instead of being copied at once.  The copy is
    # issued (a) at once, on the demand stream, when a later decision hits
    # that slot, or (b) in the background, at most `_repl_max` at a time,
    # in next-use order (the layers after the current one first).  A slot
    # whose pending admission is evicted again before any read is never
    # copied.  The decisions and the bytes every FFN reads are unchanged;
    # what changes is that a boundary token's ~8 admissions per layer no
    # longer sit in one FIFO in front of the few the next token hits.
    # Background depth (EngineConfig.repl_inflight, -1 = by block size): 0 --
    # copy only on a hit -- for blocks that cross PCIe in well under a layer
    # (DSV2 17 MB, Qwen 8 MB: background copies only compete with the
    # critical demand copies; measured 0 > 1 > 2 > 4), 1 for blocks that take
    # longer than a layer (Mixtral 352 MB, 6.3 ms: a copy started on the hit
    # would stall the layer for all of it).
    @property
    def _repl_max(self) -> int:
        n = self.cfg.repl_inflight
        return n if n >= 0 else (0 if self.w.expert_bytes <= (64 << 20) else 1)

    def _defer_repl(self, l: int, s: int, expert: int, ev_free) -> None:
        if s in self._repl_slot:                   # superseded before any read
            self._drop_repl(s)
            self.stats.replace_dropped += 1
        self._repl_pend[l][s] = (expert, ev_free)
        self._repl_slot[s] = l

    def _drop_repl(self, s: int) -> None:
        l = self._repl_slot.pop(s, None)
        if l is not None:
            del self._repl_pend[l][s]

    def _issue_repl(self, s: int, urgent: bool) -> None:
        l = self._repl_slot.pop(s)
        expert, ev_free = self._repl_pend[l].pop(s)
        st = self.copy_stream if urgent else self.repl_stream
        st.wait_event(ev_free)                     # the victim's last read
        if self.slot_ready[s] is not None:         # an earlier copy into the slot
            st.wait_event(self.slot_ready[s])
        h2d_block(self.cache_buf[s], self._host_block(l, expert), st, self.cfg.h2d_sm_ctas)
        ev = torch.cuda.Event()
        ev.record(st)
        self.slot_ready[s] = ev
        self.stats.h2d_bytes += self.w.expert_bytes
        self.stats.replace_copies += 1
        if urgent:
            self.stats.replace_urgent += 1
        else:
            self._repl_inflight.append(ev)

    def _pump_repl(self, l: int) -> None:
        """Keep `_repl_max` background replacement copies in flight, next
        use first: layers l+1, l+2, ... (wrapping into the next token)."""
        q = self._repl_inflight
        while q and q[0].query():
            q.popleft()
        budget = self._repl_max - len(q)
        L = self.arch.num_layers
        for dl in range(1, L + 1):
            if budget <= 0 or not self._repl_slot:
                return
            pend = self._repl_pend[(l + dl) % L]
            while pend and budget > 0:
                self._issue_repl(next(iter(pend)), urgent=False)
                budget -= 1

    def flush_replacements(self) -> None:
        """Issue every deferred replacement copy (background stream)."""
        for l in range(self.arch.num_layers):
            while self._repl_pend[l]:
                self._issue_repl(next(iter(self._repl_pend[l])), urgent=False)

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
            if s in self._repl_slot:               # its pending admission is evicted
                self._drop_repl(s)
                self.stats.replace_dropped += 1
            with torch.cuda.stream(self.repl_stream):
                if self.slot_ready[s] is not None:
                    self.repl_stream.wait_event(self.slot_ready[s])
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
        the layer meanwhile; prefill-sized ones are returned for the
        synchronous AMX path.  Returns the job description for
        ``_cpu_finish``.  This sits on the decode critical path between the decision and the first CPU byte,
        so the submission arrays are preallocated and filled in place."""
        C = np.frombuffer(rec.C, dtype=np.int8, count=self.NL)
        if R == 0 or not C.any():
            return None
        a = self.arch
        d, f = a.hidden_dim, a.ffn_dim
        out = self._ws("cpu_rows_h", (R, d), torch.float32, pinned=True)
        sub = self._cpu_sub
        if sub is None:
            arrs = (np.zeros(self.NL, np.uint64), np.zeros(self.NL, np.uint64),
                    np.zeros(self.NL, np.int32), np.zeros(self.NL, np.uint64))
            sub = self._cpu_sub = (arrs, tuple(x.ctypes.data for x in arrs),
                                   _lib.load().dali_cpu_expert_submit)
        (blocks, xs, rows, ys), addrs, submit = sub
        xbase, obase = rows_host.data_ptr(), out.data_ptr()
        n, big = 0, []
        lo, hi = R, 0
        for e in np.flatnonzero(C).tolist():
            r0, r1 = int(offs_np[e]), int(offs_np[e + 1])
            if r1 <= r0:
                continue
            self.stats.cpu_expert_calls += 1
            lo, hi = min(lo, r0), max(hi, r1)
            if r1 - r0 > NATIVE_MAX_ROWS:
                big.append((e, r0, r1))
            elif self._cpu_async:
                blocks[n] = self.w.expert_host_ptr(l, e)
                xs[n] = xbase + r0 * d * 2
                rows[n] = r1 - r0
                ys[n] = obase + r0 * d * 4
                n += 1
            else:                                   # synchronous (A/B switch)
                t0 = time.perf_counter()
                cpu_expert_rows(self._host_block(l, e).view(torch.bfloat16),
                                rows_host[r0:r1], d, f, self.cpu_threads, out=out[r0:r1])
                if self.cfg.trace_layers:
                    self.stats.cpu_expert_ms.append((r1 - r0, (time.perf_counter() - t0) * 1e3,
                                                     "native", t0))
        if n:
            _lib.check(submit(n, addrs[0], addrs[1], addrs[2], addrs[3], d, f, self.cpu_threads),
                       "dali_cpu_expert_submit")
        return dict(out=out, native=n > 0, big=big, lo=lo, hi=hi, l=l, rows=rows_host)

    def _cpu_submit_layer(self, l: int, rows_host: torch.Tensor, offs_host: torch.Tensor, rec,
                          R: int):
        """Decode fast path of ``_cpu_submit``: one native call reads the
        record's C vector and the offsets mirror, starts the layer's CPU
        experts and arms the completion word the launched-ahead combine polls
        (dali_cpu_submit_layer).  Returns the job (None: no CPU expert) or
        False when an expert is prefill-sized (nothing started)."""
        a = self.arch
        d = a.hidden_dim
        ent = self._sub_args.get(l)
        if ent is None:
            if self._blk_tab is None:
                self._blk_tab = np.array([[self.w.expert_host_ptr(ll, e) for e in range(self.NL)]
                                          for ll in range(a.num_layers)], dtype=np.uint64)
            n = C.c_int32()
            ent = (_lib.load().dali_cpu_submit_layer, n, C.byref(n),
                   self._blk_tab[l].ctypes.data)
            self._sub_args[l] = ent
        fn, n, n_ref, tab_p = ent
        out = self._ws("cpu_rows_h", (R, d), torch.float32, pinned=True)   # grow-only: re-fetch
        self._rows_seq += 1
        _lib.check(fn(C.addressof(rec) + _REC_C_OFF, offs_host.data_ptr(), self.NL, tab_p,
                      rows_host.data_ptr(), out.data_ptr(), d, a.ffn_dim, self.cpu_threads,
                      self._rows_flag_p, self._rows_seq, n_ref), "dali_cpu_submit_layer")
        if n.value < 0:
            return False
        if n.value == 0:
            return None
        self.stats.cpu_expert_calls += n.value
        return dict(out=out, native=True, big=[], seq=self._rows_seq)

    def _join_pending(self) -> None:
        """Join the previous decode layer's CPU experts (this thread takes the
        remaining work units).  Its combine was launched ahead and waits on
        the completion word, so nothing else is left to do here."""
        job = self._pending_cpu
        if job is None:
            return
        self._pending_cpu = None
        t0 = time.perf_counter()
        _lib.call("dali_cpu_expert_wait")
        pr = self.stats.host_ms
        pr["cpu_experts"] = pr.get("cpu_experts", 0.0) + (time.perf_counter() - t0) * 1e3

    def _cpu_finish(self, job, R: int) -> torch.Tensor | None:
        """Run the prefill-sized CPU experts and join the asynchronous ones;
        returns the pinned (R, d) f32 rows, which device kernels read over UVA."""
        if job is None:
            return None
        a = self.arch
        d, f = a.hidden_dim, a.ffn_dim
        out = job["out"]
        if job["native"]:
            _lib.call("dali_cpu_expert_wait")       # join the pool before the AMX experts use it
        for e, r0, r1 in job["big"]:
            t0 = time.perf_counter()
            cpu_expert_rows(self._host_block(job["l"], e).view(torch.bfloat16),
                            job["rows"][r0:r1], d, f, self.cpu_threads, out=out[r0:r1])
            if self.cfg.trace_layers:
                self.stats.cpu_expert_ms.append((r1 - r0, (time.perf_counter() - t0) * 1e3,
                                                 "big", t0))
        if self.cfg.trace_layers:
            self._ev_rows = torch.cuda.Event(enable_timing=True)
            self._ev_rows.record(self._cur())
        # the consumer kernel (combine / EP return) reads the rows straight from
        # the pinned buffer over UVA: no separate upload kernel and PCIe round
        # trip on the critical path.  The buffer is rewritten only by the next
        # layer's CPU experts, which start after that layer's decision event --
        # i.e. after the device has passed this layer's consumer.
        return out

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
        ev_sh = y_shared = None
        if self.shared_map_ptr is not None and self.cfg.shared_in_head:
            # the shared expert(s) need only h: they run on a side stream beside
            # routing + policy (joined at the end of the head, inside the
            # per-layer decode graph), off the host's post-decision critical path
            ss = self.shared_stream
            ss.wait_stream(cs)
            y_shared = self._shared_ffn(l, h, stream=ss)
            ev_sh = torch.cuda.Event()
            ev_sh.record(ss)
        v = self._route(l, h)
        gate_next = self.w.router[l + 1] if l + 1 < a.num_layers else None
        nn2 = self.w.router_norm2[l + 1] if l + 1 < a.num_layers else None
        if use_desc:
            pol = self.policy
            pred_p = pol.predicted_ptr(l, h, gate_next, rec_index=pol.n_records + l,
                                       gate_next_norm2=nn2)
            probs_p, n_tok = pol.gate_probs_ptr(h, self.w.router[l])
            _lib.call("dali_policy_layer_desc", C.addressof(pol.cfg), C.addressof(pol.cm_c), l,
                      self.desc_dev.data_ptr(), v["wl"].data_ptr(), pred_p,
                      pol.on_gpu.data_ptr(), pol.scores.data_ptr(), pol.counters.data_ptr(),
                      pol.arrived.data_ptr(), pol.slot_of.data_ptr(), pol.lru_state.data_ptr(),
                      probs_p, n_tok, pol.record_ptr(0), cs.cuda_stream)
            ri = None
        else:
            ri = self.policy.layer_step(step, l, token_index, is_eos, v["wl"], h, gate_next,
                                        gate_this=self.w.router[l], gate_next_norm2=nn2)
        xp_host = self._ws("xp_h", (R, d), torch.bfloat16, pinned=True)
        hv = self._host_view(v, T, xp=(xp_host, v["xp"]))
        h_host = None
        if self.cfg.capture:
            h_host = self._ws("h_h", (T, d), torch.bfloat16, pinned=True)
            h_host.copy_(h, non_blocking=True)
        if ev_sh is not None:
            cs.wait_event(ev_sh)
        return dict(v=v, hv=hv, xp_host=xp_host, h_host=h_host, ri=ri, T=T, y_shared=y_shared)

    def _moe_tail(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int, views: dict,
                  tp0: float, ev_r, out: torch.Tensor, ahead: bool = False) -> torch.Tensor:
        """Host half: wait for the decision record, execute it (GPU experts
        from cache / staging / demand copy, prefetch + replacement copies, CPU
        experts on the host worker) and queue the Eq. (2) combine into ``out``.

        ahead=True (offloaded decode): the CPU experts start through
        dali_cpu_submit_layer and the combine is launched at once, polling the
        worker's completion word on the device; the join is left to the
        caller (``_join_pending`` after it queued the next layer's head), so
        the device runs combine -> next attention -> routing -> policy as soon
        as the last CPU row lands, with no host round trip in between."""
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
        offs_np = hv["offsets"].numpy()
        # the CPU experts start first on the pool's workers while this thread
        # dispatches the GPU experts and copies of the same layer; _cpu_finish
        # then joins the pool (this thread takes the remaining work units).
        # DALI_CPU_ASYNC=0: GPU work first, then the CPU experts synchronously.
        job = None
        if ahead:
            job = self._cpu_submit_layer(l, xp_host, hv["offsets"], rec, R)
            if job is False:                        # prefill-sized expert: generic path
                ahead, job = False, None
        if not ahead and self._cpu_async:
            job = self._cpu_submit(l, xp_host, offs_np, rec, R)
        tp_sub = time.perf_counter()
        try:
            wl_np = hv["wl"].numpy().copy()
            self.stats.workloads[(step, l)] = wl_np
            if self.cfg.capture:
                self.stats.captured.append((step, l, views["h_host"].clone()))
                self.stats.topk[(step, l)] = hv["idx"].numpy().astype(np.int64).copy()
            yp, splits, gmask_p = self._exec_local(l, v["xp"], v["offsets"], wl_np, rec, R)
            y_shared = views.get("y_shared")
            if y_shared is None and self.shared_map_ptr is not None:
                y_shared = self._shared_ffn(l, h)
        except BaseException:
            if job is not None and job["native"]:
                _lib.load().dali_cpu_expert_wait()     # never leave a job in flight
            raise
        tp3 = time.perf_counter()
        if ahead:
            cpu_rows = job["out"] if job is not None else None
            self._pending_cpu = job
        else:
            if not self._cpu_async:
                job = self._cpu_submit(l, xp_host, offs_np, rec, R)
            cpu_rows = self._cpu_finish(job, R)
        tp4 = time.perf_counter()
        self._acct(tp0, tp1, tp2, tp3, tp4)
        _lib.call("dali_unpermute_combine_wait", x.data_ptr(), yp.data_ptr(), v["idx"].data_ptr(),
                  v["pos"].data_ptr(), v["wts"].data_ptr(), gmask_p,
                  cpu_rows.data_ptr() if cpu_rows is not None else None,
                  y_shared.data_ptr() if y_shared is not None else None, T, k, d, splits,
                  R, out.data_ptr(), self._rows_flag_p if (ahead and job is not None) else None,
                  job["seq"] if (ahead and job is not None) else 0, cs.cuda_stream)
        if self.cfg.capture_moe_io:
            self._capture_io(step, l, x, out)
        if tr:
            ev_c = torch.cuda.Event(enable_timing=True)
            ev_c.record(cs)
            le = self._last_exec
            self.stats.layer_trace.append(dict(
                step=step, layer=l, T=T, nC=int(sum(1 for e in range(N) if rec.C[e] and wl_np[e])),
                hit=le["hit"], pf=le["pf"], dem=le["dem"], rep=le["rep"], done=le["done"],
                host=(tp0, tp1, tp2, tp3, tp4, time.perf_counter()), tp_sub=tp_sub,
                ev_rows=self._ev_rows if (cpu_rows is not None and not ahead) else None,
                ev=(ev_r if ev_r is not None else ev_dec, ev_dec, le["t0"], ev_c)))
        return out

    def _capture_io(self, step: int, l: int, x: torch.Tensor, out: torch.Tensor) -> None:
        """Stream-ordered host copies of one MoE layer's residual input and
        output (read by the tests after the request synchronises)."""
        xi = torch.empty(x.shape, dtype=x.dtype, pin_memory=True)
        xo = torch.empty(out.shape, dtype=out.dtype, pin_memory=True)
        xi.copy_(x, non_blocking=True)
        xo.copy_(out, non_blocking=True)
        self.stats.moe_io.append((step, l, xi, xo))

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
        ev_sh = y_shared = None
        if self.shared_map_ptr is not None and self.cfg.shared_in_head:
            # shared expert(s) beside routing + the routed FFN (they need only h):
            # at decode they stream their weights while routing leaves HBM idle,
            # at prefill they fill the SMs routing leaves free
            ss = self.shared_stream
            ss.wait_stream(cs)
            y_shared = self._shared_ffn(l, h, stream=ss)
            ev_sh = torch.cuda.Event()
            ev_sh.record(ss)
        v = self._route(l, h)
        if T == self.kv.k.shape[1] and self.stats.steps_meta:     # decode: device descriptor
            ri = self.policy.n_records + l
            ps = cs
            if self.cfg.policy_side_stream:
                # nothing downstream of the decision reads it here (every expert is
                # resident, the FFN uses the static map table): the policy kernel
                # runs beside the layer; _forward joins before the step advances
                ps = self.policy_stream
                ps.wait_stream(cs)
                self._policy_side_used = True
            _lib.call("dali_policy_layer_desc", C.addressof(self.policy.cfg),
                      C.addressof(self.policy.cm_c), l, self.desc_dev.data_ptr(),
                      v["wl"].data_ptr(), None, self.policy.on_gpu.data_ptr(),
                      self.policy.scores.data_ptr(), self.policy.counters.data_ptr(),
                      self.policy.arrived.data_ptr(), self.policy.slot_of.data_ptr(),
                      self.policy.lru_state.data_ptr(), None, 0, self.policy.record_ptr(0),
                      ps.cuda_stream)
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
        if ev_sh is not None:
            cs.wait_event(ev_sh)
        elif self.shared_map_ptr is not None:
            y_shared = self._shared_ffn(l, h)
        out = torch.empty_like(x)
        _lib.call("dali_unpermute_combine", x.data_ptr(), yp.data_ptr(), v["idx"].data_ptr(),
                  v["pos"].data_ptr(), v["wts"].data_ptr(), None, None,
                  y_shared.data_ptr() if y_shared is not None else None, T, k, d, splits, R,
                  out.data_ptr(), cs.cuda_stream)
        if self.cfg.capture_moe_io and not self._in_capture:
            self._capture_io(step, l, x, out)
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
