"""Decode steps of the offload engine (mixin of ``OffloadEngine``): the
head_dim 64/128 decode attention (GEMV projections, fused RoPE/KV append,
split-K attention reading the device step descriptor), the offloaded decode
with one CUDA graph per layer for the device half, and the all-resident
decode as one CUDA graph per step.  Split out of ``offload.py``."""

from __future__ import annotations

import math
import time

import torch

from .. import _lib
from ..errors import SimulationError
from .layers import rms_norm


class DecodeGraphMixin:
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
        o = self._attn_core(l, qkv, B)
        if B <= 8:
            att = self._ws("att_dec", (B, a.hidden_dim), torch.bfloat16)
            _lib.call("dali_gemv_bf16", o.data_ptr(), W.wo[l].data_ptr(), B, a.hidden_dim,
                      H * hd, att.data_ptr(), sp)
            return att
        return o @ W.wo[l].t()

    def _attn_core(self, l: int, qkv: torch.Tensor, B: int) -> torch.Tensor:
        """Fused RoPE + KV append and split-K decode attention -> o (B, H*hd)."""
        a = self.arch
        H, KV, hd = a.num_heads, a.num_kv_heads, a.head_dim
        sp = self._cur().cuda_stream
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
        return o

    def _attn_block(self, l: int, X: torch.Tensor, X2: torch.Tensor, h: torch.Tensor,
                    B: int) -> None:
        """Whole decode attention block of layer l: X2 = X + attn(RMSNorm(X)),
        h = RMSNorm(X2).  With the fused GEMVs (B <= 8) the input norm runs
        inside the qkv projection and the residual add + MoE norm in the
        o-projection's last CTA (dali_gemv_norm_bf16): two launches fewer per
        layer than the separate add_rmsnorm kernels, bit-identical results."""
        a, W = self.arch, self.w
        d = a.hidden_dim
        sp = self._cur().cuda_stream
        if not (B <= 8 and self.cfg.fused_norm_gemv):
            hn = self._ws("hn", (B, d), torch.bfloat16)
            _lib.call("dali_add_rmsnorm", X.data_ptr(), None, W.attn_norm[l].data_ptr(),
                      a.rms_eps, B, d, None, hn.data_ptr(), sp)
            att = self._attn_decode(l, hn, B)
            _lib.call("dali_add_rmsnorm", X.data_ptr(), att.data_ptr(), W.moe_norm[l].data_ptr(),
                      a.rms_eps, B, d, X2.data_ptr(), h.data_ptr(), sp)
            return
        H, KV, hd = a.num_heads, a.num_kv_heads, a.head_dim
        nqkv = (H + 2 * KV) * hd
        if self._gemv_ctr is None:
            self._gemv_ctr = torch.zeros(1, dtype=torch.int32, device=self.dev)
        qkv = self._ws("qkv_dec", (B, nqkv), torch.bfloat16)
        _lib.call("dali_gemv_norm_bf16", X.data_ptr(), W.wqkv[l].data_ptr(), B, nqkv, d,
                  qkv.data_ptr(), W.attn_norm[l].data_ptr(), a.rms_eps, None, None, None, None,
                  None, sp)
        o = self._attn_core(l, qkv, B)
        att = self._ws("att_dec", (B, d), torch.bfloat16)
        _lib.call("dali_gemv_norm_bf16", o.data_ptr(), W.wo[l].data_ptr(), B, d, H * hd,
                  att.data_ptr(), None, a.rms_eps, X.data_ptr(), W.moe_norm[l].data_ptr(),
                  X2.data_ptr(), h.data_ptr(), self._gemv_ctr.data_ptr(), sp)

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
        h = self._ws("h", (B, d), torch.bfloat16)
        self._attn_block(l, X, X2, h, B)
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
        # launch-ahead: layer l's combine is queued before its CPU experts are
        # joined (it polls their completion word on the device), then layer
        # l+1's head graph, and only then does this thread join layer l's CPU
        # work -- the device chain starts the moment the last CPU row lands
        ahead = self._launch_ahead and self._cpu_async and self.policy.prefetch_kind != "random"
        try:
            self._decode_layers(L, X, X2, B, step, heads, capture, ahead)
        finally:
            self._join_pending()
        self._heads_warm = True
        self.policy.n_records = base + L
        return rms_norm(X, W.final_norm, a.rms_eps) @ W.lm_head.t()

    def _decode_layers(self, L: int, X: torch.Tensor, X2: torch.Tensor, B: int, step: int,
                       heads: dict, capture: bool, ahead: bool) -> None:
        cs = self._cur()
        for l in range(L):
            ev_r = None
            if self.cfg.trace_layers:
                ev_r = torch.cuda.Event(enable_timing=True)
                ev_r.record(cs)
            tq = time.perf_counter()
            if l in heads:
                g, h, views, nk = heads[l]
                g.replay()
                self.graph_kernels += nk
            elif capture:
                g = torch.cuda.CUDAGraph()
                self._capturing = True
                k0 = _lib.launch_count()
                try:
                    with torch.cuda.graph(g):
                        h, views = self._decode_head(l, X, X2, B)
                finally:
                    self._capturing = False
                nk = _lib.launch_count() - k0         # our kernels in the graph body
                g.replay()
                self.graph_kernels += nk
                heads[l] = (g, h, views, nk)
            else:
                h, views = self._decode_head(l, X, X2, B)
            tl = time.perf_counter()
            self._join_pending()                     # layer l-1's CPU experts
            # launch time of the head, excluding the join (accounted as CPU time)
            tp0 = time.perf_counter() - (tl - tq)
            self._moe_tail(l, X2, h, step, views, tp0, ev_r, X, ahead=ahead)

    def _set_desc(self, step: int, token_index: int, eos_at: int, rec_index: int, pos: int):
        """Write the device step descriptor (stream-ordered kernel copy from
        pinned memory: never queued behind expert DMA on a copy engine)."""
        dh = self.desc_host
        dh.copy_(torch.tensor([step, token_index, eos_at, rec_index, pos, pos + 1,
                               self.arch.num_layers, 0], dtype=torch.int32))
        _lib.call("dali_copy_mapped", self.desc_dev.data_ptr(), dh.data_ptr(), 32,
                  self._cur().cuda_stream)

    def _graphable(self) -> bool:
        return (self.resident_mode and self.use_tc and self.cfg.resident_fast and
                self.cfg.use_graph and self.arch.head_dim == 128 and self.ep is None and
                not self.cfg.capture)

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
            self.graph_kernels += self._graph_nk
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
        k0 = _lib.launch_count()
        with torch.cuda.graph(g):
            out = self._forward(self._graph_in.view(B, 1), B, 1, 0, 0, 0, False)
            _lib.call("dali_step_advance", self.desc_dev.data_ptr(),
                      self._cur().cuda_stream)
        self._graph_nk = _lib.launch_count() - k0
        self._in_capture = False
        self._capturing = False
        self.cfg.time_ffn = saved
        self.policy.n_records = n0
        self._graph, self._graph_logits = g, out
        g.replay()
        self.graph_kernels += self._graph_nk
        self.policy.n_records += L
        return out
