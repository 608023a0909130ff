"""Expert parallelism: token dispatch / combine exchange over NCCL all-to-all.

Layout: with G ranks, rank r owns routed experts [r*NL, (r+1)*NL) of every
layer (NL = N / G).  Because the routing plan sorts a rank's (token, slot)
rows by expert, the rows for each destination rank are one contiguous range
of the permuted buffer, so the dispatch is a single ``all_to_all_single``
with per-destination split sizes:

  1. counts : all_to_all of the (N,) local histogram with equal splits NL
              -> recv_counts (G, NL): rows each source sends to each local expert
  2. rows   : all_to_all of the permuted bf16 rows (split = rows per owner)
  3. regroup: received rows are ordered (source, local expert); one gather
              (``dali_permute``) regroups them by local expert for the
              grouped FFN -- ``plan_regroup`` builds that permutation
  4. the owner runs the DALI policy + expert execution on its NL experts
              with the GLOBAL workloads sum_s recv_counts[s]
  5. return : expert outputs (fp32 rows) go back through the inverse
              permutation and the reverse all_to_all; the source rank's
              combine kernel applies Eq. (2) exactly as in the 1-GPU path.

The residual prefetch predictor needs next-layer workloads over all ranks'
tokens: the (N,) predicted histogram is all-reduced (sum) before the owner
slices its NL entries.  Everything here is plain torch.distributed, so the
same code runs on NCCL (GPU tensors) and gloo (CPU tensors, tests).
"""

from __future__ import annotations

import time

import numpy as np
import torch

from .. import _lib
from ..errors import SimulationError
from ..trace import route_device
import torch.distributed as dist


class EPGroup:
    def __init__(self, num_experts: int, group=None):
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if num_experts % self.world:
            raise ValueError(f"{num_experts} experts do not split over {self.world} ranks")
        self.N = num_experts
        self.NL = num_experts // self.world
        self.peer = None                 # PeerExchange, built by the engine on first use

    @property
    def local_experts(self) -> list[int]:
        return list(range(self.rank * self.NL, (self.rank + 1) * self.NL))

    # -- collectives -----------------------------------------------------------
    def exchange_counts(self, wl: torch.Tensor) -> torch.Tensor:
        """(N,) local histogram -> (G*NL,) rows each source sends to my experts."""
        out = torch.empty_like(wl)
        dist.all_to_all_single(out, wl.contiguous(), group=self.group)
        return out

    def all_reduce_sum_(self, t: torch.Tensor) -> torch.Tensor:
        dist.all_reduce(t, group=self.group)
        return t

    def exchange_rows(self, send: torch.Tensor, send_sizes: list[int],
                      recv_sizes: list[int]) -> torch.Tensor:
        out = send.new_empty((int(sum(recv_sizes)),) + tuple(send.shape[1:]))
        dist.all_to_all_single(out, send.contiguous(), output_split_sizes=recv_sizes,
                               input_split_sizes=send_sizes, group=self.group)
        return out


# ---------------------------------------------------------------------------
# peer-memory exchange (the product path on one node; NCCL stays as baseline)
# ---------------------------------------------------------------------------

class PeerExchange:
    """Per-rank IPC buffers of the fused EP exchange (csrc/ep.cu): recv /
    ret / cnt / flags of every rank mapped into this process, with device
    pointer tables for the dispatch and return kernels.  ``cap`` = the most
    rows one rank can send another in one layer (tokens x top_k)."""

    MAX_SPINS = 200_000_000            # ~20 s of 64 ns sleeps: a lost peer errors out

    def __init__(self, ep: "EPGroup", cap: int, d: int, device):
        import ctypes as C
        self.ep, self.cap, self.d = ep, int(cap), int(d)
        G, NL = ep.world, ep.NL
        lay = (C.c_int64 * 5)()
        _lib.call("dali_ep_layout", G, NL, self.cap, self.d, lay)
        self.off = list(lay)
        ptr = C.c_void_p()
        handle = (C.c_uint8 * 64)()
        _lib.call("dali_ipc_alloc", self.off[4], C.byref(ptr), handle)
        self.base = int(ptr.value)
        handles = [None] * G
        dist.all_gather_object(handles, bytes(handle), group=ep.group)
        self.opened = []
        bases = []
        for g in range(G):
            if g == ep.rank:
                bases.append(self.base)
                continue
            hp = (C.c_uint8 * 64).from_buffer_copy(handles[g])
            pp = C.c_void_p()
            _lib.call("dali_ipc_open", hp, C.byref(pp))
            self.opened.append(int(pp.value))
            bases.append(int(pp.value))

        def table(off):
            return torch.tensor([b + off for b in bases], dtype=torch.int64, device=device)
        self.peer_recv = table(self.off[0])
        self.peer_ret = table(self.off[1])
        self.peer_cnt = table(self.off[2])
        self.peer_flag_d = table(self.off[3])
        self.peer_flag_r = table(self.off[3] + 8)
        self.recv = self.base + self.off[0]
        self.ret = self.base + self.off[1]
        self.cnt = self.base + self.off[2]
        self.flag_d = self.base + self.off[3]
        self.flag_r = self.base + self.off[3] + 8
        self.epoch = 0
        # timeout flag in mapped pinned memory: the host checks it with no copy
        self.err = torch.zeros((1,), dtype=torch.int32, pin_memory=True)
        dist.barrier(group=ep.group)

    def check(self):
        if int(self.err[0]):
            raise RuntimeError("expert-parallel peer exchange timed out (a rank stopped)")

    def close(self):
        for p in self.opened:
            _lib.load().dali_ipc_close(p)
        self.opened = []


# ---------------------------------------------------------------------------
# host-side planning (pure numpy; tested on CPU)
# ---------------------------------------------------------------------------

def send_sizes(wl: np.ndarray, world: int) -> list[int]:
    """Rows for each destination rank (contiguous expert blocks)."""
    nl = len(wl) // world
    return [int(wl[q * nl:(q + 1) * nl].sum()) for q in range(world)]


def plan_regroup(recv_counts: np.ndarray):
    """recv_counts (G, NL) -> (perm, offsets, recv_sizes).

    Received rows are ordered by (source, local expert).  ``perm[i]`` is the
    received-row index of grouped row i, where grouped rows are ordered by
    (local expert, source); ``offsets`` (NL+1) delimit each local expert's
    rows in the grouped order; ``recv_sizes`` are the per-source row counts.
    """
    rc = np.asarray(recv_counts, dtype=np.int64)
    G, NL = rc.shape
    recv_sz = rc.sum(axis=1)
    src_base = np.concatenate([[0], np.cumsum(recv_sz)[:-1]])
    within = np.concatenate([np.zeros((G, 1), np.int64), np.cumsum(rc, axis=1)[:, :-1]], axis=1)
    perm = []
    for j in range(NL):
        for s in range(G):
            st = src_base[s] + within[s, j]
            perm.extend(range(int(st), int(st + rc[s, j])))
    per_expert = rc.sum(axis=0)
    offsets = np.concatenate([[0], np.cumsum(per_expert)]).astype(np.int32)
    return (np.asarray(perm, dtype=np.int32), offsets, [int(x) for x in recv_sz])


class EPMoEMixin:
    """Expert-parallel MoE layer of ``OffloadEngine`` (dispatch / combine
    exchange around the 1-GPU execution path)."""

    def _moe_ep(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int, token_index: int,
                is_eos: bool) -> torch.Tensor:
        if self.cfg.ep_transport == "p2p":
            return self._moe_ep_p2p(l, x, h, step, token_index, is_eos)
        return self._moe_ep_nccl(l, x, h, step, token_index, is_eos)

    def _moe_ep_p2p(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int,
                    token_index: int, is_eos: bool) -> torch.Tensor:
        """Expert-parallel MoE layer over peer memory (csrc/ep.cu): the
        dispatch kernel gathers this rank's permuted rows straight into the
        owners' receive buffers; owners regroup, decide (DALI policy on the
        GLOBAL workloads) and execute, then the return kernel sums split-K
        planes / takes CPU rows and stores each result into its source's
        return buffer; the source gathers and combines (Eq. 2)."""
        a, ep = self.arch, self.ep
        N, k, d, NL, G = a.num_experts, a.top_k, a.hidden_dim, self.NL, ep.world
        T = h.shape[0]
        cs = self._cur()
        sp = cs.cuda_stream
        tp0 = time.perf_counter()
        if ep.peer is None:
            ep.peer = PeerExchange(ep, self.max_batch * self.max_seq * k, d, self.dev)
        ex = ep.peer
        if T * k > ex.cap:
            raise SimulationError(f"{T * k} rows exceed the EP exchange capacity {ex.cap}")
        ex.epoch += 1
        v = self._route(l, h)
        _lib.call("dali_ep_dispatch", h.data_ptr(), v["perm"].data_ptr(),
                  v["offsets"].data_ptr(), N, NL, G, ep.rank, ex.cap, d, T * k,
                  ex.peer_recv.data_ptr(), ex.peer_cnt.data_ptr(), ex.peer_flag_d.data_ptr(), sp)
        _lib.call("dali_ep_wait", ex.flag_d, ex.epoch * G, PeerExchange.MAX_SPINS,
                  ex.err.data_ptr(), sp)
        perm2 = self._ws("ep_perm2", (G * ex.cap,), torch.int32)
        offs_l = self._ws("ep_offs", (NL + 1,), torch.int32)
        wl_glob = self._ws("ep_wl", (NL,), torch.int64)
        meta = self._ws("ep_meta", (4,), torch.int32)
        xl = self._ws("ep_xl", (G * ex.cap, d), torch.bfloat16)
        _lib.call("dali_ep_recv", ex.cnt, G, NL, ex.cap, ex.recv, d, G * ex.cap,
                  perm2.data_ptr(), offs_l.data_ptr(), wl_glob.data_ptr(), meta.data_ptr(),
                  xl.data_ptr(), sp)
        pred = None
        if self.policy.prefetch_size > 0 and l + 1 < a.num_layers:
            _, _, pw = route_device(h, self.w.router[l + 1], k, residual=self.policy.residuals[l],
                                    want_idx=False, want_weights=False,
                                    norm2=self.w.router_norm2[l + 1])
            pred = ep.all_reduce_sum_(pw)[ep.rank * NL:(ep.rank + 1) * NL].contiguous()
        ri = self.policy.layer_step(step, l, token_index, is_eos, wl_glob, None, None,
                                    predicted=pred)
        hv = self._host_view(v, T)
        cnt_host = self._ws("ep_cnt_h", (G * NL,), torch.int32, pinned=True)
        _lib.call("dali_copy_mapped", cnt_host.data_ptr(), ex.cnt, G * NL * 4, sp)
        if self.cfg.capture:
            h_host = self._ws("h_h", (T, d), torch.bfloat16, pinned=True)
            h_host.copy_(h, non_blocking=True)
        ev_dec = torch.cuda.Event()
        ev_dec.record(cs)
        tp1 = time.perf_counter()
        ev_dec.synchronize()
        tp2 = time.perf_counter()
        ex.check()
        rec = self.policy.record(ri)
        rc = cnt_host.numpy().astype(np.int64).reshape(G, NL)
        wl_np = rc.sum(axis=0)
        R = int(wl_np.sum())
        offs_np = np.concatenate([[0], np.cumsum(wl_np)]).astype(np.int32)
        self.stats.workloads[(step, l)] = wl_np
        if self.cfg.capture:
            self.stats.captured.append((step, l, h_host.clone()))
            self.stats.topk[(step, l)] = hv["idx"].numpy().astype(np.int64).copy()
        yp, splits, gmask_p = self._exec_local(l, xl, offs_l, wl_np, rec, R)
        y_shared = self._shared_ffn(l, h) if self.shared_map_ptr is not None else None
        tp3 = time.perf_counter()
        cpu_rows = None
        if R and np.frombuffer(rec.C, dtype=np.int8, count=NL).any():
            xl_host = self._ws("xl_h", (R, d), torch.bfloat16, pinned=True)
            xl_host.copy_(xl[:R])
            cpu_rows = self._cpu_rows(l, xl_host, offs_np, rec, R)
        tp4 = time.perf_counter()
        self._acct(tp0, tp1, tp2, tp3, tp4)
        _lib.call("dali_ep_return", yp.data_ptr(), splits, yp.shape[1] * d,
                  cpu_rows.data_ptr() if cpu_rows is not None else None, gmask_p,
                  offs_l.data_ptr(), ex.cnt, G, NL, ep.rank, ex.cap, d, G * ex.cap,
                  ex.peer_ret.data_ptr(), ex.peer_flag_r.data_ptr(), sp)
        _lib.call("dali_ep_wait", ex.flag_r, ex.epoch * G, PeerExchange.MAX_SPINS,
                  ex.err.data_ptr(), sp)
        back = self._ws("ep_back", (T * k, d), torch.float32)
        _lib.call("dali_ep_gather_back", ex.ret, v["offsets"].data_ptr(), N, NL, ex.cap, d, T * k,
                  back.data_ptr(), sp)
        out = torch.empty_like(x)
        _lib.call("dali_unpermute_combine", x.data_ptr(), back.data_ptr(), v["idx"].data_ptr(),
                  v["pos"].data_ptr(), v["wts"].data_ptr(), None, None,
                  y_shared.data_ptr() if y_shared is not None else None, T, k, d, 1, T * k,
                  out.data_ptr(), sp)
        return out

    def _moe_ep_nccl(self, l: int, x: torch.Tensor, h: torch.Tensor, step: int,
                     token_index: int, is_eos: bool) -> torch.Tensor:
        """Expert-parallel MoE layer over NCCL (the baseline transport):
        dispatch all-to-all, DALI policy + execution on this rank's NL experts
        with global workloads, return all-to-all, Eq. (2) combine on the
        source rank."""
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
                                    want_idx=False, want_weights=False,
                                    norm2=self.w.router_norm2[l + 1])
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
            cpu_rows = cpu_rows[:R].to(y_l.device)          # pinned host rows -> HBM, once
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
