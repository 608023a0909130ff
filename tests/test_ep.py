"""Expert-parallel dispatch/combine logic on CPU (gloo, world_size 2).

Each rank routes its own tokens (reference gating), dispatches the permuted
rows to the owners of their experts with all_to_all_single, the owner runs
its experts (fp32 SwiGLU of the engine's block layout) on rows regrouped by
``plan_regroup``, results return by the reverse all-to-all and the source
applies Eq. (2).  The result must equal a single-process MoE over the same
tokens -- the correctness-by-construction check for the NCCL path."""

import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_03495_b200.engine.ep import plan_regroup, send_sizes

D, F, N, K = 64, 128, 8, 2


def _blocks():
    g = torch.Generator().manual_seed(7)
    return [(torch.randn(3 * F * D, generator=g) * 0.05) for _ in range(N)]


def _gate():
    return np.random.default_rng(3).normal(size=(D, N))


def _tokens(rank, T):
    g = torch.Generator().manual_seed(100 + rank)
    return torch.randn(T, D, generator=g)


def _moe_reference(x, blocks, gate):
    from oracle import model_cpu as M
    from oracle import policy as P
    idx, sc, _ = P.route(x.double().numpy(), gate, K)
    sc = sc / sc.sum(1, keepdims=True)
    y = torch.zeros_like(x)
    for t in range(x.shape[0]):
        for j in range(K):
            y[t] += float(sc[t, j]) * M.expert_forward(x[t:t + 1], blocks[idx[t, j]], D, F)[0]
    return y


def test_plan_regroup_hand_case():
    rc = np.array([[2, 0, 1], [1, 3, 0]])          # (G=2 sources, NL=3 local experts)
    perm, offs, recv = plan_regroup(rc)
    # received order: src0 [e0 e0 | e2], src1 [e0 | e1 e1 e1]
    assert recv == [3, 4]
    assert offs.tolist() == [0, 3, 6, 7]
    assert perm.tolist() == [0, 1, 3, 4, 5, 6, 2]
    assert send_sizes(np.array([1, 2, 3, 4, 5, 6]), 2) == [6, 15]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from oracle import model_cpu as M
    from oracle import policy as P
    from paper_2602_03495_b200.engine.ep import EPGroup
    ep = EPGroup(N)
    blocks, gate = _blocks(), _gate()
    x = _tokens(rank, 5 + 3 * rank)
    T = x.shape[0]
    idx, sc, wl = P.route(x.double().numpy(), gate, K)
    sc = sc / sc.sum(1, keepdims=True)
    order = np.argsort(idx.reshape(-1), kind="stable")           # plan: stable by expert
    pos = np.empty(T * K, np.int64)
    pos[order] = np.arange(T * K)
    xp = x[torch.from_numpy(order // K)]
    rc = ep.exchange_counts(torch.from_numpy(wl)).view(ep.world, ep.NL).numpy()
    perm2, offs, recv_sz = plan_regroup(rc)
    snd = send_sizes(wl, ep.world)
    recv_x = ep.exchange_rows(xp, snd, recv_sz)
    xl = recv_x[torch.from_numpy(perm2.astype(np.int64))]
    yl = torch.zeros_like(xl)
    for j in range(ep.NL):
        r0, r1 = offs[j], offs[j + 1]
        if r1 > r0:
            yl[r0:r1] = M.expert_forward(xl[r0:r1], blocks[ep.local_experts[j]], D, F)
    y_recv = torch.empty_like(yl)
    y_recv.index_copy_(0, torch.from_numpy(perm2.astype(np.int64)), yl)
    y_back = ep.exchange_rows(y_recv, recv_sz, snd)
    y = torch.zeros_like(x)
    for t in range(T):
        for j in range(K):
            y[t] += float(sc[t, j]) * y_back[pos[t * K + j]]
    ref = _moe_reference(x, blocks, gate)
    out[rank] = float((y - ref).abs().max())
    dist.destroy_process_group()


def test_ep_dispatch_combine_equals_single_process():
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _port(), out), nprocs=2, join=True)
    assert out[0] < 1e-5 and out[1] < 1e-5, dict(out)
