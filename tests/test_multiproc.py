"""Multi-process host logic on CPU (gloo, world_size 2): replica aggregation
(max-over-ranks time, summed tokens) used by bench.py for N > 1, and the
replica-independence of policy decisions (each rank replays its own stream
through the oracle with no cross-rank state)."""

import os
import socket

import numpy as np
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    from oracle import driver as D
    from oracle import policy as P
    t = bench.max_over_ranks(10.0 + rank, ws)
    n = bench.sum_over_ranks(100.0 * (rank + 1), ws)
    # each replica runs its own request stream (different seed) through the policies
    tr = P.synth_trace(4, 8, 2, 64, 1, 12, locality=0.9, drift_scale=0.4, noise_scale=0.08,
                       seed=rank)
    res = P.calibrate([s.hidden for s in tr.steps])
    cfg = D.DriverConfig(tables=P.default_tables(non_moe_layer_time=3.0), prefetch_size=1,
                         residuals=res, cache_capacity=2, w_size=4, u_size=1, seed=3)
    rep, _ = D.run([D.StepInput(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                    for s in tr.steps], tr.gates, cfg, 4, 8, 2)
    obj = [None] * ws
    dist.all_gather_object(obj, rep["cache_hit_rate"])
    out[rank] = (t, n, obj)
    dist.destroy_process_group()


def test_replica_aggregation_gloo_ws2():
    ws = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
    assert out[0][0] == out[1][0] == 11.0          # time = max over ranks
    assert out[0][1] == out[1][1] == 300.0         # tokens = sum over ranks
    assert out[0][2] == out[1][2]                  # every rank sees the same gathered rates
    # replicas are independent: rank r's hit rate equals a single-process run of seed r
    from oracle import driver as D
    from oracle import policy as P
    for r in range(ws):
        tr = P.synth_trace(4, 8, 2, 64, 1, 12, locality=0.9, drift_scale=0.4,
                           noise_scale=0.08, seed=r)
        res = P.calibrate([s.hidden for s in tr.steps])
        cfg = D.DriverConfig(tables=P.default_tables(non_moe_layer_time=3.0), prefetch_size=1,
                             residuals=res, cache_capacity=2, w_size=4, u_size=1, seed=3)
        rep, _ = D.run([D.StepInput(s.token_index, s.tokens, s.workloads, s.hidden, s.eos)
                        for s in tr.steps], tr.gates, cfg, 4, 8, 2)
        assert out[0][2][r] == rep["cache_hit_rate"]
