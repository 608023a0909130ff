"""Node-shared host expert store (memfd) across two processes on one GPU:
rank 0 creates and fills it, rank 1 maps the same pages, registers them and
copies a block H2D (the data-parallel replica path of bench.py)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE="2")
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    from paper_2602_03495_b200.engine.sharing import shared_host_store
    n = 64 << 20
    st = shared_host_store(n, rank, 2, 0, 4)
    if rank == 0:
        st.bytes[:] = torch.arange(n, dtype=torch.int64).remainder(251).to(torch.uint8)
    dist.barrier()
    if rank == 1:
        dev = st.bytes[(n // 2):(n // 2) + 4096].to("cuda", non_blocking=True)
        torch.cuda.synchronize()
        want = torch.arange(n // 2, n // 2 + 4096, dtype=torch.int64).remainder(251)
        out[1] = bool(torch.equal(dev.cpu().to(torch.int64), want))
    dist.barrier()
    dist.destroy_process_group()


def test_shared_store_two_processes():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(_port(), out), nprocs=2, join=True)
    assert out[1] is True
