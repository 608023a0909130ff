"""Node-local sharing of the host expert store between data-parallel ranks.

Local rank 0 creates the memfd-backed store (``dali_host_alloc_shared``) and
hands its descriptor to the other local ranks over a Unix-domain socket
(SCM_RIGHTS) -- unlike opening /proc/<pid>/fd this works under Yama ptrace
restrictions between sibling processes.  Each rank registers the mapping
with CUDA itself.  One store per node instead of one per GPU: Mixtral-8x7B
needs 90 GB of host memory once, not 8 times.
"""

from __future__ import annotations

import os
import socket

import torch.distributed as dist

from .weights import HostStore


def shared_host_store(nbytes: int, local_rank: int, local_world: int, leader_rank: int,
                      threads: int) -> HostStore:
    info = [None]
    srv = None
    store = None
    if local_rank == 0:
        store = HostStore(nbytes, threads, shared="create")
        path = f"/tmp/dali_store_{os.getpid()}.sock"
        if os.path.exists(path):
            os.unlink(path)
        srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        srv.bind(path)
        srv.listen(max(local_world, 1))
        info = [path]
    dist.broadcast_object_list(info, src=leader_rank)
    if local_rank == 0:
        for _ in range(local_world - 1):
            conn, _ = srv.accept()
            socket.send_fds(conn, [b"d"], [store.fd])
            conn.close()
        srv.close()
        os.unlink(info[0])
    else:
        c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        c.connect(info[0])
        _, fds, _, _ = socket.recv_fds(c, 1, 1)
        c.close()
        store = HostStore(nbytes, 1, shared="open", fd=fds[0], owner_pid=-1)
    return store
