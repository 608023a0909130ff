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

import numpy as np
import torch
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
