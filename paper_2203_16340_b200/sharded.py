"""Host side of the column-sharded (N > 1) path: partitioning, NCCL bootstrap
through torch.distributed, and the multi-GPU bench step.

The device side lives in the library (lbfgsb_create_sharded, DESIGN.md
section 8): each rank owns a contiguous block of columns of M~ (and the
matching variables, bounds and ring slice); per iteration the ranks
all-gather the m-length partial of q = M~p and small packs (Alg. 2 sums,
separable Armijo sums, the Gram of Alg. 3) and reduce them in rank order, so
every rank takes bit-identical decisions.  torch.distributed is only the
bootstrap (broadcast of the 128-byte ncclUniqueId, or the all-gather of the
64-byte CUDA IPC handles of the P2P mailboxes) and the bench's barrier /
max-over-ranks timing; the per-iteration exchange is the library's own NCCL
communicator (xchg="nccl") or its own kernels' stores into the peers'
mailboxes over NVLink (xchg="p2p", lbfgsb_create_sharded_p2p).
"""
from __future__ import annotations

import json
import os
import time


def column_range(ncols: int, nranks: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced block [c0, c1) of rank `rank` (block sizes differ by <= 1)."""
    if not (0 <= rank < nranks):
        raise ValueError("rank out of range")
    return rank * ncols // nranks, (rank + 1) * ncols // nranks


def broadcast_bytes(payload: bytes | None, src: int = 0) -> bytes:
    """Broadcast a small byte string (the ncclUniqueId) from `src` over the
    default torch.distributed group (works for gloo and nccl)."""
    import torch.distributed as dist
    obj = [payload if dist.get_rank() == src else None]
    dist.broadcast_object_list(obj, src=src)
    return obj[0]


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank float over the default group (the bench's timing rule)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def all_gather_bytes(payload: bytes) -> list[bytes]:
    """All-gather one small byte string per rank (rank order) over the default group."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size()
    dist.all_gather_object(out, payload)
    return out


def make_sharded_solver(n_local, n_global, m_hist, lower, opts, stream, xchg="nccl", m_max=None):
    """Sharded handle on the current rank.  xchg="nccl": lbfgsb_create_sharded
    (rank 0 makes the NCCL id).  xchg="p2p": lbfgsb_create_sharded_p2p with a
    mailbox for residuals of length <= m_max, IPC handles all-gathered and
    opened, then a barrier so that no rank signals an unmapped peer."""
    import torch.distributed as dist
    import paper_2203_16340_b200 as lb
    rank, world = dist.get_rank(), dist.get_world_size()
    if xchg == "p2p":
        if m_max is None:
            raise ValueError("xchg='p2p' needs m_max")
        s = lb.Solver(n_local, m_hist, lower=lower, opts=opts, stream=stream, rank=rank, nranks=world,
                      n_global=n_global, p2p_m_max=int(m_max))
        s.p2p_open(all_gather_bytes(s.ipc_handle()))
        dist.barrier()
        return s
    if xchg != "nccl":
        raise ValueError(f"unknown exchange {xchg!r}")
    nid = lb.nccl_unique_id() if rank == 0 else None
    nid = broadcast_bytes(nid, src=0)
    return lb.Solver(n_local, m_hist, lower=lower, opts=opts, stream=stream, nccl_id=nid,
                     rank=rank, nranks=world, n_global=n_global)
