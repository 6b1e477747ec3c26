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


# --------------------------------------------------------------------------- P-invariant groups
def local_chunks(nchunks: int, world: int, rank: int) -> list[int]:
    """Logical ranks (fixed column chunks) hosted by process `rank` of `world`:
    a contiguous block of nchunks // world (world must divide nchunks)."""
    if nchunks % world:
        raise ValueError(f"{world} processes cannot host {nchunks} chunks evenly")
    k = nchunks // world
    return list(range(rank * k, (rank + 1) * k))


def merge_chunk_handles(parts: list, nchunks: int, complete: bool = True) -> list:
    """Merge the {logical rank: IPC handle} dicts of all processes into the C
    handles in logical-rank order; a chunk hosted twice (or, with `complete`,
    a chunk hosted nowhere) is an error."""
    allh = {}
    for part in parts:
        dup = set(part) & set(allh)
        if dup:
            raise ValueError(f"chunks {sorted(dup)} hosted twice")
        allh.update(part)
    if complete and sorted(allh) != list(range(nchunks)):
        raise ValueError(f"chunks not covered: {sorted(set(range(nchunks)) - set(allh))}")
    return [allh.get(l, bytes(64)) for l in range(nchunks)]


def gather_chunk_handles(mine: dict, nchunks: int, world: int) -> list:
    """Every process contributes {logical rank: 64-byte IPC handle} for the chunks
    it hosts; returns the C handles in logical-rank order (all-gathered over the
    default torch.distributed group when world > 1)."""
    import pickle
    if world == 1:
        return merge_chunk_handles([mine], nchunks, complete=False)
    return merge_chunk_handles([pickle.loads(b) for b in all_gather_bytes(pickle.dumps(mine))], nchunks)


class ShardedGroup:
    """SURVEY 8(e) bitwise P-invariance: the global problem is cut into
    ``nchunks`` (C) fixed column chunks -- logical ranks, each a P2P-sharded
    library handle -- independent of the number of processes; this process
    hosts C / world of them (``local_chunks``).  The C mailboxes are wired
    with lbfgsb_p2p_open_group (IPC handles all-gathered over
    torch.distributed when world > 1) and one solve (lbfgsb_solve_group)
    runs all local logical ranks on one stream.  x, f and the iteration count
    do not depend on ``world``.

    ``ranges[l]`` is the global column range [c0, c1) of logical rank l;
    ``make_lower(l, c0, c1)`` returns its lower-bound tensor (or None)."""

    def __init__(self, ncols: int, m_max: int, m_hist=5, nchunks=8, opts=None, stream=None,
                 make_lower=None, make_upper=None, world=1, rank=0):
        import paper_2203_16340_b200 as lb
        self.ncols, self.nchunks, self.world, self.rank = ncols, nchunks, world, rank
        self.ranges = [column_range(ncols, nchunks, l) for l in range(nchunks)]
        self.local = local_chunks(nchunks, world, rank)
        self.solvers = []
        for l in self.local:
            c0, c1 = self.ranges[l]
            lo = make_lower(l, c0, c1) if make_lower else None
            up = make_upper(l, c0, c1) if make_upper else None
            self.solvers.append(lb.Solver(c1 - c0, m_hist, lower=lo, upper=up, opts=opts, stream=stream,
                                          rank=l, nranks=nchunks, n_global=ncols, p2p_m_max=int(m_max)))
        mine = {l: s.ipc_handle() for l, s in zip(self.local, self.solvers)}
        handles = gather_chunk_handles(mine, nchunks, world)
        lb.p2p_open_group(self.solvers, handles)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()                 # every mailbox mapped before anyone signals

    def solve(self, objs, xs, tol=0.0):
        import paper_2203_16340_b200 as lb
        return lb.solve_group(self.solvers, objs, xs, tol)

    def close(self):
        for s in reversed(self.solvers):   # hs[0] owns the IPC mappings: close it last
            s.close()
        self.solvers = []
