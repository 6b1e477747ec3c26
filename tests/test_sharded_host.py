"""CPU (-m "not gpu") multi-process tests of the N > 1 host path with the
gloo backend, world_size 2: column partitioning, the ncclUniqueId broadcast,
max-over-ranks timing, and the decomposition the sharded library uses
(rank-local partials of q = M~p, of the Alg. 2 sums and of the Gram pack,
all-gathered and reduced in rank order) checked against the unsharded
quantities computed by the oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2203_16340_b200.sharded import column_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("ncols,P", [(10, 2), (10000, 8), (7, 3), (1, 1), (200000, 8), (5, 5)])
def test_column_range_partition(ncols, P):
    rs = [column_range(ncols, P, r) for r in range(P)]
    assert rs[0][0] == 0 and rs[-1][1] == ncols
    for (a0, a1), (b0, b1) in zip(rs, rs[1:]):
        assert a1 == b0
    sizes = [b - a for a, b in rs]
    assert max(sizes) - min(sizes) <= 1


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_16340_b200 import sharded
    import oracle

    # 1) the unique-id broadcast used by make_sharded_solver
    nid = bytes(range(128)) if rank == 0 else None
    got = sharded.broadcast_bytes(nid, src=0)
    # 2) max-over-ranks timing
    mx = sharded.max_over_ranks(1.5 + rank)
    # 2b) the IPC-handle all-gather of the P2P exchange (64 bytes per rank, rank order)
    hs = sharded.all_gather_bytes(bytes([rank]) * 64)
    # 3) the sharded decomposition on a small NNLS instance
    m, n = 60, 37
    rng = np.random.default_rng(0)
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    x = np.abs(rng.standard_normal(n)) * (rng.random(n) < 0.6)
    g = rng.standard_normal(n)
    d = -g * (rng.random(n) < 0.7)
    l = np.zeros(n)
    c0, c1 = sharded.column_range(n, world, rank)
    # rank-local q partial and Alg. 2 sums (projected candidate)
    q_loc = oracle.matvec(A[:, c0:c1], d[c0:c1])
    pp = np.maximum(x[c0:c1] + d[c0:c1], 0.0) - x[c0:c1]
    dir_loc = np.array([pp @ g[c0:c1], pp @ pp])
    q_all = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(q_all, torch.from_numpy(q_loc))
    dir_all = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(dir_all, torch.from_numpy(dir_loc))
    q = np.zeros(m)
    for t in q_all:                      # rank order
        q = q + t.numpy()
    sums = np.zeros(2)
    for t in dir_all:
        sums = sums + t.numpy()
    q_ref = oracle.matvec(A, d)
    pp_ref = np.maximum(x + d, 0.0) - x
    res = dict(got=got, mx=mx, hs=hs, q_err=float(np.max(np.abs(q - q_ref) / (np.abs(A) @ np.abs(d) + 1e-300))),
               s_err=float(abs(sums[0] - pp_ref @ g) + abs(sums[1] - pp_ref @ pp_ref)),
               q_bits=q.tobytes())
    out[rank] = res
    dist.destroy_process_group()


def test_gloo_world2_sharded_host_logic():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        assert out[r]["got"] == bytes(range(128))
        assert out[r]["mx"] == 2.5
        assert out[r]["hs"] == [bytes([k]) * 64 for k in range(world)]
        assert out[r]["q_err"] <= 1e-12
        assert out[r]["s_err"] <= 1e-12
    # every rank reduced the same gathered partials in the same order: identical bits
    assert out[0]["q_bits"] == out[1]["q_bits"]


def test_make_sharded_solver_argument_checks():
    from paper_2203_16340_b200 import sharded
    import torch.distributed as dist
    if dist.is_initialized():
        pytest.skip("default group already initialised")
    port = _free_port()
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    try:
        with pytest.raises(ValueError):
            sharded.make_sharded_solver(10, 10, 5, None, None, None, xchg="p2p")          # no m_max
        with pytest.raises(ValueError):
            sharded.make_sharded_solver(10, 10, 5, None, None, None, xchg="mpi")
    finally:
        dist.destroy_process_group()


def test_local_chunks_partition():
    """P-invariant grouping: C = 8 fixed chunks, world in {1, 2, 4, 8}
    processes each host a contiguous block of 8 / world logical ranks; together
    they cover every chunk exactly once; a world that does not divide C is refused."""
    from paper_2203_16340_b200.sharded import column_range, local_chunks
    for world in (1, 2, 4, 8):
        got = [l for r in range(world) for l in local_chunks(8, world, r)]
        assert got == list(range(8))
    with pytest.raises(ValueError):
        local_chunks(8, 3, 0)
    # the chunk ranges do not depend on the process count
    rng = [column_range(200000, 8, l) for l in range(8)]
    assert rng[0] == (0, 25000) and rng[-1] == (175000, 200000)


def _group_worker(rank, world, port, out):
    import pickle
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2203_16340_b200 import sharded
    import oracle
    C = 8
    mine = sharded.local_chunks(C, world, rank)
    # 1) the IPC-handle exchange of ShardedGroup: every process gets all C handles in chunk order
    hs = sharded.gather_chunk_handles({l: bytes([l]) * 64 for l in mine}, C, world)
    # 2) the chunk-ordered reduction that makes the solve P-invariant (R36): q = sum over the C fixed
    #    chunks, in chunk order, of the chunk's partial A_l p_l
    m, n = 50, 83
    rng = np.random.default_rng(1)
    A = rng.standard_normal((m, n))
    p = rng.standard_normal(n)
    parts = {}
    for l in mine:
        c0, c1 = sharded.column_range(n, C, l)
        parts[l] = oracle.matvec(A[:, c0:c1], p[c0:c1])
    allp = {}
    for blob in sharded.all_gather_bytes(pickle.dumps(parts)):
        allp.update(pickle.loads(blob))
    q = np.zeros(m)
    for l in range(C):
        q = q + allp[l]
    out[rank] = dict(hs=hs, q_bits=q.tobytes())
    dist.destroy_process_group()


def test_gloo_world2_group_host_logic():
    """world_size 2 (gloo): the P-invariant group's handle exchange and its
    chunk-ordered reduction give every process the same handles and the same
    bits, equal to the single-process (world 1) result."""
    from paper_2203_16340_b200 import sharded
    import oracle
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_group_worker, args=(world, port, out), nprocs=world, join=True)
    ref_h = [bytes([l]) * 64 for l in range(8)]
    assert out[0]["hs"] == ref_h and out[1]["hs"] == ref_h
    # world 1: the same chunks, the same order
    m, n = 50, 83
    rng = np.random.default_rng(1)
    A = rng.standard_normal((m, n))
    p = rng.standard_normal(n)
    q = np.zeros(m)
    for l in range(8):
        c0, c1 = sharded.column_range(n, 8, l)
        q = q + oracle.matvec(A[:, c0:c1], p[c0:c1])
    assert out[0]["q_bits"] == out[1]["q_bits"] == q.tobytes()
    # a chunk hosted twice, or a chunk hosted nowhere, is refused
    with pytest.raises(ValueError):
        sharded.merge_chunk_handles([{3: bytes(64)}, {3: bytes(64)}], 8)
    with pytest.raises(ValueError):
        sharded.merge_chunk_handles([{l: bytes(64) for l in range(7)}], 8)
