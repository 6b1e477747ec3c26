"""Worker of tests/test_gpu_group.py: process `rank` of `world` hosts
nchunks/world logical ranks (fixed column chunks) of one P2P-sharded NNLS
solve (paper_2203_16340_b200.sharded.ShardedGroup; lbfgsb_solve_group).
Runs standalone (world = 1) or under torch.distributed.run (gloo bootstrap;
every process may sit on the same GPU).  Rank 0 writes the gathered x, f,
iterations and status to argv[1] (.npz).

argv: out m n seed kind(gauss|c5) nchunks use_graph scale max_backtracks tol"""
import os
import pickle
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(out, m, n, seed, kind, nchunks, use_graph, scale, max_bt, tol):
    import paper_2203_16340_b200 as lb
    import synth
    from paper_2203_16340_b200.sharded import ShardedGroup
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    opts = lb.Options(use_graph=bool(use_graph), max_backtracks=max_bt, tol=tol)
    grp = ShardedGroup(n, m, nchunks=nchunks, opts=opts, world=world, rank=rank,
                       make_lower=lambda l, c0, c1: torch.zeros(c1 - c0, dtype=torch.float64, device="cuda"))
    objs, xs, keep = [], [], []
    if kind == "gauss":
        prob = synth.nnls_gaussian(m, n, seed)
        b = torch.from_numpy(prob.b * scale).cuda()
    for l in grp.local:
        c0, c1 = grp.ranges[l]
        if kind == "gauss":
            M = lb.colmajor(prob.M[:, c0:c1] * scale)
        else:
            M, bh, _ = synth.c5_device(m, n, seed=seed, col0=c0, ncols=c1 - c0)
            b = torch.from_numpy(bh).cuda()
        objs.append(lb.LSQObjective(M, b=b))
        xs.append(torch.zeros(c1 - c0, dtype=torch.float64, device="cuda"))
        keep.append((M, b))
    r = grp.solve(objs, xs)
    mine = pickle.dumps({l: x.cpu().numpy() for l, x in zip(grp.local, xs)})
    if world > 1:
        from paper_2203_16340_b200.sharded import all_gather_bytes
        parts = {}
        for blob in all_gather_bytes(mine):
            parts.update(pickle.loads(blob))
    else:
        parts = pickle.loads(mine)
    if rank == 0:
        xg = np.concatenate([parts[l] for l in range(nchunks)])
        np.savez(out, x=xg, f=r.f, iters=r.iters, status=r.status, pg=r.pg_inf, n_bt=r.n_backtracks,
                 n_fb=r.n_fallbacks)
    if world > 1:
        dist.barrier()
    grp.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    a = sys.argv[1:]
    main(a[0], int(a[1]), int(a[2]), int(a[3]), a[4], int(a[5]), int(a[6]), float(a[7]), int(a[8]), float(a[9]))
