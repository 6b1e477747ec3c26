"""Worker of tests/test_gpu_p2p.py::test_p2p_two_processes: one rank of a
column-sharded NNLS solve whose exchange runs over CUDA-IPC-mapped peer
memory (lbfgsb_create_sharded_p2p).  Launched with torch.distributed.run
(gloo bootstrap); every rank may sit on the same GPU (the test box has one).
Writes rank 0's gathered x, f, iterations to argv[1] (.npz)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402


def main(out, m, n, seed, use_graph):
    import paper_2203_16340_b200 as lb
    import synth
    from paper_2203_16340_b200.sharded import all_gather_bytes, column_range, make_sharded_solver
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    ngpu = torch.cuda.device_count()
    torch.cuda.set_device(rank % ngpu)
    prob = synth.nnls_gaussian(m, n, seed)
    c0, c1 = column_range(prob.ncols, world, rank)
    M = lb.colmajor(prob.M[:, c0:c1])
    b = torch.from_numpy(prob.b).cuda()
    lo = torch.zeros(c1 - c0, dtype=torch.float64, device="cuda")
    s = make_sharded_solver(c1 - c0, prob.nvars, 5, lo, lb.Options(use_graph=bool(use_graph)), None,
                            xchg="p2p", m_max=m)
    obj = lb.LSQObjective(M, b=b)
    x = torch.zeros(c1 - c0, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    xs = all_gather_bytes(x.cpu().numpy().tobytes())
    if rank == 0:
        xg = np.concatenate([np.frombuffer(v, dtype=np.float64) for v in xs])
        np.savez(out, x=xg, f=r.f, iters=r.iters, status=r.status, pg=r.pg_inf)
    dist.barrier()
    s.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]))
