"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
every kernel family of the library on a shape that exercises its tails.
  python tools/sanitize_cases.py CASE     (CASE in CASES)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402


def _nnls(m, n, seed, graph=True, **kw):
    p = synth.nnls_gaussian(m, n, seed)
    obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda())
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"),
                  opts=lb.Options(use_graph=graph, **kw))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    print("nnls", m, n, r.status_name, r.iters, r.f)


def c1():
    _nnls(200, 100, 1)
    _nnls(200, 100, 1, graph=False)


def c2s():
    _nnls(3000, 1500, 2)                 # k_bwd_s, long-column k_fwd
    _nnls(30000, 300, 3)                 # generic k_bwd, tall k_fwd


def c4s():
    _nnls(500, 20000, 4)                 # k_bwd_w, short-column k_fwd


def lasso():
    p = synth.lasso_split(300, 700, 5)
    obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda(), c=torch.from_numpy(p.c).cuda(),
                          delta=p.delta, split=True)
    s = lb.Solver(p.nvars, 5, lower=torch.zeros(p.nvars, dtype=torch.float64, device="cuda"))
    x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
    print("lasso", s.solve(obj, x).status_name)


def c4split():
    p = synth.lasso_split(400, 20000, 64)          # split operator on k_bwd_wo (>= 64 columns per CTA)
    obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda(), c=torch.from_numpy(p.c).cuda(),
                          delta=p.delta, split=True)
    s = lb.Solver(p.nvars, 5, lower=torch.zeros(p.nvars, dtype=torch.float64, device="cuda"),
                  opts=lb.Options(max_iters=30))
    x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
    print("c4split", s.solve(obj, x).status_name)


def al():
    p = synth.svm_dual_linear(400, 20, 6)
    M = lb.colmajor(p.M)
    y = torch.from_numpy(p.colscale).cuda()
    obj = lb.LSQObjective(M, colscale=y, c=torch.from_numpy(p.c).cuda())
    s = lb.Solver(p.nvars, 5, lower=torch.zeros(p.nvars, dtype=torch.float64, device="cuda"),
                  upper=torch.from_numpy(p.upper).cuda())
    x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, E=y.reshape(-1, 1), e=np.zeros(1))
    print("al", r.status, r.outer_iters)


def algen():
    """general Alg. 4: 24 linear equalities (GEMV kernels on E) + a nonlinear ball through callbacks"""
    rng = np.random.default_rng(12)
    m, n = 300, 150
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    E = rng.standard_normal((n, 24)) / np.sqrt(n)
    e = E.T @ np.abs(rng.standard_normal(n))
    obj = lb.LSQObjective(lb.colmajor(A), b=torch.from_numpy(rng.standard_normal(m)).cuda())
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    R = 4.0 * float(np.abs(rng.standard_normal(n)) @ np.abs(rng.standard_normal(n)))

    def hg(x, h, g):
        g[0] = torch.dot(x, x) - R

    def jtv(x, ve, vi, out):
        out.copy_(2.0 * vi[0] * x)
    r = s.al_solve(obj, x, E=torch.from_numpy(E).cuda(), e=e, hg=hg, jtv=jtv, p_nl=1)
    print("algen", r.status, r.outer_iters)


def loop3():
    from paper_2203_16340_b200.sharded import column_range
    p = synth.nnls_gaussian(900, 600, 7)
    sv, ob, xs, keep = [], [], [], []
    for r in range(3):
        c0, c1_ = column_range(600, 3, r)
        M = lb.colmajor(p.M[:, c0:c1_])
        b = torch.from_numpy(p.b).cuda()
        sv.append(lb.Solver(c1_ - c0, 5, lower=torch.zeros(c1_ - c0, dtype=torch.float64, device="cuda")))
        ob.append(lb.LSQObjective(M, b=b))
        xs.append(torch.zeros(c1_ - c0, dtype=torch.float64, device="cuda"))
        keep.append((M, b))
    lb.p2p_connect_local(sv, 900)
    print("loop3", lb.solve_loopback(sv, ob, xs).status_name)


def group():
    from paper_2203_16340_b200.sharded import ShardedGroup
    p = synth.nnls_gaussian(1200, 800, 8)
    g = ShardedGroup(800, 1200, nchunks=8,
                     make_lower=lambda l, c0, c1: torch.zeros(c1 - c0, dtype=torch.float64, device="cuda"))
    b = torch.from_numpy(p.b).cuda()
    objs, xs, keep = [], [], []
    for l in g.local:
        c0, c1_ = g.ranges[l]
        M = lb.colmajor(p.M[:, c0:c1_])
        keep.append(M)
        objs.append(lb.LSQObjective(M, b=b))
        xs.append(torch.zeros(c1_ - c0, dtype=torch.float64, device="cuda"))
    print("group", g.solve(objs, xs).status_name)
    g.close()


def batch():
    probs = [synth.nnls_gaussian(60, 30, s) for s in range(5, 9)]
    A = np.stack([q.M for q in probs]); b = np.stack([q.b for q in probs])
    x = torch.zeros(4, 30, dtype=torch.float64, device="cuda")
    res = lb.solve_batched_lsq(lb.colmajor_batch(A), torch.from_numpy(b).cuda(), x,
                               lower=torch.zeros(4, 30, dtype=torch.float64, device="cuda"),
                               opts=lb.Options(max_backtracks=0))
    print("batch", [r.status_name for r in res])


def qp():
    X, y = synth.blobs(300, 5, 9)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    K = lb.op_gaussian_kernel(Xd, 1.0)
    obj = lb.QPObjective(K, colscale=torch.from_numpy(y).cuda(), c=-torch.ones(300, dtype=torch.float64,
                                                                              device="cuda"))
    s = lb.Solver(300, 5, lower=torch.zeros(300, dtype=torch.float64, device="cuda"),
                  upper=torch.ones(300, dtype=torch.float64, device="cuda"))
    x = torch.zeros(300, dtype=torch.float64, device="cuda")
    print("qp", s.solve(obj, x).status_name)


def transport():
    T = synth.transport_ds2(40, 10)
    for reg in ("gaussian", "entropy"):
        M = torch.from_numpy(np.asfortranarray(T.cost)).cuda().T.contiguous().T
        obj = lb.TransportObjective(M, reg=reg, lam=0.5)
        lo = torch.full((obj.nvars,), 0.0 if reg == "gaussian" else 1e-300, dtype=torch.float64, device="cuda")
        s = lb.Solver(obj.nvars, 5, lower=lo, opts=lb.Options(eps=1e-9 if reg == "gaussian" else 1e-20))
        x = torch.zeros(obj.nvars, dtype=torch.float64, device="cuda")
        r = s.al_solve_transport(obj, x, torch.from_numpy(T.u).cuda(), torch.from_numpy(T.v).cuda())
        print("transport", reg, r.status, r.outer_iters)


CASES = {f.__name__: f for f in (c1, c2s, c4s, lasso, al, algen, loop3, group, batch, qp, transport)}

if __name__ == "__main__":
    torch.cuda.init()
    for name in sys.argv[1:]:
        CASES[name]()
    torch.cuda.synchronize()
