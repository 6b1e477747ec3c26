"""N2 side-line: joint probability / regularised OT
on the paper's synthetic data sets; prints one JSON line per (data set, reg, n)."""
import os, sys, json, time, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--cases", default="ds2:entropy:1000")
ap.add_argument("--tol", type=float, default=1e-6)
ap.add_argument("--max-outer", type=int, default=100)
ap.add_argument("--max-iters", type=int, default=100000)
ap.add_argument("--eps", type=float, default=None,
                help="epsilon of Eq. (1) (default: 1e-20 for the entropy, 1e-9 for the Gaussian; reading R30)")
a = ap.parse_args()
for case in a.cases.split(","):
    ds, reg, n = case.split(":"); n = int(n)
    t = synth.transport_ds1(n) if ds == "ds1" else synth.transport_ds2(n, 1)
    m = t.m
    Md = torch.from_numpy(t.cost.reshape(-1, order="F")).cuda().reshape(n, m).T
    obj = lb.TransportObjective(Md, reg, t.lam)
    lo = torch.full((m * n,), 1e-300 if reg == "entropy" else 0.0, dtype=torch.float64, device="cuda")
    s = lb.Solver(m * n, 5, lower=lo, opts=lb.Options(tol=a.tol, max_iters=a.max_iters,
                                                      eps=a.eps if a.eps is not None else (1e-20 if reg == "entropy" else 1e-9)))
    x = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    u = torch.from_numpy(t.u).cuda(); v = torch.from_numpy(t.v).cuda()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = s.al_solve_transport(obj, x, u, v, al_opts=lb.ALOptions(feas_tol=a.tol, max_outer=a.max_outer))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(json.dumps(dict(case=case, m=m, n=n, nvars=m * n, tol=a.tol, solve_s=dt, status=r.status, f=r.f,
                          violation=r.violation_inf, outer=r.outer_iters, inner=r.inner_iters_total,
                          us_per_inner=1e6 * dt / max(r.inner_iters_total, 1))), flush=True)
