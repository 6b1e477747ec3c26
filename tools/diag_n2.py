"""N2 entropy diagnostics (DS2): solve with al_solve_transport at
the given n / tol, then compare with the Sinkhorn scaling (plain torch) and
report the entries that end at the R30 lower bound 1e-300: their count, the
Sinkhorn value there, and the gradient / multiplier sums.
  python tools/diag_n2.py [n] [tol]"""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
tol = float(sys.argv[2]) if len(sys.argv) > 2 else 2e-6
t = synth.transport_ds2(n, 9)
m = t.m
Md = torch.from_numpy(t.cost.reshape(-1, order="F")).cuda().reshape(n, m).T
obj = lb.TransportObjective(Md, "entropy", t.lam)
lo = torch.full((m * n,), 1e-300, dtype=torch.float64, device="cuda")
s = lb.Solver(m * n, 5, lower=lo, opts=lb.Options(tol=tol, max_iters=200000, eps=1e-20))
x = torch.zeros(m * n, dtype=torch.float64, device="cuda")
lam = torch.zeros(m + n, dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
r = s.al_solve_transport(obj, x, torch.from_numpy(t.u).cuda(), torch.from_numpy(t.v).cuda(), lam_out=lam,
                         al_opts=lb.ALOptions(feas_tol=tol, max_outer=60))
dt = time.perf_counter() - t0
X = x.cpu().numpy().reshape(m, n, order="F")
L = lam.cpu().numpy()
G = t.cost + t.lam * (np.log(X) + 1) + L[:m, None] + L[None, m:]
K = torch.exp(-torch.from_numpy(t.cost).cuda() / t.lam)
u, v = torch.from_numpy(t.u).cuda(), torch.from_numpy(t.v).cuda()
a, b = torch.ones_like(u), torch.ones_like(v)
for _ in range(20000):
    a = u / (K @ b)
    b = v / (K.T @ a)
Ps = (a[:, None] * K * b[None, :]).cpu().numpy()
at = X <= 1e-290
out = {"n": n, "tol": tol, "status": r.status, "outer": r.outer_iters, "inner": r.inner_iters_total, "s": dt,
       "f": r.f, "rho": r.rho, "viol": r.violation_inf, "at_lb": int(at.sum()),
       "max_abs_G_free": float(np.abs(G[~at]).max()),
       "min_G_at_lb": float(G[at].min()) if at.any() else None,
       "max_sinkhorn_at_lb": float(Ps[at].max()) if at.any() else None,
       "max_abs_err": float(np.abs(X - Ps).max()), "max_P": float(Ps.max()),
       "max_rel_err_rows": float(np.max(np.abs(X.sum(1) - t.u))),
       "min_P_free": float(X[~at].min()), "min_sinkhorn": float(Ps.min())}
print(json.dumps(out))
