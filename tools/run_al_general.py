"""General Alg. 4 (al_solve's general path) at C2 scale: NNLS 20000 x 10000 with
64 linear equalities (E 10000 x 64, the GEMV kernels) and, second, one
nonlinear inequality ||x||^2 <= R through torch callbacks.  Reports time,
outer / inner iterations, objective evaluations and the time per evaluation
(each evaluation = GEMV + GEMV^T over A, E^T x and E w, the callbacks)."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

p = synth.nnls_gaussian(20000, 10000, 2)
n = p.nvars
rng = np.random.default_rng(7)
E = rng.standard_normal((n, 64)) / np.sqrt(n)
x_feas = np.abs(rng.standard_normal(n)) * (rng.random(n) < 0.5)
e = E.T @ x_feas
obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda())
Ed = torch.from_numpy(E).cuda()
out = []
for case in ("64eq", "ball"):
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"), opts=lb.Options(max_iters=100000))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    kw = {}
    if case == "64eq":
        kw = dict(E=Ed, e=e)
    else:
        R = 0.25 * float(x_feas @ x_feas)

        def hg(x, h, g):
            g[0] = torch.dot(x, x) - R

        def jtv(x, ve, vi, o):
            o.copy_(2.0 * vi[0] * x)
        kw = dict(hg=hg, jtv=jtv, p_nl=1)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = s.al_solve(obj, x, **kw)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out.append(dict(case=case, seconds=dt, status=r.status, outer=r.outer_iters, inner=r.inner_iters_total,
                    f=r.f, violation=r.violation_inf, rho=r.rho, ms_per_inner=1e3 * dt / max(r.inner_iters_total, 1)))
    print(json.dumps(out[-1]), flush=True)
