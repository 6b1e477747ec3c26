"""Correctness of a k_bwd_wt build on short-column shapes against the oracle
(run through tools/_prof_with_lib.py with the variant library)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as orc  # noqa: E402
import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

out = []
for (m, n, seed, split) in [(1000, 5000, 3, False), (600, 3000, 4, True), (1000, 2400, 5, False), (1998, 4001, 6, False)]:
    p = synth.lasso_split(m, n, seed) if split else synth.nnls_gaussian(m, n, seed)
    cu = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    obj = lb.LSQObjective(lb.colmajor(p.M), b=cu(p.b), c=cu(p.c), delta=p.delta, split=p.split)
    s = lb.Solver(p.nvars, 5, lower=cu(p.lower))
    x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    P = orc.LSQ(p.M, b=p.b, c=p.c, delta=p.delta, split=p.split)
    ro = orc.minimize_lsq(P, l=p.lower)
    out.append(dict(m=m, n=n, split=split, status=r.status, ostatus=ro.status, f=r.f, fo=ro.f,
                    rel=abs(r.f - ro.f) / abs(ro.f), pg=r.pg_inf, iters=r.iters, oiters=ro.iters))
print(json.dumps({"lib": os.environ.get("LB_LIB", "default"), "cases": out}))
