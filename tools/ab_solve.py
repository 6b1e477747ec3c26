"""Whole-solve device time (CUDA events around solve(), no per-kernel event
nodes, so PDL edges stay intact) on a named shape, for A/B runs against
variant builds (tools/_prof_with_lib.py):
  python tools/ab_solve.py c2|c4|c1 [reps]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

shape = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
if shape == "c2":
    m, n = 20000, 10000
    p = synth.nnls_gaussian(m, n, 2)
    A, b = lb.colmajor(p.M), torch.from_numpy(p.b).cuda()
elif shape == "c1":
    m, n = 200, 100
    p = synth.nnls_gaussian(m, n, 1)
    A, b = lb.colmajor(p.M), torch.from_numpy(p.b).cuda()
else:
    m, n = 1000, 100000
    rng = np.random.default_rng(4)
    A = lb.colmajor(rng.standard_normal((m, n)) / np.sqrt(m))
    b = torch.from_numpy(rng.standard_normal(m)).cuda()
obj = lb.LSQObjective(A, b=b)
s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"), opts=lb.Options())
x = torch.zeros(n, dtype=torch.float64, device="cuda")
s.solve(obj, x)
st = torch.cuda.current_stream()
out = []
for _ in range(reps):
    x.zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    r = s.solve(obj, x)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out.append({"ms": ms, "iters": r.iters, "iters_per_s": r.iters / ms * 1e3, "f": r.f, "x_sum": float(x.sum())})
med = sorted(o["iters_per_s"] for o in out)[len(out) // 2]
print(json.dumps({"lib": os.environ.get("LB_LIB", "default"), "shape": shape, "iters_per_s_median": med,
                  "runs": out}))
