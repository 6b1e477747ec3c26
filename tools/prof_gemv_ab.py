"""Per-launch k_bwd / k_fwd times inside a solve (CUDA events, profile=True) on
a named shape, for A/B runs against variant builds (tools/_prof_with_lib.py).
  python tools/prof_gemv_ab.py c5chunk|c2|c4 [reps]"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

shape = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if shape == "c5chunk":
    m, n = 100000, 25000
    A, b, _ = synth.c5_device(m, n, seed=5)
    b = torch.from_numpy(b).cuda()
elif shape == "c2":
    m, n = 20000, 10000
    p = synth.nnls_gaussian(m, n, 2)
    A, b = lb.colmajor(p.M), torch.from_numpy(p.b).cuda()
else:
    m, n = 1000, 100000
    rng = np.random.default_rng(4)
    A = lb.colmajor(rng.standard_normal((m, n)) / np.sqrt(m))
    b = torch.from_numpy(rng.standard_normal(m)).cuda()
obj = lb.LSQObjective(A, b=b)
s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"), opts=lb.Options(profile=True))
x = torch.zeros(n, dtype=torch.float64, device="cuda")
s.solve(obj, x)
out = []
for _ in range(reps):
    s.profile(reset=True)
    x.zero_()
    r = s.solve(obj, x)
    pr = s.profile(reset=True)
    bw, fw = pr["gemvT_epi (k_bwd)"], pr["gemv_active (k_fwd)"]
    nact = pr["fwd_active_columns"][1] / max(fw[1], 1)
    out.append({"bwd_us": 1e3 * bw[0] / bw[1], "bwd_gbs": (8 * m * n + 8 * m + 72 * n) / (bw[0] / bw[1] / 1e3) / 1e9,
                "fwd_us": 1e3 * fw[0] / fw[1], "fwd_gbs": (8 * m * nact) / (fw[0] / fw[1] / 1e3) / 1e9,
                "iters": r.iters, "f": r.f, "x_sum": float(x.sum())})
print(json.dumps({"lib": os.environ.get("LB_LIB", "default"), "shape": shape, "runs": out}))
