"""Per-kernel times of a plain (no AL) LSQ solve of a SURVEY config, for A/B
runs of the GEMV kernels: python tools/prof_bwdw.py [C4|C1|...] [max_iters]"""
import os
import sys
import json
sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 200
p = synth.CONFIGS[name]()
cu = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
obj = lb.LSQObjective(lb.colmajor(p.M), b=cu(p.b), c=cu(p.c), delta=p.delta, colscale=cu(p.colscale),
                      split=p.split)
s = lb.Solver(p.nvars, 5, lower=cu(p.lower), upper=cu(p.upper),
              opts=lb.Options(max_iters=iters, profile=True))
x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
x.zero_(); s.solve(obj, x)
s.profile(reset=True)
x.zero_()
t0 = torch.cuda.Event(enable_timing=True); t1 = torch.cuda.Event(enable_timing=True)
t0.record(); r = s.solve(obj, x); t1.record(); torch.cuda.synchronize()
pr = s.profile(reset=True)
bms, bn = pr["gemvT_epi (k_bwd)"]; fms, fn = pr["gemv_active (k_fwd)"]
nact = pr.get("fwd_active_columns", (0, 0))[1] / max(fn, 1)
print(json.dumps({"lib": lb._build.LIB, "config": name, "iters": r.iters, "f": r.f, "ms": t0.elapsed_time(t1),
                  "bwd_us": 1e3 * bms / max(bn, 1), "fwd_us": 1e3 * fms / max(fn, 1),
                  "bwd_gbs": 8 * p.M.shape[0] * p.M.shape[1] / (bms / max(bn, 1) / 1e3) / 1e9,
                  "fwd_active_cols": nact,
                  "fwd_gbs": 8 * p.M.shape[0] * nact / (fms / max(fn, 1) / 1e3) / 1e9 if fn else None}))
