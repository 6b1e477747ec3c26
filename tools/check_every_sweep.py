"""C2 solve time vs the host check interval (iterations per graph replay)."""
import os
import sys
import json
sys.path.insert(0, os.getcwd())
import torch  # noqa: E402
import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

p = synth.nnls_gaussian(20000, 10000, 2)
M = lb.colmajor(p.M)
b = torch.from_numpy(p.b).cuda()
lo = torch.zeros(10000, dtype=torch.float64, device="cuda")
obj = lb.LSQObjective(M, b=b)
for ce in (4, 8, 12, 16, 24, 32):
    s = lb.Solver(10000, 5, lower=lo, opts=lb.Options(check_every=ce))
    x = torch.zeros(10000, dtype=torch.float64, device="cuda")
    for _ in range(3):
        x.zero_(); s.solve(obj, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        x.zero_(); r = s.solve(obj, x)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"check_every": ce, "ms_per_solve": e0.elapsed_time(e1) / 20, "iters": r.iters}), flush=True)
