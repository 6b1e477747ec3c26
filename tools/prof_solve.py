"""Minimal driver for ncu: C2 solve(s) through the C ABI (no CPU work besides data gen)."""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2203_16340_b200 as lb
import synth

ap = argparse.ArgumentParser()
ap.add_argument("--solves", type=int, default=2)
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--config", default="C2")
a = ap.parse_args()
p = synth.CONFIGS[a.config]()
M = lb.colmajor(p.M)
b = torch.from_numpy(p.b).cuda()
obj = lb.LSQObjective(M, b=b)
s = lb.Solver(p.nvars, 5, lower=torch.zeros(p.nvars, dtype=torch.float64, device="cuda"),
              opts=lb.Options(use_graph=bool(a.graph)))
x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
for i in range(a.solves):
    x.zero_()
    r = s.solve(obj, x)
    print(i, r.iters, r.f, r.pg_inf, r.seconds)
