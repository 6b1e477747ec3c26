"""Kernel time breakdown of an N2 run measured in situ (torch.profiler / CUPTI),
to compare with the serialized ncu launch list."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb, synth
from torch.profiler import profile, ProfilerActivity
n = int(os.environ.get("N", "1000")); reg = os.environ.get("REG", "entropy")
t = synth.transport_ds2(n, 1); m = t.m
Md = torch.from_numpy(t.cost.reshape(-1, order="F")).cuda().reshape(n, m).T
obj = lb.TransportObjective(Md, reg, t.lam)
lo = torch.full((m * n,), 1e-300 if reg == "entropy" else 0.0, dtype=torch.float64, device="cuda")
s = lb.Solver(m * n, 5, lower=lo, opts=lb.Options(tol=1e-6, max_iters=100000, eps=1e-20))
x = torch.zeros(m * n, dtype=torch.float64, device="cuda")
u = torch.from_numpy(t.u).cuda(); v = torch.from_numpy(t.v).cuda()
s.al_solve_transport(obj, x, u, v, al_opts=lb.ALOptions(feas_tol=1e-6, max_outer=2))
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    t0 = time.perf_counter()
    r = s.al_solve_transport(obj, x, u, v, al_opts=lb.ALOptions(feas_tol=1e-6, max_outer=12))
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
print(r, dt, dt / max(r.inner_iters_total, 1) * 1e6, "us/inner")
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=15))
