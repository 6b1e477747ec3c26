"""N3 full: the original L-BFGS-B (Cauchy point on one thread) vs the modified
method on the paper's NNLS data set (ii) at n = 6000..12000
variables (A: 2n x n), tol 1e-6, plus the oracle's original L-BFGS-B on the
host (one core) -- the rows of the paper's appendix table."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth, oracle
with_oracle = "--oracle" in sys.argv
for n in [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [6000, 8000, 10000, 12000]:
    p = synth.nnls_ds2(n / 3000.0, 12)
    obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda())
    s = lb.Solver(p.nvars, 5, lower=torch.zeros(p.nvars, dtype=torch.float64, device="cuda"),
                  opts=lb.Options(tol=1e-6, max_iters=5000))
    x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
    s.solve(obj, x)                                                         # warm-up
    x.zero_(); torch.cuda.synchronize(); t0 = time.perf_counter()
    rm = s.solve(obj, x); torch.cuda.synchronize(); tm = time.perf_counter() - t0
    x.zero_(); torch.cuda.synchronize(); t0 = time.perf_counter()
    ro, cp_ms = s.solve_original(obj, x); torch.cuda.synchronize(); to = time.perf_counter() - t0
    row = dict(n=p.nvars, m=p.m, modified_gpu_s=tm, modified_iters=rm.iters, original_gpu_s=to,
               original_gpu_cp_s=cp_ms / 1e3, original_iters=ro.iters, f_mod=rm.f, f_orig=ro.f)
    if with_oracle:
        t0 = time.perf_counter()
        rc, tcp = oracle.minimize_lsq_original(oracle.LSQ(p.M, b=p.b), l=p.lower,
                                               opts=oracle.Options(tol=1e-6, max_iters=5000))
        row.update(original_cpu_s=time.perf_counter() - t0, original_cpu_cp_s=tcp, original_cpu_iters=rc.iters)
    print(json.dumps(row), flush=True)
