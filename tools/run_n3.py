"""N3 side-line: the original L-BFGS-B's generalized
Cauchy point on B200, its breakpoint loop on one thread (lbfgsb_op_cauchy_point),
against one full iteration of the modified method at the same n.  Inputs: box
[0, 1], x ~ U(0.05, 0.95) (every variable has a finite breakpoint), g ~ N(0, 1),
h = 5 random curvature pairs with s^T y > 0, theta = y^T y / s^T y."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
for n in [int(a) for a in sys.argv[1:]] or [6000, 8000, 10000, 12000, 100000, 1000000]:
    rng = np.random.default_rng(n)
    h = 5
    x = rng.uniform(0.05, 0.95, n); g = rng.standard_normal(n)
    S = rng.standard_normal((h, n)) / np.sqrt(n); Y = S + 0.3 * rng.standard_normal((h, n)) / np.sqrt(n)
    theta = float(Y[-1] @ Y[-1] / (S[-1] @ Y[-1]))
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"),
                  upper=torch.ones(n, dtype=torch.float64, device="cuda"))
    out = []
    for theta_k in [theta, theta * 1e-3]:          # a flatter model passes more breakpoints
        s.op_cauchy_point(cu(x), cu(g), cu(S), cu(Y), theta_k)          # warm-up
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = s.op_cauchy_point(cu(x), cu(g), cu(S), cu(Y), theta_k)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        out.append(dict(theta=theta_k, passed=r["passed"], scan_ms=r["scan_ms"], op_ms=1e3 * dt,
                        us_per_breakpoint=1e3 * r["scan_ms"] / max(r["passed"], 1)))
    print(json.dumps(dict(n=n, h=h, runs=out)), flush=True)
