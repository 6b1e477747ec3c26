"""N4 side-line: B independent C1-size NNLS problems (200 x 100) solved in one
launch (one CTA per problem) vs one lbfgsb_solve per problem."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth
m, n = 200, 100
for B in [int(a) for a in sys.argv[1:]] or [148, 1184, 4736]:
    probs = [synth.nnls_gaussian(m, n, 5000 + k) for k in range(B)]
    A = np.stack([p.M for p in probs]); b = np.stack([p.b for p in probs])
    M = lb.colmajor_batch(A); bd = torch.from_numpy(b).cuda()
    lo = torch.zeros(B, n, dtype=torch.float64, device="cuda")
    x = torch.zeros(B, n, dtype=torch.float64, device="cuda")
    lb.solve_batched_lsq(M, bd, x, lower=lo)                                  # warm-up
    x.zero_(); torch.cuda.synchronize(); t0 = time.perf_counter()
    res = lb.solve_batched_lsq(M, bd, x, lower=lo)
    torch.cuda.synchronize(); tb = time.perf_counter() - t0
    iters = np.array([r.iters for r in res]); ok = sum(r.status == 0 for r in res)
    # one-at-a-time reference on the first 32
    k1 = min(B, 32); ts = 0.0
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"))
    for k in range(k1):
        obj = lb.LSQObjective(lb.colmajor(probs[k].M), b=torch.from_numpy(probs[k].b).cuda())
        xk = torch.zeros(n, dtype=torch.float64, device="cuda")
        torch.cuda.synchronize(); t0 = time.perf_counter()
        s.solve(obj, xk)
        torch.cuda.synchronize(); ts += time.perf_counter() - t0
    print(json.dumps(dict(batch=B, m=m, n=n, batched_s=tb, problems_per_s=B / tb, converged=int(ok),
                          iters_mean=float(iters.mean()), iters_max=int(iters.max()),
                          single_solve_ms=1e3 * ts / k1, speedup=(ts / k1) / (tb / B))), flush=True)
