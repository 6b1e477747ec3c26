"""N1 side-line: Gaussian-kernel dual SVM (gamma = 1, c = 1) on
synthetic blobs at the paper's subsample size N = 10000 (and larger)."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth
sizes = [int(a) for a in sys.argv[1:]] or [10000, 30000]
for N, d in [(N, 22) for N in sizes]:
    X, y = synth.blobs(N, d, seed=10, sep=2.0, scale=1.0 / np.sqrt(d))
    Xd = torch.from_numpy(X).cuda(); yd = torch.from_numpy(y).cuda()
    torch.cuda.synchronize(); t0 = time.perf_counter()
    K = lb.op_gaussian_kernel(Xd, 1.0)
    torch.cuda.synchronize(); tk = time.perf_counter() - t0
    obj = lb.QPObjective(K, c=-torch.ones(N, dtype=torch.float64, device="cuda"), colscale=yd)
    s = lb.Solver(N, 5, lower=torch.zeros(N, dtype=torch.float64, device="cuda"),
                  upper=torch.ones(N, dtype=torch.float64, device="cuda"), opts=lb.Options(max_iters=100000))
    x = torch.zeros(N, dtype=torch.float64, device="cuda")
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = s.al_solve(obj, x, E=yd.reshape(N, 1), e=[0.0])
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    a = x.cpu().numpy()
    print(json.dumps(dict(N=N, d=d, kernel_build_s=tk, solve_s=dt, status=r.status, f=r.f,
                          violation=r.violation_inf, outer=r.outer_iters, inner=r.inner_iters_total,
                          n_sv=int((a > 1e-8).sum()), n_bound=int((a > 1 - 1e-8).sum()))), flush=True)
    del K, obj, s
