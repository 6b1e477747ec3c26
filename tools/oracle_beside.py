"""The oracle timed beside the GPU path on the same seeded inputs for the
NEXT rows (N1 kernel SVM, N2 joint probability, N3 Cauchy point, N4 batched),
at sizes the oracle finishes in seconds.  One JSON line per case."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth
import paper_2203_16340_b200 as lb

cu = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
out = []

def emit(**kw):
    print(json.dumps(kw), flush=True)

# N1: Gaussian-kernel dual SVM (AL), N = 600
prob = synth.svm_dual_kernel(600, 5, 7, gamma=1.0, C=1.0)
P = oracle.LSQ(prob.M, c=prob.c, colscale=prob.colscale, qp=True, E=prob.E, e=prob.e)
t0 = time.perf_counter()
ro = oracle.al_solve(P, l=prob.lower, u=prob.upper, opts=oracle.Options(tol=1e-6, max_iters=50000),
                     al_opts=oracle.ALOptions(feas_tol=1e-6))
to = time.perf_counter() - t0
Kd = lb.op_gaussian_kernel(cu(prob.meta["X"]), 1.0)
obj = lb.QPObjective(Kd, c=cu(prob.c), colscale=cu(prob.colscale))
s = lb.Solver(prob.nvars, 5, lower=cu(prob.lower), upper=cu(prob.upper), opts=lb.Options(tol=1e-6, max_iters=50000))
x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
s.al_solve(obj, x, E=cu(prob.E), e=prob.e)
torch.cuda.synchronize(); t0 = time.perf_counter()
r = s.al_solve(obj, x, E=cu(prob.E), e=prob.e, al_opts=lb.ALOptions(feas_tol=1e-6))
torch.cuda.synchronize(); tg = time.perf_counter() - t0
emit(case="N1 kernel SVM N=600 (AL, tol 1e-6)", oracle_s=to, oracle_f=ro.f, oracle_inner=ro.inner_iters_total,
     gpu_s=tg, gpu_f=r.f, gpu_inner=r.inner_iters_total, rel_df=abs(r.f - ro.f) / abs(ro.f))

# N2: DS2 n = 60 (120 x 60), both regularisers
for reg in ["gaussian", "entropy"]:
    t = synth.transport_ds2(60, 3)
    m, n = t.m, t.n
    lo = 1e-300 if reg == "entropy" else 0.0
    P = oracle.LSQ.transport(t.cost, t.u, t.v, reg, t.lam)
    t0 = time.perf_counter()
    ro = oracle.al_solve(P, l=np.full(m * n, lo), opts=oracle.Options(tol=1e-6, armijo_diff=True, max_iters=100000),
                         al_opts=oracle.ALOptions(feas_tol=1e-6))
    to = time.perf_counter() - t0
    Md = cu(t.cost.reshape(-1, order="F")).reshape(n, m).T
    obj = lb.TransportObjective(Md, reg, t.lam)
    s = lb.Solver(m * n, 5, lower=torch.full((m * n,), lo, dtype=torch.float64, device="cuda"),
                  opts=lb.Options(tol=1e-6, max_iters=100000))
    x = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = s.al_solve_transport(obj, x, cu(t.u), cu(t.v), al_opts=lb.ALOptions(feas_tol=1e-6))
    torch.cuda.synchronize(); tg = time.perf_counter() - t0
    emit(case=f"N2 DS2 {m}x{n} {reg} (tol 1e-6)", oracle_s=to, oracle_f=ro.f, oracle_inner=ro.inner_iters_total,
         gpu_s=tg, gpu_f=r.f, gpu_inner=r.inner_iters_total, rel_df=abs(r.f - ro.f) / max(abs(ro.f), 1e-12))

# N3: one Cauchy point, n = 10000, h = 5
n = 10000
rng = np.random.default_rng(n)
xx = rng.uniform(0.05, 0.95, n); g = rng.standard_normal(n)
S = rng.standard_normal((5, n)) / np.sqrt(n); Y = S + 0.3 * rng.standard_normal((5, n)) / np.sqrt(n)
theta = float(Y[-1] @ Y[-1] / (S[-1] @ Y[-1]))
t0 = time.perf_counter()
xo, co, po = oracle.cauchy_point(xx, g, np.zeros(n), np.ones(n), S, Y, theta)
to = time.perf_counter() - t0
sv = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"),
               upper=torch.ones(n, dtype=torch.float64, device="cuda"))
rr = sv.op_cauchy_point(cu(xx), cu(g), cu(S), cu(Y), theta)
emit(case="N3 Cauchy point n=10000 h=5", oracle_s=to, oracle_passed=po, gpu_scan_s=rr["scan_ms"] / 1e3,
     gpu_passed=rr["passed"], max_dx=float(np.max(np.abs(rr["xcp"].cpu().numpy() - xo))))

# N4: 148 C1 problems
B, m, n = 148, 200, 100
probs = [synth.nnls_gaussian(m, n, 5000 + k) for k in range(B)]
t0 = time.perf_counter()
fo = [oracle.minimize_lsq(oracle.LSQ(p.M, b=p.b), l=p.lower).f for p in probs]
to = time.perf_counter() - t0
A = np.stack([p.M for p in probs]); b = np.stack([p.b for p in probs])
M = lb.colmajor_batch(A); bd = cu(b)
xb = torch.zeros(B, n, dtype=torch.float64, device="cuda"); lo = torch.zeros(B, n, dtype=torch.float64, device="cuda")
lb.solve_batched_lsq(M, bd, xb, lower=lo)
xb.zero_(); torch.cuda.synchronize(); t0 = time.perf_counter()
res = lb.solve_batched_lsq(M, bd, xb, lower=lo)
torch.cuda.synchronize(); tg = time.perf_counter() - t0
emit(case="N4 148 x C1 NNLS (200x100)", oracle_s=to, gpu_s=tg,
     max_rel_df=max(abs(r.f - f) / abs(f) for r, f in zip(res, fo)), cores=1)
