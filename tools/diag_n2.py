import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2203_16340_b200 as lb, synth
t = synth.transport_ds2(1000, 9); tol = 2e-6
m, n = t.m, t.n
Md = torch.from_numpy(t.cost.reshape(-1, order="F")).cuda().reshape(n, m).T
obj = lb.TransportObjective(Md, "entropy", t.lam)
lo = torch.full((m*n,), 1e-300, dtype=torch.float64, device="cuda")
s = lb.Solver(m*n, 5, lower=lo, opts=lb.Options(tol=tol, max_iters=200000, eps=float(os.environ.get("EPS", "1e-9"))))
x = torch.zeros(m*n, dtype=torch.float64, device="cuda"); lam = torch.zeros(m+n, dtype=torch.float64, device="cuda")
r = s.al_solve_transport(obj, x, torch.from_numpy(t.u).cuda(), torch.from_numpy(t.v).cuda(), lam_out=lam, al_opts=lb.ALOptions(feas_tol=tol, max_outer=60))
print(r)
X = x.cpu().numpy().reshape(m, n, order="F"); L = lam.cpu().numpy()
G = t.cost + t.lam*(np.log(X)+1) + L[:m, None] + L[None, m:]
i, j = np.unravel_index(np.argmax(np.abs(G)), G.shape)
print("max|G|", np.abs(G).max(), "at", i, j, "X", X[i, j], "u_i", t.u[i], "v_j", t.v[j], "rowsum", X[i].sum(), "L_i", L[i], "L_j", L[m+j])
bad = np.abs(G) > 1e-4
print("nbad", bad.sum(), "rows", np.unique(np.nonzero(bad)[0])[:10], "cols", np.unique(np.nonzero(bad)[1])[:10])
print("u smallest", np.sort(t.u)[:5], "X min", X.min())
