import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth
N, d = 10000, 22
X, y = synth.blobs(N, d, seed=10, sep=2.0, scale=1.0 / np.sqrt(d))
Xd = torch.from_numpy(X).cuda(); yd = torch.from_numpy(y).cuda()
K = lb.op_gaussian_kernel(Xd, 1.0)
obj = lb.QPObjective(K, c=-torch.ones(N, dtype=torch.float64, device="cuda"), colscale=yd)
s = lb.Solver(N, 5, lower=torch.zeros(N, dtype=torch.float64, device="cuda"),
              upper=torch.ones(N, dtype=torch.float64, device="cuda"), opts=lb.Options(max_iters=60))
x = torch.zeros(N, dtype=torch.float64, device="cuda")
r = s.solve(obj, x); print(r)
