import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth
p = synth.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]()
cu = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
obj = lb.LSQObjective(lb.colmajor(p.M), b=cu(p.b), c=cu(p.c), delta=p.delta, colscale=cu(p.colscale), split=p.split)
s = lb.Solver(p.nvars, 5, lower=cu(p.lower), upper=cu(p.upper), opts=lb.Options(max_iters=int(sys.argv[2]) if len(sys.argv) > 2 else 40))
x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
for _ in range(2):
    x.zero_(); r = s.solve(obj, x); print(r)
