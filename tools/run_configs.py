"""Run the BASELINE configs C1-C4 end to end on the GPU (exploration / bench side-lines)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth

def run(name, prob, al=False, tol=1e-6):
    M = lb.colmajor(prob.M)
    cu = lambda a: None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()
    obj = lb.LSQObjective(M, b=cu(prob.b), c=cu(prob.c), delta=prob.delta, colscale=cu(prob.colscale), split=prob.split)
    s = lb.Solver(prob.nvars, 5, lower=cu(prob.lower), upper=cu(prob.upper), opts=lb.Options(tol=tol, max_iters=100000))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    out = {}
    for rep in range(2):
        x.zero_(); torch.cuda.synchronize(); t0 = time.perf_counter()
        if al:
            r = s.al_solve(obj, x, E=cu(prob.E), e=prob.e)
        else:
            r = s.solve(obj, x)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
        out = dict(name=name, wall_s=dt, **{k: getattr(r, k) for k in r.__dataclass_fields__ if not isinstance(getattr(r, k), list)})
    print(json.dumps(out), flush=True)
    return x.cpu().numpy(), r

which = sys.argv[1:] or ["C1", "C2", "C3", "C3en", "C4"]
for c in which:
    p = synth.CONFIGS[c]()
    run(c, p, al=(p.kind == "svm"))
