"""C5 (100000 x 200000, 160 GB, device-generated) on one B200: solve + kernel timings."""
import os, sys, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2203_16340_b200 as lb
import synth
m, n = (int(a) for a in sys.argv[1:3]) if len(sys.argv) > 2 else (100000, 200000)
t0 = time.perf_counter()
A, b, xp = synth.c5_device(m, n, seed=5)
torch.cuda.synchronize(); tg = time.perf_counter() - t0
obj = lb.LSQObjective(A, b=torch.from_numpy(b).cuda())
s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"), opts=lb.Options(profile=True, max_iters=20000))
x = torch.zeros(n, dtype=torch.float64, device="cuda")
for rep in range(2):
    s.profile(reset=True)
    x.zero_(); torch.cuda.synchronize(); t0 = time.perf_counter()
    r = s.solve(obj, x); torch.cuda.synchronize(); dt = time.perf_counter() - t0
prof = s.profile()
bw = prof["gemvT_epi (k_bwd)"]; fw = prof["gemv_active (k_fwd)"]; nact = prof["fwd_active_columns"][1]
out = dict(m=m, n=n, gen_s=tg, solve_s=dt, iters=r.iters, f=r.f, pg=r.pg_inf, status=r.status_name,
           n_fg=r.n_fg, bwd_avg_ms=bw[0] / max(bw[1], 1), fwd_avg_ms=fw[0] / max(fw[1], 1),
           bwd_gbs=8 * m * n / (bw[0] / bw[1] / 1e3) / 1e9 if bw[1] else None,
           fwd_active=nact / max(fw[1], 1),
           fwd_gbs=8 * m * (nact / fw[1]) / (fw[0] / fw[1] / 1e3) / 1e9 if fw[1] else None,
           iters_per_s=r.iters / dt)
print(json.dumps(out))
