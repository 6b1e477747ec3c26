"""Per-CTA phase timeline of the iteration kernels inside a solve (A/B tool).

Needs a variant library built with -DLB_TRACE (tools/_var/lib_trace.so):
  python tools/_prof_with_lib.py tools/_var/lib_trace.so tools/trace_phases.py c2|c4|c5chunk

Every CTA of k_bwd_s (kid 1), k_bwd_w (2), k_fwd (4) and k_dir (5) appends one
record with %globaltimer stamps at its phase boundaries (common.cuh TR_*); the
last CTA of k_fwd / k_dir appends a second record for the global tail (14, 15).
Launches are separated by the append order (the stream serialises them).
Prints, per kernel, the median over the solve's launches of: launch span
(first CTA entry -> last CTA exit), the phase lengths averaged over CTAs, and
the spread of CTA finish times (load balance)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2203_16340_b200 as lb  # noqa: E402
import synth  # noqa: E402

shape = sys.argv[1] if len(sys.argv) > 1 else "c2"
if shape == "c5chunk":
    m, n = 100000, 25000
    A, b, _ = synth.c5_device(m, n, seed=5)
    b = torch.from_numpy(b).cuda()
elif shape == "c2":
    m, n = 20000, 10000
    p = synth.nnls_gaussian(m, n, 2)
    A, b = lb.colmajor(p.M), torch.from_numpy(p.b).cuda()
else:
    m, n = 1000, 100000
    rng = np.random.default_rng(4)
    A = lb.colmajor(rng.standard_normal((m, n)) / np.sqrt(m))
    b = torch.from_numpy(rng.standard_normal(m)).cuda()

L = lb.load(build_if_needed=False)
CAP = 1 << 20
recs = torch.zeros(CAP * 8, dtype=torch.int64, device="cuda")       # 64-byte records
cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
L.lbfgsb_trace_set.argtypes = [C.c_void_p, C.c_void_p]

obj = lb.LSQObjective(A, b=b)
s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"), opts=lb.Options())
x = torch.zeros(n, dtype=torch.float64, device="cuda")
s.solve(obj, x)                                     # warm (graph capture)
x.zero_()
torch.cuda.synchronize()
L.lbfgsb_trace_set(C.c_void_p(recs.data_ptr()), C.c_void_p(cnt.data_ptr()))
r = s.solve(obj, x)
torch.cuda.synchronize()
L.lbfgsb_trace_set(None, None)
k = min(int(cnt.item()), CAP)
raw = recs[: k * 8].view(k, 8).cpu().numpy()
t = raw[:, :6].astype(np.float64)
meta = raw[:, 6:8].copy().view(np.int32).reshape(k, 4)   # kid, cta, smid, aux
kid = meta[:, 0]

names = {1: "k_bwd_s", 2: "k_bwd_w", 3: "k_bwd_wd", 4: "k_fwd", 5: "k_dir"}
nmarks = {1: 5, 2: 4, 3: 6, 4: 2, 5: 2}
out = {"shape": shape, "iters": r.iters, "records": k, "kernels": {}}
allspans = []
for kd, nm in names.items():
    idx = np.nonzero(kid == kd)[0]
    if idx.size == 0:
        continue
    # split into launches: a new launch starts when the cta index repeats
    launches, cur, seen = [], [], set()
    for i in idx:
        c = meta[i, 1]
        if c in seen:
            launches.append(cur); cur, seen = [], set()
        cur.append(i); seen.add(c)
    if cur:
        launches.append(cur)
    nm_ = nmarks[kd]
    per = []
    for ln in launches:
        allspans.append((t[ln, 0].min(), t[ln, nmarks[kd] - 1].max(), nm))
        T = t[ln, :nm_]
        start = T[:, 0].min()
        ends = T[:, nm_ - 1]
        ph = np.diff(T, axis=1)
        per.append({"ctas": len(ln), "span_us": (ends.max() - start) / 1e3,
                    "entry_spread_us": (T[:, 0].max() - start) / 1e3,
                    "phase_mean_us": (ph.mean(axis=0) / 1e3).round(2).tolist(),
                    "phase_max_us": (ph.max(axis=0) / 1e3).round(2).tolist(),
                    "end_p50_us": (np.median(ends) - start) / 1e3,
                    "end_min_us": (ends.min() - start) / 1e3})
    # the iteration launches: the most common CTA count, drop the first and last (setup / refresh)
    body = per[1:-1] if len(per) > 3 else per
    med = {key: float(np.median([p[key] for p in body])) for key in ("span_us", "entry_spread_us", "end_p50_us",
                                                                     "end_min_us")}
    med["phase_mean_us"] = np.median(np.array([p["phase_mean_us"] for p in body]), axis=0).round(2).tolist()
    med["phase_max_us"] = np.median(np.array([p["phase_max_us"] for p in body]), axis=0).round(2).tolist()
    med["launches"] = len(per)
    med["ctas"] = per[len(per) // 2]["ctas"]
    out["kernels"][nm] = med
# optional: per-CTA records of one mid-solve launch of a kernel (TRACE_DUMP=name), for placement analysis
dump = os.environ.get("TRACE_DUMP")
if dump:
    kd = {v: k for k, v in names.items()}[dump]
    idx = np.nonzero(kid == kd)[0]
    launches, cur, seen = [], [], set()
    for i in idx:
        c = meta[i, 1]
        if c in seen:
            launches.append(cur); cur, seen = [], set()
        cur.append(i); seen.add(c)
    ln = launches[len(launches) // 2]
    t0 = t[ln, 0].min()
    recs = [{"cta": int(meta[i, 1]), "sm": int(meta[i, 2]), "aux": int(meta[i, 3]),
             "t": [round((t[i, q] - t0) / 1e3, 3) for q in range(nmarks[kd])]} for i in ln]
    out["dump"] = {"kernel": dump, "records": recs}
# k_fwd tails: row-block finisher (kid 24: [entry, stream end, row-block ticket won, q + trial sums done]) and
# the global finisher (kid 14: [.., global ticket won, Armijo done]); k_dir global tail (kid 15: [.., ticket, done])
idx = np.nonzero(kid == 24)[0]
if idx.size:
    out["kernels"]["k_fwd_rowblock_tail"] = {"work_us_median": float(np.median((t[idx, 3] - t[idx, 2]) / 1e3)),
                                             "records": int(idx.size)}
idx = np.nonzero(kid == 14)[0]
if idx.size:
    out["kernels"]["k_fwd_tail"] = {"rowblock_work_us_median": float(np.median((t[idx, 3] - t[idx, 2]) / 1e3)),
                                    "ticket_us_median": float(np.median((t[idx, 4] - t[idx, 3]) / 1e3)),
                                    "global_work_us_median": float(np.median((t[idx, 5] - t[idx, 4]) / 1e3)),
                                    "launches": int(idx.size)}
idx = np.nonzero(kid == 15)[0]
if idx.size:
    out["kernels"]["k_dir_tail"] = {"tail_us_median": float(np.median((t[idx, 3] - t[idx, 2]) / 1e3)),
                                    "launches": int(idx.size)}
# launch ends of k_fwd / k_dir: their global tails (the i-th tail record belongs to the i-th launch)
for kd, nm, col in ((14, "k_fwd", 5), (15, "k_dir", 3)):
    idx = np.nonzero(kid == kd)[0]
    spans_k = [i for i, sp in enumerate(allspans) if sp[2] == nm]
    for i, rec in zip(spans_k, idx):
        s0, e0, n0 = allspans[i]
        allspans[i] = (s0, max(e0, t[rec, col]), n0)
# Gram tail of the last CTA (kid 11): level-1 ticket | level-1 reduce | level-2 ticket | level-2 reduce | Alg. 3
idx = np.nonzero(kid == 11)[0]
if idx.size:
    ph = np.diff(t[idx, :6], axis=1) / 1e3
    out["kernels"]["gram_tail_last_cta"] = {"phases_us_median": np.median(ph, axis=0).round(2).tolist(),
                                            "total_us_median": float(np.median((t[idx, 5] - t[idx, 0]) / 1e3)),
                                            "launches": int(idx.size)}
# gaps between kernels: launches in time order, exit of one -> entry of the next
allspans.sort()
gaps = {}
for (s0, e0, n0), (s1, e1, n1) in zip(allspans, allspans[1:]):
    gaps.setdefault(f"{n0}->{n1}", []).append((s1 - e0) / 1e3)
out["gaps_us_median"] = {kk: round(float(np.median(v)), 2) for kk, v in gaps.items() if len(v) > 2}
tot = (allspans[-1][1] - allspans[0][0]) / 1e3 if allspans else 0.0
out["solve_span_us"] = tot
print(json.dumps(out))
