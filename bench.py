#!/usr/bin/env python
"""bench.py -- NNLS L-BFGS-B iterations/s and time-to-KKT-tolerance on B200.

One "step" = one complete ``lbfgsb_solve`` of the north-star workload from
x^0 = 0 to ||g[S]||_inf <= 1e-6 (every row of SURVEY.md 8(a): setup, all
Alg. 1 iterations with working set, vector-free two-loop, Alg. 2, Armijo
trials, fused GEMV / GEMV^T, and the final residual refresh + KKT report).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N = 1 runs BASELINE.json configs[1] (C2: dense NNLS 20000 x 10000 fp64).
N > 1 (torchrun, one rank per GPU) runs the column-sharded solve: every rank
holds a C2-sized block of columns (weak scaling, n = 10000 N) and the ranks
exchange the m-length residual partials and the packed scalar reductions
each iteration: over peer memory (--xchg p2p, default: the producing kernels
store into every rank's CUDA-IPC mailbox) or NCCL all-gathers (--xchg nccl).

value      = Alg. 1 iterations (summed over steps) / device time of the K steps
             (for N > 1: x N, i.e. C2-shard-iterations/s of the whole job)
e2e        = same metric through the C ABI with HOST (pinned) buffers:
             lbfgsb_solve_lsq_host_batch over the e2e steps' problems, every
             H2D of A and b and D2H of x* inside the call, the next problem's
             H2D overlapping the current solve (double buffering); the
             one-call-per-problem lbfgsb_solve_lsq_host number beside it.
             N > 1: the public API (Solver.solve) on pinned-host inputs,
             double-buffered the same way
roofline   = the dominant kernel (gemvT_epi, k_bwd): algorithmic bytes per
             launch / average CUDA-event launch time over K profiled steps
             (a second handle with event nodes in its graph; `value` is timed
             on a plain handle)
cpu_baseline = the CPU oracle (oracle/oracle.c, single thread) solving the
             same C2 instance to the same tolerance (rank 0, N = 1 only)

--impl reference times the oracle itself as the reference arm (bounded
sample: 2 Alg. 1 iterations of C2 per step).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

M_ROWS, N_COLS, SEED, M_HIST, TOL = 20000, 10000, 2, 5, 1e-6
METRIC = "NNLS L-BFGS-B iters/s to KKT tol 1e-6 (dense 20000x10000 fp64 per GPU)"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.idx = gpu_index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.idx), "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
            time.sleep(0.25)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if not self.proc or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sms, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [t.strip() for t in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sms) if sms else None, "sm_max_mhz": mx,
                "samples": len(sms), "reasons": sorted(reasons)}


def e2e_pipelined(lb, solvers, Mh, bh, ncols, stream, steps, dev):
    """End-to-end steps through the public API (LSQObjective + Solver.solve)
    with HOST inputs: every step copies its A (Mh: pinned (ncols, m) row-major =
    A column-major) and b from pinned memory into one of two device buffers on
    a copy stream, solves from x = 0 and reads x* back to pinned memory.  The
    copy of step k+1 is issued before the (host-synchronous) solve of step k,
    so the PCIe transfer of the next problem overlaps the current solve (double
    buffering); every step's H2D and D2H stay inside the timed region.
    solvers: two handles, one per buffer (each keeps its captured graph).
    Returns (iterations, seconds)."""
    import torch
    m = Mh.shape[1]
    cs = torch.cuda.Stream(device=dev)
    Md = [torch.empty((ncols, m), dtype=torch.float64, device=dev) for _ in range(2)]
    bd = [torch.empty(m, dtype=torch.float64, device=dev) for _ in range(2)]
    objs = [lb.LSQObjective(Md[i].t(), b=bd[i]) for i in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    x = torch.zeros(ncols, dtype=torch.float64, device=dev)
    xh = torch.zeros(ncols, dtype=torch.float64).pin_memory()

    def issue_copy(k):
        with torch.cuda.stream(cs):
            Md[k % 2].copy_(Mh, non_blocking=True)
            bd[k % 2].copy_(bh, non_blocking=True)
            done[k % 2].record(cs)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    iters = 0
    issue_copy(0)
    for k in range(steps):
        if k + 1 < steps:
            issue_copy(k + 1)          # buffer (k+1)%2 was last read by solve k-1, which has returned
        with torch.cuda.stream(stream):
            stream.wait_event(done[k % 2])
            x.zero_()
            iters += solvers[k % 2].solve(objs[k % 2], x).iters
            xh.copy_(x, non_blocking=True)
            stream.synchronize()
    dt = time.perf_counter() - t0
    return iters, dt


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    import numpy as np
    import oracle
    import synth
    p = synth.nnls_gaussian(M_ROWS, N_COLS, SEED)
    P = oracle.LSQ(p.M, b=p.b)
    iters_per_step = 2
    o = oracle.Options(tol=TOL, max_iters=iters_per_step)
    for _ in range(args.warmup):
        oracle.minimize_lsq(P, l=p.lower, m_hist=M_HIST, opts=o)
    t0 = time.perf_counter()
    tot = 0
    for _ in range(args.steps):
        r = oracle.minimize_lsq(P, l=p.lower, m_hist=M_HIST, opts=o)
        tot += r.iters
    dt = time.perf_counter() - t0
    v = tot / dt
    sample = f"C2 (20000x10000, seed {SEED}): setup + {iters_per_step} Alg. 1 iterations + final refresh per step"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "C2 dense NNLS m=20000 n=10000 fp64 (CPU oracle sample)",
                       "m": M_ROWS, "n": N_COLS, "m_hist": M_HIST},
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": 1, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def cpu_baseline_full():
    """Oracle (single thread, as it stands) solving the same C2 instance to tol."""
    import oracle
    import synth
    p = synth.nnls_gaussian(M_ROWS, N_COLS, SEED)
    t0 = time.perf_counter()
    r = oracle.minimize_lsq(oracle.LSQ(p.M, b=p.b), l=p.lower, m_hist=M_HIST,
                            opts=oracle.Options(tol=TOL))
    dt = time.perf_counter() - t0
    return {"value": r.iters / dt, "unit": "iters/s", "cores": 1, "kind": "oracle",
            "sample": f"full C2 solve to tol {TOL}: {r.iters} iterations in {dt:.2f} s "
                      f"(time-to-tol {dt:.2f} s, f={r.f:.12g}, pg={r.pg_inf:.2e})",
            "time_to_tol_s": dt, "iters": r.iters, "f": r.f}


def run_ours(args):
    import numpy as np
    import torch
    import paper_2203_16340_b200 as lb
    import synth

    ws, rank, local = _dist()
    if ws > 1 or args.force_sharded:
        return run_sharded(args)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p = synth.nnls_gaussian(M_ROWS, N_COLS, SEED)
    M = lb.colmajor(p.M, device=dev)
    b = torch.from_numpy(p.b).to(dev)
    lo = torch.zeros(N_COLS, dtype=torch.float64, device=dev)
    obj = lb.LSQObjective(M, b=b)
    stream = torch.cuda.Stream(device=dev)
    # `value` is timed on a plain handle; the per-kernel CUDA events (3 event-record nodes per
    # iteration inside the replayed graph, ~4% of the step) ride on a second, profiled handle
    # whose own K timed steps give the roofline numbers.
    solver = lb.Solver(N_COLS, M_HIST, lower=lo, opts=lb.Options(tol=TOL), stream=stream)
    solver_p = lb.Solver(N_COLS, M_HIST, lower=lo, opts=lb.Options(tol=TOL, profile=True), stream=stream)
    x = torch.zeros(N_COLS, dtype=torch.float64, device=dev)

    def timed(sv, k):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its, res = 0, []
        torch.cuda.synchronize()
        ev0.record(stream)
        for _ in range(k):
            x.zero_()
            r = sv.solve(obj, x)
            its += r.iters
            res.append(r)
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1), its, res

    with torch.cuda.stream(stream):
        for sv in (solver, solver_p):
            for _ in range(max(args.warmup, 3)):
                x.zero_()
                sv.solve(obj, x)
        torch.cuda.synchronize()
        solver.profile(reset=True)
        with ClockSampler(local) as clk:
            ms, iters, results = timed(solver, args.steps)
        launches = solver.profile(reset=True)["all_kernel_launches"][1]
        solver_p.profile(reset=True)
        ms_p, _, _ = timed(solver_p, args.steps)
        prof = solver_p.profile(reset=True)
    clocks = clk.summary()
    value = iters / (ms / 1e3)
    r0 = results[-1]
    ms_per_step = ms / args.steps

    # ---- roofline of the dominant kernel (k_bwd = gemvT_epi), live CUDA events
    peak, peak_src = _peaks()
    bwd_ms, bwd_n = prof["gemvT_epi (k_bwd)"]
    fwd_ms, fwd_n = prof["gemv_active (k_fwd)"]
    nact = prof.get("fwd_active_columns", (0, 0))[1]
    # algorithmic bytes of one k_bwd launch: A (8 m n) + r (8 m) + per-variable
    # epilogue reads x, g, p, l, u and writes x, g, s, y (9 x 8 n)
    bwd_bytes = 8 * M_ROWS * N_COLS + 8 * M_ROWS + 9 * 8 * N_COLS
    bwd_avg_s = (bwd_ms / max(bwd_n, 1)) / 1e3
    achieved = bwd_bytes / bwd_avg_s / 1e9 if bwd_n else None
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "r01_kbwd_dram_bytes.json")
    if os.path.exists(tfile):
        traffic = json.load(open(tfile)).get("dram_bytes_per_launch")
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "kernel": "k_bwd_s (gemvT_epi: g = M^T r + fused Alg. 1 epilogue, Gram, Alg. 3 tail)",
                "bytes_per_launch": bwd_bytes, "avg_launch_us": bwd_avg_s * 1e6,
                "launches": bwd_n, "peak_source": peak_src,
                "share_of_step": (bwd_ms / ms_p) if ms_p else None,
                "k_fwd_share_of_step": (fwd_ms / ms_p) if ms_p else None,
                "events": f"CUDA events around every k_fwd / k_bwd launch of {args.steps} profiled steps "
                          f"({ms_p / args.steps:.3f} ms per step with the event nodes)",
                "k_fwd_avg_launch_us": 1e3 * fwd_ms / max(fwd_n, 1)}
    if fwd_n and nact:
        # k_fwd reads only the active columns: 8 m n_p + qpart / r / q vectors
        cols = nact / fwd_n
        fb = 8 * M_ROWS * cols + 8 * M_ROWS * 4 + 8 * 3 * N_COLS
        roofline["k_fwd_active_cols_avg"] = cols
        roofline["k_fwd_bytes_per_launch"] = fb
        roofline["k_fwd_achieved_gbs"] = fb / (fwd_ms / fwd_n / 1e3) / 1e9
        # whole-iteration algorithmic bandwidth (B_it = 8 m (n + n_p) + V)
        v_bytes = 8 * ((4 * M_HIST + 16) * N_COLS + 8 * M_ROWS)
        roofline["iteration_bytes_avg"] = 8 * M_ROWS * (N_COLS + cols) + v_bytes

    # ---- e2e: the C-ABI call with HOST buffers.  lbfgsb_solve_lsq_host_batch solves the
    # e2e steps' problems (each its own pinned copy of A, b, x) in one call, double-buffered:
    # problem k+1's H2D overlaps problem k's solve; every H2D / D2H is inside the timed call.
    # The one-problem-per-call lbfgsb_solve_lsq_host (copy, then solve) is reported beside it.
    e2e_steps = max(3, min(args.steps, 10))
    Mt = torch.from_numpy(np.ascontiguousarray(p.M.T)).pin_memory()            # (n, m) = A col-major
    bt = torch.from_numpy(p.b.copy()).pin_memory()
    Mhs = [Mt.numpy().T] + [torch.empty_like(Mt).pin_memory().copy_(Mt).numpy().T for _ in range(1)]
    bhs = [bt.numpy(), torch.empty_like(bt).pin_memory().copy_(bt).numpy()]
    xhs = [torch.zeros(N_COLS, dtype=torch.float64).pin_memory().numpy() for _ in range(e2e_steps)]
    solver_h = lb.Solver(N_COLS, M_HIST, lower=lo, opts=lb.Options(tol=TOL), stream=stream)
    Ms = [Mhs[k % 2] for k in range(e2e_steps)]           # consecutive problems live in distinct host buffers
    bs = [bhs[k % 2] for k in range(e2e_steps)]
    solver_h.solve_lsq_host_batch(Ms[:2], bs[:2], xhs[:2])                      # warm-up (graphs, buffers)
    for xx in xhs:
        xx[:] = 0.0
    t0 = time.perf_counter()
    rs_ = solver_h.solve_lsq_host_batch(Ms, bs, xhs)
    e2e_dt = time.perf_counter() - t0
    e2e_iters = sum(r_.iters for r_ in rs_)
    xh = xhs[0]
    xh[:] = 0.0
    solver_h.solve_lsq_host(Mhs[0], bhs[0], xh)
    t0 = time.perf_counter()
    s_iters = 0
    for _ in range(e2e_steps):
        xh[:] = 0.0
        s_iters += solver_h.solve_lsq_host(Mhs[0], bhs[0], xh).iters
    s_dt = time.perf_counter() - t0
    e2e = {"value": e2e_iters / e2e_dt, "unit": "iters/s",
           "h2d_bytes_per_step": 8 * (M_ROWS * N_COLS + M_ROWS + N_COLS),
           "d2h_bytes_per_step": 8 * N_COLS, "steps": e2e_steps,
           "ms_per_step": 1e3 * e2e_dt / e2e_steps,
           "api": "lbfgsb_solve_lsq_host_batch (C ABI, pinned HOST A, b, x per problem; H2D of problem k+1 "
                  "overlaps the solve of problem k; host wall clock around the call)",
           "serial_lbfgsb_solve_lsq_host": {"value": s_iters / s_dt, "ms_per_step": 1e3 * s_dt / e2e_steps}}

    cpu = None if args.no_cpu_baseline else cpu_baseline_full()
    line = {
        "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy: A_ij ~ N(0,1)/sqrt(m), b ~ N(0,1); SURVEY 8(d) C2)",
        "config": {"workload": "C2: dense NNLS m=20000 n=10000 fp64, x>=0, m_hist=5, tol 1e-6 "
                               "(BASELINE.json configs[1])",
                   "m": M_ROWS, "n": N_COLS, "m_hist": M_HIST, "tol": TOL, "seed": SEED,
                   "l2": "inputs larger than L2 (A = 1.6 GB > 126 MB); no flush",
                   "parallelism": "single GPU"},
        "time_to_tol_ms": ms_per_step, "iters_per_solve": r0.iters, "f": r0.f,
        "pg_inf": r0.pg_inf, "status": r0.status_name,
        "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
        "gpu_launches": launches, "clocks": clocks,
        "paper_context": "paper: 0.8 s modified L-BFGS-B GPU / 4.9 s CPU L-BFGS-B on NNLS size 12000 "
                         "(Quadro RTX 4000 / i9-10980XE, PAPER.md:449-451); different sizes/hardware",
    }
    print(json.dumps(line), flush=True)
    return 0


def run_sharded(args) -> int:
    """N > 1 step: every rank holds a C2-sized column block (weak scaling,
    n = 10000 N); value = Alg. 1 iterations x N / max-over-ranks device time.
    The per-iteration exchange runs over peer memory (--xchg p2p, the
    default: the producing kernels store their packs into every rank's CUDA-IPC
    mapped mailbox) or through the library's NCCL communicator (--xchg nccl);
    if any rank cannot map its peers, all ranks fall back to NCCL and the
    line says so."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2203_16340_b200 as lb
    import synth
    from paper_2203_16340_b200 import sharded

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29517")
    os.environ.setdefault("RANK", "0")
    os.environ.setdefault("WORLD_SIZE", "1")
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    m, ncl, seed, mh, tol = 20000, 10000, 2, 5, 1e-6
    p = synth.weak_shard(m, ncl, rank, seed)
    dev = torch.device("cuda", local)
    M = lb.colmajor(p.M, device=dev)
    b = torch.from_numpy(p.b).to(dev)
    lo = torch.zeros(ncl, dtype=torch.float64, device=dev)
    stream = torch.cuda.Stream(device=dev)
    xchg, err = args.xchg, ""

    def make(profile):
        """One sharded handle per timing pass (plain for `value`, profiled for the roofline)."""
        nonlocal xchg, err
        opts = lb.Options(tol=tol, profile=profile)
        sv = None
        if xchg == "p2p":
            try:
                sv = lb.Solver(ncl, mh, lower=lo, opts=opts, stream=stream, rank=rank, nranks=world,
                               n_global=ncl * world, p2p_m_max=m)
                sv.p2p_open(sharded.all_gather_bytes(sv.ipc_handle()))
            except Exception as e:      # noqa: BLE001 -- collective decision below
                sv, err = None, f"{type(e).__name__}: {e}"[:200]
            oks = sharded.all_gather_bytes(b"1" if sv is not None else err.encode() or b"0")
            if any(o != b"1" for o in oks):
                sv, xchg = None, "nccl"
                err = "; ".join(o.decode() for o in oks if o != b"1")
            dist.barrier()
        if sv is None:
            sv = sharded.make_sharded_solver(ncl, ncl * world, mh, lo, opts, stream, xchg="nccl")
        return sv

    solver = make(False)
    solver_p = make(True)
    obj = lb.LSQObjective(M, b=b)
    x = torch.zeros(ncl, dtype=torch.float64, device=dev)

    def timed(sv):
        torch.cuda.synchronize()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = 0
        e0.record(stream)
        for _ in range(args.steps):
            x.zero_()
            rr = sv.solve(obj, x)
            its += rr.iters
        e1.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
        return sharded.max_over_ranks(e0.elapsed_time(e1), device=dev), its, rr

    with torch.cuda.stream(stream):
        for sv in (solver, solver_p):
            for _ in range(max(args.warmup, 3)):
                x.zero_()
                sv.solve(obj, x)
        solver.profile(reset=True)
        with ClockSampler(local) as clk:
            ms, iters, r = timed(solver)
        launches = solver.profile(reset=True)["all_kernel_launches"][1]
        solver_p.profile(reset=True)
        ms_p, _, _ = timed(solver_p)
    prof = solver_p.profile(reset=True)
    clocks = clk.summary()
    all_reasons = sharded.all_gather_bytes(json.dumps(clocks.get("reasons", [])).encode())

    # ---- e2e through the public API: every rank copies its A block and b from pinned
    # host memory (double-buffered, e2e_pipelined), solves, reads x back; max over ranks
    Mt = torch.from_numpy(np.ascontiguousarray(p.M.T)).pin_memory()     # (ncl, m) row-major = A col-major
    bt = torch.from_numpy(p.b.copy()).pin_memory()
    e2e_steps = max(3, min(args.steps, 10))
    pair = [solver, make(False)]
    e2e_pipelined(lb, pair, Mt, bt, ncl, stream, 2, dev)
    torch.cuda.synchronize()
    dist.barrier()
    e2e_iters, e2e_dt = e2e_pipelined(lb, pair, Mt, bt, ncl, stream, e2e_steps, dev)
    e2e_dt = sharded.max_over_ranks(e2e_dt, device=dev)
    if rank == 0:
        peak, peak_src = _peaks()
        value = iters * world / (ms / 1e3)
        bwd_ms, bwd_n = prof["gemvT_epi (k_bwd)"]
        bwd_bytes = 8 * m * ncl + 8 * m + 9 * 8 * ncl
        achieved = (bwd_bytes / (bwd_ms / bwd_n / 1e3) / 1e9) if bwd_n else None
        reasons = sorted({x for rs in all_reasons for x in json.loads(rs)})
        clocks["reasons"] = reasons
        clocks["note"] = "sm_mhz sampled on rank 0's GPU; reasons merged over all ranks"
        line = {"metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded numpy per rank: A_r ~ N(0,1)/sqrt(m), b ~ N(0,1))",
                "config": {"workload": f"column-sharded NNLS m={m} n={ncl}x{world} fp64 "
                                       f"(C2-sized block per GPU, weak scaling)",
                           "m": m, "n_local": ncl, "n_global": ncl * world, "m_hist": mh,
                           "tol": tol,
                           "parallelism": f"column-sharded x{world} ("
                                          + ("P2P mailboxes over NVLink, pushes fused in the producing "
                                             "kernels" if xchg == "p2p" else "NCCL all-gather") + ")",
                           "xchg": xchg, "xchg_fallback_reason": err or None,
                           "l2": "inputs larger than L2"},
                "iters_per_solve": r.iters, "f": r.f, "pg_inf": r.pg_inf,
                "roofline": {"bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": peak,
                             "frac": (achieved / peak) if achieved else None, "traffic": None,
                             "peak_source": peak_src, "bytes_per_launch": bwd_bytes,
                             "avg_launch_us": 1e3 * bwd_ms / max(bwd_n, 1),
                             "kernel": "k_bwd_s (rank 0)",
                             "events": f"CUDA events around every k_bwd launch of {args.steps} profiled steps "
                                       f"({ms_p / args.steps:.3f} ms per step with the event nodes)"},
                "e2e": {"value": e2e_iters * world / e2e_dt, "unit": "iters/s",
                        "h2d_bytes_per_step": 8 * (m * ncl + m) * world, "d2h_bytes_per_step": 8 * ncl * world,
                        "steps": e2e_steps, "ms_per_step": 1e3 * e2e_dt / e2e_steps,
                        "api": "Solver.solve (lbfgsb_solve) on pinned-host inputs: per step every rank's "
                               "A block and b copied H2D (double-buffered, overlapping the previous solve), "
                               "D2H of x; host wall clock, max over ranks"},
                "gpu_launches": launches, "clocks": clocks}
        print(json.dumps(line), flush=True)
    dist.barrier()
    for sv in (solver, solver_p, pair[1]):
        sv.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--xchg", choices=["p2p", "nccl"], default="p2p",
                    help="N>1 exchange: peer-memory mailboxes (default) or NCCL all-gather")
    ap.add_argument("--force-sharded", action="store_true",
                    help="run the N>1 sharded code path even at N=1 (1-rank communicator)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
