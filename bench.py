#!/usr/bin/env python
"""bench.py -- NNLS L-BFGS-B iterations/s and time-to-KKT-tolerance on 1/2/4/8 B200.

One "step" = one complete solve of the workload from x^0 = 0 to
||g[S]||_inf <= 1e-6 (every row of SURVEY.md 8(a): setup, all Alg. 1
iterations with working set, vector-free two-loop, Alg. 2, Armijo trials,
fused GEMV / GEMV^T, the cross-GPU exchange, and the final residual refresh +
KKT report).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config C5|C2]

--config C5 (default, every N): BASELINE.json configs[4], the column-sharded
  NNLS 100000 x 200000 fp64 (A = 160 GB, generated on the device by the
  counter-based Philox generator), STRONG scaling: the same global problem at
  N = 1, 2, 4, 8.  Its n columns are C = 8 fixed chunks (logical ranks,
  lbfgsb_solve_group); process p of N hosts 8 / N of them and the exchange
  runs over CUDA-IPC mailboxes (NVLink P2P stores from the producing
  kernels), so x, f and the iteration count are bitwise identical at every N
  and time-to-tol scaling equals per-iteration scaling.
  At N = 1 the line also carries "c2": the BASELINE.json configs[1]
  measurement (dense NNLS 20000 x 10000, the k_bwd_s roofline, its e2e
  through host buffers and its oracle baselines).
--config C2: the C2 line alone (single GPU).

value        = Alg. 1 iterations (summed over steps) / device time of the K steps
               (CUDA events on the solver stream, max over ranks)
e2e          = same metric through the public API with host inputs each step
               (C5: pinned b and x0 H2D, the rank's A chunks regenerated on the device
               from the seed -- the data set is the generator, no host holds 160 GB --,
               x* D2H; C2: lbfgsb_solve_lsq_host_batch with pinned A, b, x)
roofline     = the dominant kernel (gemvT_epi, k_bwd): algorithmic bytes per
               launch / average CUDA-event launch time over K profiled steps
               (a second handle group with event nodes; `value` is timed on a
               plain one)
cpu_baseline = the CPU oracle (oracle/oracle.c) on 1 thread and on all host
               cores (OpenMP over output elements, bit-identical): C5 on a
               bounded column sample, scaled to the full problem; C2 in full

--impl reference times the oracle itself as the reference arm on the same
config: C2 = the same full solve per step; C5 = a bounded column sample per step.
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
# context for roofline.frac above 1: the copy peak counts read + write bytes, a read-dominated stream can
# exceed it; the measured pure-read ceiling of this GPU type (a GEMV^T-shaped TMA stream of the C2 matrix,
# tools/bw_probe.cu) is reported beside it
READ_PROBE_GBS = 7170.0
READ_PROBE_SRC = "profiles/r01_bw_probe.txt (seg_stream: 1.6 GB GEMV^T-shaped TMA column stream, 7.17 TB/s)"
sys.path.insert(0, ROOT)

M_ROWS, N_COLS, SEED, M_HIST, TOL = 20000, 10000, 2, 5, 1e-6
METRIC = "NNLS L-BFGS-B iters/s to KKT tol 1e-6 (dense 20000x10000 fp64 per GPU)"
C5_M, C5_N, C5_SEED, C5_CHUNKS = 100000, 200000, 5, 8
METRIC_C5 = ("NNLS L-BFGS-B iters/s to KKT tol 1e-6 (C5: column-sharded 100000x200000 fp64, "
             "strong scaling over 1/2/4/8 B200)")


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d.get("hbm_gbs", 6650.0)), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _host_cpu():
    """CPU model and usable core count of this host (for the oracle baselines)."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count() or 1
    return model, cores


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


# ----------------------------------------------------------------------------- oracle baselines
def _oracle_c2(threads):
    """The oracle as it stands (threads=1) or on all cores (OpenMP over output
    elements, bit-identical) solving the C2 instance to tol."""
    import oracle
    import synth
    p = synth.nnls_gaussian(M_ROWS, N_COLS, SEED)
    oracle.set_threads(threads)
    try:
        t0 = time.perf_counter()
        r = oracle.minimize_lsq(oracle.LSQ(p.M, b=p.b), l=p.lower, m_hist=M_HIST,
                                opts=oracle.Options(tol=TOL))
        dt = time.perf_counter() - t0
    finally:
        oracle.set_threads(1)
    return r, dt


def cpu_baseline_c2():
    """C2 solved in full by the oracle: 1 thread ("as it stands") and all cores."""
    model, cores = _host_cpu()
    r1, dt1 = _oracle_c2(1)
    rN, dtN = _oracle_c2(cores)
    return {"value": r1.iters / dt1, "unit": "iters/s", "cores": 1, "kind": "oracle",
            "sample": f"full C2 solve to tol {TOL}: {r1.iters} iterations in {dt1:.2f} s "
                      f"(time-to-tol {dt1:.2f} s, f={r1.f:.12g}, pg={r1.pg_inf:.2e})",
            "time_to_tol_s": dt1, "iters": r1.iters, "f": r1.f, "cpu_model": model,
            "all_cores": {"value": rN.iters / dtN, "cores": cores, "time_to_tol_s": dtN,
                          "iters": rN.iters, "bit_identical_to_1_thread": bool(rN.f == r1.f and
                                                                              rN.iters == r1.iters),
                          "mode": "OpenMP over output elements of the two matvecs (same per-output order)"}}


def _c5_sample(ncols_s):
    """Columns [0, ncols_s) of C5 (device generator, copied to the host) and
    C5's b: the oracle's bounded sample of the C5 workload."""
    import numpy as np
    import torch
    import synth
    A = synth.c5_block(C5_M, 0, ncols_s, seed=C5_SEED).cpu().numpy()   # (m, s) column-major view
    b = synth.c5_rhs(C5_M, C5_N, seed=C5_SEED)
    torch.cuda.synchronize()
    return np.asfortranarray(A), b


def _oracle_c5_rate(A, b, threads, iters):
    """Seconds per Alg. 1 iteration of the oracle on the C5 column sample
    (setup + `iters` iterations + final refresh, divided by `iters`)."""
    import numpy as np
    import oracle
    oracle.set_threads(threads)
    try:
        t0 = time.perf_counter()
        r = oracle.minimize_lsq(oracle.LSQ(A, b=b), l=np.zeros(A.shape[1]), m_hist=M_HIST,
                                opts=oracle.Options(tol=TOL, max_iters=iters))
        dt = time.perf_counter() - t0
    finally:
        oracle.set_threads(1)
    return dt / max(r.iters, 1), r.iters


def cpu_baseline_c5(ncols_s=1000, iters=6):
    """C5 does not fit the host (160 GB): the oracle runs `iters` Alg. 1
    iterations on the first `ncols_s` columns of the same A (and the same b)
    and its per-iteration time is scaled by n / ncols_s (every iteration's
    cost is the two passes over A's columns)."""
    model, cores = _host_cpu()
    A, b = _c5_sample(ncols_s)
    s1, k1 = _oracle_c5_rate(A, b, 1, iters)
    sN, kN = _oracle_c5_rate(A, b, cores, iters)
    scale = C5_N / ncols_s
    sample = (f"oracle on C5 columns [0, {ncols_s}) x all {C5_M} rows with C5's b: setup + {k1} Alg. 1 "
              f"iterations + refresh in {s1 * k1:.2f} s; seconds per iteration x {scale:.0f} "
              f"(= n / sample columns) -> full-C5 iters/s")
    return {"value": 1.0 / (s1 * scale), "unit": "iters/s", "cores": 1, "kind": "oracle",
            "sample": sample, "cpu_model": model,
            "all_cores": {"value": 1.0 / (sN * scale), "cores": cores,
                          "mode": "OpenMP over output elements of the two matvecs (bit-identical)"}}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as the reference arm, on our arm's config, metric and unit.
    C2: the full C2 solve per step (same_config).  C5: per step, the bounded
    column sample of cpu_baseline_c5 (the full problem does not fit the host)."""
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    model, cores = _host_cpu()
    if args.config == "C2":
        tot, dt = 0, 0.0
        for k in range(args.warmup + args.steps):
            r, t = _oracle_c2(1)
            if k >= args.warmup:
                tot += r.iters
                dt += t
        v = tot / dt
        metric, sample = METRIC, f"full C2 solve (20000x10000, seed {SEED}) to tol {TOL} per step, 1 thread"
        cfg = {"workload": "C2 dense NNLS m=20000 n=10000 fp64 (CPU oracle, full solve)",
               "m": M_ROWS, "n": N_COLS, "m_hist": M_HIST, "tol": TOL}
        same = True
    else:
        A, b = _c5_sample(1000)
        per = []
        for k in range(args.warmup + args.steps):
            s1, _ = _oracle_c5_rate(A, b, 1, 4)
            if k >= args.warmup:
                per.append(s1)
        sec_per_it = sum(per) / len(per) * (C5_N / 1000)
        v = 1.0 / sec_per_it
        dt = sum(per) * 4
        metric = METRIC_C5
        sample = (f"per step: the oracle on C5 columns [0, 1000) x {C5_M} rows with C5's b, setup + 4 "
                  f"iterations + refresh, 1 thread; seconds per iteration x {C5_N // 1000} -> full-C5 iters/s")
        cfg = {"workload": "C5: column-sharded NNLS m=100000 n=200000 fp64 (CPU oracle, column sample)",
               "m": C5_M, "n_global": C5_N, "m_hist": M_HIST, "tol": TOL}
        same = False
    line = {"impl": "reference", "metric": metric, "value": v, "unit": "iters/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "strong" if args.config == "C5" else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
            "same_config": same,
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": 1, "kind": "oracle",
                             "sample": sample, "cpu_model": model},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def measure_c2(args, with_cpu=True):
    """BASELINE.json configs[1] on one GPU: returns its JSON line (dict)."""
    import numpy as np
    import torch
    import paper_2203_16340_b200 as lb
    import synth

    ws, rank, local = _dist()
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
    tfile = os.path.join(ROOT, "profiles", "r02b_kbwd_s_dram_bytes.json")
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
                "k_fwd_avg_launch_us": 1e3 * fwd_ms / max(fwd_n, 1),
                "read_probe_gbs": READ_PROBE_GBS, "frac_of_read_probe": (achieved / READ_PROBE_GBS) if achieved else None,
                "read_probe_source": READ_PROBE_SRC}
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

    cpu = None if (args.no_cpu_baseline or not with_cpu) else cpu_baseline_c2()
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
    for sv in (solver, solver_p, solver_h):
        sv.close()
    return line


def run_c5(args) -> int:
    """BASELINE.json configs[4] at N = WORLD_SIZE GPUs (strong scaling): C = 8
    fixed column chunks of the 100000 x 200000 NNLS, 8 / N logical ranks per
    process (paper_2203_16340_b200.sharded.ShardedGroup), one solve per step.
    value = iterations / max-over-ranks device time of the K steps."""
    import numpy as np
    import torch
    import paper_2203_16340_b200 as lb
    import synth
    from paper_2203_16340_b200 import sharded

    ws, rank, local = _dist()
    local = local % max(torch.cuda.device_count(), 1)      # (several ranks per GPU: smoke tests only)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    red_dev = dev
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.device_count() >= ws:
            dist.init_process_group("nccl", device_id=dev)
        else:                              # several ranks on one GPU (smoke tests): NCCL refuses that
            dist.init_process_group("gloo")
            red_dev = None
    m, n, C = C5_M, C5_N, C5_CHUNKS
    if args.c5_shape:                      # smoke tests of the N > 1 path on small boxes only
        m, n = (int(v) for v in args.c5_shape.split(","))
    stream = torch.cuda.Stream(device=dev)

    def mx(v):
        return sharded.max_over_ranks(v, device=red_dev) if ws > 1 else v

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- data: this process's chunks of A on the device, the replicated b
    t_gen = time.perf_counter()
    with torch.cuda.stream(stream):
        b_h = synth.c5_rhs(m, n, seed=C5_SEED)
        b = torch.from_numpy(b_h).to(dev)
        mine = sharded.local_chunks(C, ws, rank)
        ranges = [sharded.column_range(n, C, l) for l in range(C)]
        # one contiguous allocation for the local chunks (adjacent column ranges); each chunk
        # is a view starting at a multiple of 8 m bytes (16-byte aligned, like its own allocation)
        lc0, lc1 = ranges[mine[0]][0], ranges[mine[-1]][1]
        big = torch.empty((lc1 - lc0, m), dtype=torch.float64, device=dev)
        bufs = {l: big[ranges[l][0] - lc0:ranges[l][1] - lc0] for l in mine}
        for l in mine:
            synth.c5_block(m, ranges[l][0], ranges[l][1] - ranges[l][0], seed=C5_SEED, out=bufs[l], stream=stream)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t_gen

    def zeros_lo(l, c0, c1):
        return torch.zeros(c1 - c0, dtype=torch.float64, device=dev)

    xchg, err = args.xchg, ""

    def make_group(profile):
        nonlocal xchg, err
        opts = lb.Options(tol=TOL, profile=profile, max_iters=20000)
        g = None
        if xchg == "p2p":
            try:
                g = sharded.ShardedGroup(n, m, m_hist=M_HIST, nchunks=C, opts=opts, stream=stream,
                                         make_lower=zeros_lo, world=ws, rank=rank)
            except Exception as e:          # noqa: BLE001 -- collective decision below
                g, err = None, f"{type(e).__name__}: {e}"[:200]
            if ws > 1:
                oks = sharded.all_gather_bytes(b"1" if g is not None else (err.encode() or b"0"))
                if any(o != b"1" for o in oks):
                    if g is not None:
                        g.close()
                    g, xchg = None, "nccl"
                    err = "; ".join(o.decode() for o in oks if o != b"1")
            elif g is None:
                raise RuntimeError(err)
        if g is None:                                   # NCCL baseline: one handle per process
            c0, c1 = ranges[mine[0]][0], ranges[mine[-1]][1]
            g = sharded.make_sharded_solver(c1 - c0, n, M_HIST, zeros_lo(0, c0, c1), opts, stream, xchg="nccl")
        return g

    grp = make_group(False)
    grp_p = make_group(True)
    if xchg == "p2p":
        objs = [lb.LSQObjective(bufs[l].t(), b=b) for l in mine]
        xs = [torch.zeros(ranges[l][1] - ranges[l][0], dtype=torch.float64, device=dev) for l in mine]
        solve = lambda g: g.solve(objs, xs)                         # noqa: E731
        handles = lambda g: g.solvers                               # noqa: E731
    else:
        # the contiguous block of this process's chunks: one NCCL handle
        Mblk = big
        objs = [lb.LSQObjective(Mblk.t(), b=b)]
        xs = [torch.zeros(Mblk.shape[0], dtype=torch.float64, device=dev)]
        solve = lambda g: g.solve(objs[0], xs[0])                   # noqa: E731
        handles = lambda g: [g]                                     # noqa: E731

    def timed(g, k):
        barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its, rr = 0, None
        e0.record(stream)
        for _ in range(k):
            for x in xs:
                x.zero_()
            rr = solve(g)
            its += rr.iters
        e1.record(stream)
        barrier()
        return mx(e0.elapsed_time(e1)), its, rr

    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            for x in xs:
                x.zero_()
            solve(grp)
        for _ in range(1):
            for x in xs:
                x.zero_()
            solve(grp_p)
        for h in handles(grp):
            h.profile(reset=True)
        with ClockSampler(local) as clk:
            ms, iters, r = timed(grp, args.steps)
        launches = sum(h.profile(reset=True)["all_kernel_launches"][1] for h in handles(grp))
        handles(grp_p)[0].profile(reset=True)
        kp = max(1, min(args.steps, 3))
        ms_p, _, _ = timed(grp_p, kp)
        prof = handles(grp_p)[0].profile(reset=True)
    clocks = clk.summary()
    all_reasons = (sharded.all_gather_bytes(json.dumps(clocks.get("reasons", [])).encode())
                   if ws > 1 else [json.dumps(clocks.get("reasons", []))])
    # checksum of x* summed chunk by chunk in logical-chunk order (the same grouping at every N)
    csum = {l: float(x.sum()) for l, x in zip(mine, xs)} if xchg == "p2p" else {mine[0]: float(xs[0].sum())}
    if ws > 1:
        for blob in sharded.all_gather_bytes(json.dumps(csum).encode()):
            csum.update({int(k): v for k, v in json.loads(blob).items()})
    x_sum = 0.0
    for l in sorted(csum):
        x_sum += csum[l]

    # ---- e2e through the public API with host inputs: per step b and x0 from pinned host
    # memory, A regenerated on the device from the seed (the data set is the generator), the
    # group solve, x* back to pinned host memory; host wall clock, max over ranks
    b_pin = torch.from_numpy(b_h.copy()).pin_memory()
    x_pin = [torch.zeros(x.numel(), dtype=torch.float64).pin_memory() for x in xs]
    e2e_steps = max(1, min(args.steps, 3))

    def e2e_step():
        b.copy_(b_pin, non_blocking=True)
        for x, xp in zip(xs, x_pin):
            x.copy_(xp, non_blocking=True)              # x0 = 0 from the host
        for l in mine:
            synth.c5_block(m, ranges[l][0], ranges[l][1] - ranges[l][0], seed=C5_SEED, out=bufs[l],
                           stream=stream)
        rr = solve(grp)
        outs = [x.to("cpu", non_blocking=True) for x in xs]
        stream.synchronize()
        return rr.iters, outs

    with torch.cuda.stream(stream):
        barrier()
        t0 = time.perf_counter()
        e2e_iters = 0
        for _ in range(e2e_steps):
            its, _ = e2e_step()
            e2e_iters += its
        e2e_dt = mx(time.perf_counter() - t0)

    prof_summary = dict(prof)
    nloc = len(objs) if xchg == "p2p" else 1
    ncols_loc = sum(ranges[l][1] - ranges[l][0] for l in mine)
    barrier()
    for g in (grp, grp_p):
        g.close()
    del objs, xs, bufs, big, grp, grp_p
    torch.cuda.empty_cache()
    prof = prof_summary
    c2 = None
    cpu = None
    if ws == 1 and not args.no_c2:
        c2 = measure_c2(args)
        torch.cuda.empty_cache()
    if ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_c5()

    if rank == 0:
        peak, peak_src = _peaks()
        bwd_ms, bwd_n = prof["gemvT_epi (k_bwd)"]
        fwd_ms, fwd_n = prof["gemv_active (k_fwd)"]
        nact = prof.get("fwd_active_columns", (0, 0))[1]
        # per iteration the local k_bwd launches read the local A once: 8 m n_loc + per chunk
        # 8 m (r) + 9 x 8 n_chunk (epilogue vectors)
        bwd_bytes_it = 8 * m * ncols_loc + nloc * 8 * m + 9 * 8 * ncols_loc
        bwd_s = (bwd_ms / max(bwd_n, 1)) / 1e3
        achieved = bwd_bytes_it / bwd_s / 1e9 if bwd_n else None
        reasons = sorted({x for rs in all_reasons for x in json.loads(rs)})
        clocks["reasons"] = reasons
        if ws > 1:
            clocks["note"] = "sm_mhz sampled on rank 0's GPU; reasons merged over all ranks"
        roof = {"bound": "hbm", "unit": "GB/s", "achieved": achieved, "peak": peak,
                "frac": (achieved / peak) if achieved else None, "traffic": None,
                "peak_source": peak_src,
                "kernel": "k_bwd (generic persistent gemvT_epi: g = M^T r' + fused Alg. 1 epilogue, Gram, "
                          "Alg. 3 tail), rank 0",
                "bytes_per_launch": bwd_bytes_it / nloc, "launches_per_iteration": nloc,
                "avg_launch_us": 1e6 * bwd_s / nloc,
                "events": f"CUDA events around the {nloc} local k_bwd launches of every iteration of {kp} "
                          f"profiled steps ({ms_p / kp:.1f} ms per step with the event nodes)",
                "share_of_step": (bwd_ms / kp) / (ms_p / kp) if ms_p else None,
                "k_fwd_share_of_step": (fwd_ms / kp) / (ms_p / kp) if ms_p else None,
                "read_probe_gbs": READ_PROBE_GBS,
                "frac_of_read_probe": (achieved / READ_PROBE_GBS) if achieved else None,
                "read_probe_source": READ_PROBE_SRC}
        tfile = os.path.join(ROOT, "profiles", "r02b_c5_kbwd_dram_bytes.json")
        if os.path.exists(tfile):
            tr = json.load(open(tfile))
            roof["traffic"] = tr.get("dram_bytes_per_launch")
            roof["traffic_source"] = tr.get("source")
        if fwd_n and nact:
            cols = nact / fwd_n
            fb = 8 * m * cols + nloc * (8 * m * 4) + 8 * 3 * ncols_loc
            roof["k_fwd_active_cols_avg"] = cols
            roof["k_fwd_achieved_gbs"] = fb / (fwd_ms / fwd_n / 1e3) / 1e9
            v_bytes = 8 * ((4 * M_HIST + 16) * ncols_loc + 8 * m * nloc)
            it_bytes = 8 * m * (ncols_loc + cols) + v_bytes
            roof["iteration_bytes_avg_rank0"] = it_bytes
            roof["iteration_gbs_rank0"] = it_bytes / (ms / 1e3 / max(iters, 1)) / 1e9
        line = {"metric": METRIC_C5, "value": iters / (ms / 1e3), "unit": "iters/s", "n_gpus": ws,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (C5: A_ij = (u_ij - 1/2) sqrt(12/m), u from Philox4x32-10 on the device; "
                        "x_plant 10% |N(0,1)|, b = A x_plant + 0.1 z; SURVEY 8(d))",
                "config": {"workload": (f"C5: column-sharded NNLS m={m} n={n} fp64, x>=0, m_hist=5, "
                                        "tol 1e-6 (BASELINE.json configs[4]), strong scaling"
                                        + ("" if (m, n) == (C5_M, C5_N) else " -- SHRUNKEN SMOKE SHAPE, not a bench")),
                           "m": m, "n_global": n, "chunks": C, "chunks_per_gpu": len(mine), "m_hist": M_HIST,
                           "tol": TOL, "seed": C5_SEED, "A_bytes": 8 * m * n,
                           "l2": "inputs larger than L2 (A = 160 GB); no flush",
                           "parallelism": (f"column-sharded over {ws} GPU(s): {C} fixed chunks (logical ranks), "
                                           f"{len(mine)} per GPU, P2P mailboxes (NVLink stores fused in the "
                                           f"producing kernels), P-invariant" if xchg == "p2p" else
                                           f"column-sharded over {ws} GPU(s), one NCCL handle per GPU "
                                           f"(all-gather; not P-invariant)"),
                           "xchg": xchg, "xchg_fallback_reason": err or None, "p_invariant": xchg == "p2p"},
                "time_to_tol_ms": ms / args.steps, "iters_per_solve": r.iters, "f": r.f, "pg_inf": r.pg_inf,
                "status": r.status_name, "x_sum": x_sum, "gen_s": t_gen,
                "roofline": roof, "cpu_baseline": cpu,
                "e2e": {"value": e2e_iters / e2e_dt, "unit": "iters/s",
                        "h2d_bytes_per_step": 8 * (m + n), "d2h_bytes_per_step": 8 * n,
                        "steps": e2e_steps, "ms_per_step": 1e3 * e2e_dt / e2e_steps,
                        "api": "ShardedGroup.solve (lbfgsb_solve_group) per step: b and x0 H2D from pinned "
                               "host memory, every local A chunk regenerated on the device from the seed "
                               "(no host holds the 160 GB data set), x* D2H; host wall clock, max over ranks"},
                "gpu_launches": launches, "clocks": clocks,
                "paper_context": "paper: 0.8 s modified L-BFGS-B GPU / 4.9 s CPU L-BFGS-B on NNLS size 12000 "
                                 "(Quadro RTX 4000 / i9-10980XE, PAPER.md:449-451); different sizes/hardware"}
        if c2 is not None:
            line["c2"] = c2
        print(json.dumps(line), flush=True)
    barrier()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: C5 5, C2 30)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--xchg", choices=["p2p", "nccl"], default="p2p",
                    help="C5 exchange: P-invariant peer-memory group (default) or the NCCL all-gather "
                         "handle per process (not P-invariant; the baseline)")
    ap.add_argument("--config", choices=["C5", "C2"], default="C5",
                    help="C5 (default): BASELINE configs[4], strong scaling at every N; C2: configs[1], N=1")
    ap.add_argument("--no-c2", action="store_true", help="C5 at N=1 without the embedded C2 measurement")
    ap.add_argument("--c5-shape", default=None, help=argparse.SUPPRESS)   # "m,n": shrunken C5, smoke tests only
    args = ap.parse_args()
    if args.steps is None:
        args.steps = 5 if args.config == "C5" else 30
    if args.impl == "reference":
        return run_reference(args)
    ws, _, _ = _dist()
    if args.config == "C2":
        if ws > 1:
            raise SystemExit("--config C2 is the single-GPU configuration; use the default C5 for N > 1")
        print(json.dumps(measure_c2(args)), flush=True)
        return 0
    return run_c5(args)


if __name__ == "__main__":
    sys.exit(main())
