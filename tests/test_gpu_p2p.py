"""GPU tests of the P2P exchange of the column-sharded path (p2p.cu,
DESIGN.md section 8): the producing kernels store their packs into every
rank's mailbox and bump its counters; a wait kernel gates the rank-order
reduction.  The exchanged bytes and their order are those of the all-gather,
so every P2P solve must equal the copy-exchange loopback solve BITWISE.
  * loopback: P logical ranks on one device wired with
    lbfgsb_p2p_connect_local (NNLS; lasso split, whose separable sums ride
    in the q section and need the Armijo continuation path);
  * a 1-rank lbfgsb_create_sharded_p2p handle (graph and eager);
  * two PROCESSES (torch.distributed.run, gloo bootstrap) on the one GPU,
    mailboxes mapped with CUDA IPC: the real multi-process protocol.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_16340_b200 as lb
    lb.load()
    return lb


from test_gpu_sharded import _cuda, _gather_x, _shards  # noqa: E402


def _loopback(lb, prob, P, p2p):
    sv, ob, xs, keep = _shards(lb, prob, P)
    if p2p:
        lb.p2p_connect_local(sv, prob.M.shape[0])
    r = lb.solve_loopback(sv, ob, xs)
    return r, _gather_x(prob, P, xs), (sv, ob, xs, keep)


@pytest.mark.parametrize("P", [2, 3, 4])
def test_p2p_loopback_bitwise_equals_copy_exchange(lb, orc, P):
    import synth
    prob = synth.nnls_gaussian(3000, 2000, 77)
    r0, x0, _ = _loopback(lb, prob, P, False)
    r1, x1, _ = _loopback(lb, prob, P, True)
    assert r1.status == lb.CONVERGED and r1.pg_inf <= 1e-6
    assert np.array_equal(x0, x1) and r0.f == r1.f and r0.iters == r1.iters
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
    assert abs(r1.f - ro.f) <= 1e-8 * abs(ro.f)


def test_p2p_loopback_lasso_split(lb, orc):
    import synth
    prob = synth.lasso_split(500, 1200, 79, alpha=1.0)
    r0, x0, _ = _loopback(lb, prob, 2, False)
    r1, x1, _ = _loopback(lb, prob, 2, True)
    assert np.array_equal(x0, x1) and r0.f == r1.f and r0.n_backtracks == r1.n_backtracks
    P = orc.LSQ(prob.M, b=prob.b, c=prob.c, delta=prob.delta, split=True)
    ro = orc.minimize_lsq(P, l=prob.lower)
    assert r1.pg_inf <= 1e-6 and abs(r1.f - ro.f) <= 1e-8 * abs(ro.f)


def test_p2p_loopback_repeated_solves(lb):
    """Counters are monotonic across solves on the same wired handles."""
    import synth
    prob = synth.nnls_gaussian(1500, 900, 81)
    r0, x0, _ = _loopback(lb, prob, 3, False)
    sv, ob, xs, keep = _shards(lb, prob, 3)
    lb.p2p_connect_local(sv, 1500)
    for _ in range(3):
        for x in xs:
            x.zero_()
        r = lb.solve_loopback(sv, ob, xs)
        assert np.array_equal(_gather_x(prob, 3, xs), x0) and r.f == r0.f


def test_p2p_mailbox_too_small(lb):
    import synth
    prob = synth.nnls_gaussian(400, 300, 82)
    sv, ob, xs, keep = _shards(lb, prob, 2)
    lb.p2p_connect_local(sv, 399)
    with pytest.raises(lb.LbfgsbError):
        lb.solve_loopback(sv, ob, xs)


def test_p2p_one_rank_handle_graph_and_eager(lb, orc):
    import synth
    prob = synth.nnls_gaussian(2000, 1500, 80)
    lo = _cuda(prob.lower)
    obj = lb.LSQObjective(lb.colmajor(prob.M), b=_cuda(prob.b))
    out = []
    for graph in (True, False):
        s = lb.Solver(prob.nvars, 5, lower=lo, opts=lb.Options(use_graph=graph), rank=0, nranks=1,
                      n_global=prob.nvars, p2p_m_max=2000)
        s.p2p_open([s.ipc_handle()])
        x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
        r = s.solve(obj, x)
        out.append((x.cpu().numpy(), r))
    (xa, ra), (xb, rb) = out
    assert np.array_equal(xa, xb) and ra.f == rb.f
    s1 = lb.Solver(prob.nvars, 5, lower=lo, nccl_id=lb.nccl_unique_id(), rank=0, nranks=1,
                   n_global=prob.nvars)
    x1 = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r1 = s1.solve(obj, x1)
    assert np.array_equal(xa, x1.cpu().numpy()) and ra.f == r1.f     # == the NCCL exchange
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
    assert ra.status == lb.CONVERGED and abs(ra.f - ro.f) <= 1e-8 * abs(ro.f)


@pytest.mark.parametrize("graph", [1, 0])
def test_p2p_two_processes(lb, tmp_path, graph):
    """Two ranks in two processes (CUDA IPC mailboxes) == loopback P = 2, bitwise."""
    import synth
    m, n, seed = 2500, 1700, 83
    out = tmp_path / "p2p.npz"
    port = 29500 + (os.getpid() % 2000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "_p2p_worker.py"), str(out), str(m), str(n), str(seed), str(graph)]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    d = np.load(out)
    prob = synth.nnls_gaussian(m, n, seed)
    r0, x0, _ = _loopback(lb, prob, 2, False)
    assert int(d["status"]) == lb.CONVERGED
    assert np.array_equal(d["x"], x0) and float(d["f"]) == r0.f and int(d["iters"]) == r0.iters
