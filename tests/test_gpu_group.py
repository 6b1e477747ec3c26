"""Bitwise P-invariance of the column-sharded solve (
VERDICT r1 "Next" 3): C = 8 fixed column chunks are logical ranks
(lbfgsb_solve_group), hosted 8 / 4 / 2 / 1 per process by P = 1 / 2 / 4 / 8
processes (all on the test box's one GPU, mailboxes mapped with CUDA IPC).
x, f and the iteration count must be identical bit for bit at every P, and
the P = 1 solve must match the oracle's optimum.  The "c5" cases use the C5
generator (device Philox, centred uniform A) at 30000 rows, so the tall
generic backward GEMV and tall forward GEMV run (the C5 kernels)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WORKER = os.path.join(ROOT, "tests", "_group_worker.py")


def _run(tmp_path, P, m, n, seed, kind, graph=1, scale=1.0, max_bt=50, tol=1e-6, timeout=900):
    out = tmp_path / f"group_P{P}_{kind}_{graph}_{scale}_{max_bt}.npz"
    args = [str(out), str(m), str(n), str(seed), kind, "8", str(graph), repr(scale), str(max_bt), repr(tol)]
    if P == 1:
        cmd = [sys.executable, WORKER] + args
    else:
        port = 29600 + (os.getpid() * 7 + P) % 2000
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={P}",
               "--master-addr=127.0.0.1", f"--master-port={port}", WORKER] + args
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    d = np.load(out)
    return {k: d[k] for k in d.files}


@pytest.fixture(scope="module")
def cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _same(a, b):
    assert np.array_equal(a["x"], b["x"]), np.max(np.abs(a["x"] - b["x"]))
    assert float(a["f"]) == float(b["f"]) and int(a["iters"]) == int(b["iters"])
    assert int(a["status"]) == int(b["status"])


def test_group_p_invariant_gauss(cuda, tmp_path, orc):
    import synth
    m, n, seed = 3000, 1608, 91
    d1 = _run(tmp_path, 1, m, n, seed, "gauss")
    prob = synth.nnls_gaussian(m, n, seed)
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
    assert int(d1["status"]) == 0 and float(d1["pg"]) <= 1e-6
    assert abs(float(d1["f"]) - ro.f) <= 1e-8 * abs(ro.f)
    for P in (2, 4, 8):
        _same(_run(tmp_path, P, m, n, seed, "gauss"), d1)


def test_group_eager_equals_graph(cuda, tmp_path):
    a = _run(tmp_path, 1, 2000, 800, 92, "gauss", graph=1)
    b = _run(tmp_path, 1, 2000, 800, 92, "gauss", graph=0)
    _same(a, b)
    _same(_run(tmp_path, 2, 2000, 800, 92, "gauss", graph=0), a)


def test_group_p_invariant_c5_shape(cuda, tmp_path, orc):
    """C5 generator at 30000 x 2400 (tall columns: the generic k_bwd and the tall
    k_fwd), P = 1 vs 2 vs 8 bitwise; the optimum against the oracle on the same
    A regenerated on the host by the numpy Philox twin."""
    import synth
    from synth import philox
    m, n, seed = 30000, 2400, 5
    d1 = _run(tmp_path, 1, m, n, seed, "c5")
    assert int(d1["status"]) == 0 and float(d1["pg"]) <= 1e-6
    A = np.empty((m, n), order="F")
    for c0 in range(0, n, 300):                      # host twin of the device generator
        A[:, c0:c0 + 300] = philox.centered_block(np.arange(m), np.arange(c0, min(n, c0 + 300)), m, seed)
    _, b, _ = synth.c5_device(m, n, seed=seed, col0=0, ncols=1)
    ro = orc.minimize_lsq(orc.LSQ(A, b=b), l=np.zeros(n), opts=orc.Options(max_iters=5000))
    f0 = 0.5 * float(b @ b)
    assert ro.status == orc.CONVERGED
    assert abs(float(d1["f"]) - ro.f) <= 1e-8 * max(abs(ro.f), 1e-8 * f0)
    for P in (2, 8):
        _same(_run(tmp_path, P, m, n, seed, "c5"), d1)


def test_group_stall_paths_p_invariant(cuda, tmp_path):
    """A x1000-scaled problem (> 16 Armijo trials: the host-driven continuation)
    and max_backtracks = 0 (the R14 fallback relaunch, which converges): the stall
    paths run the P2P quiescence barrier (k_p2p_ack / k_p2p_wait_ack) and stay
    bitwise P-invariant across processes.  (tol = 1e-6 scale^2 for the x1000
    case: the gradient scales with scale^2.)"""
    a = _run(tmp_path, 1, 600, 240, 93, "gauss", scale=1000.0, tol=1.0)
    assert int(a["n_bt"]) > 16
    _same(_run(tmp_path, 2, 600, 240, 93, "gauss", scale=1000.0, tol=1.0), a)
    b = _run(tmp_path, 1, 600, 240, 94, "gauss", max_bt=0)     # one trial per search: R14 fallbacks
    assert int(b["n_fb"]) >= 1 and int(b["status"]) == 0
    _same(_run(tmp_path, 4, 600, 240, 94, "gauss", max_bt=0), b)
