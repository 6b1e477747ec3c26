"""GPU tests of the host-buffer entry points (the bench's e2e path):
lbfgsb_solve_lsq_host (one problem: H2D of M, b, x0, solve, D2H of x*) and
lbfgsb_solve_lsq_host_batch (several problems, the H2D of problem k+1 on a
copy stream overlapping the solve of problem k, two device copies and two
captured graphs alternating).  Each result must equal, bit for bit, the
device-buffer lbfgsb_solve of the same problem (same kernels, same
reduction order), and agree with the oracle."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_16340_b200 as lb
    lb.load()
    return lb


def _device_solve(lb, p, tol=1e-6):
    lo = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
    s = lb.Solver(p.nvars, 5, lower=lo, opts=lb.Options(tol=tol))
    obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda())
    x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    return x.cpu().numpy(), r


def _host(p):
    M = np.asfortranarray(torch.from_numpy(np.ascontiguousarray(p.M.T)).pin_memory().numpy().T)
    b = torch.from_numpy(p.b.copy()).pin_memory().numpy()
    x = torch.zeros(p.nvars, dtype=torch.float64).pin_memory().numpy()
    return M, b, x


def test_solve_lsq_host_matches_device(lb, orc):
    import synth
    p = synth.nnls_gaussian(3000, 2000, 91)
    xd, rd = _device_solve(lb, p)
    M, b, x = _host(p)
    s = lb.Solver(p.nvars, 5, lower=torch.zeros(p.nvars, dtype=torch.float64, device="cuda"))
    r = s.solve_lsq_host(M, b, x)
    assert np.array_equal(x, xd) and r.f == rd.f and r.iters == rd.iters
    ro = orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower)
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)


@pytest.mark.parametrize("count", [1, 2, 5])
def test_solve_lsq_host_batch_matches_device(lb, count):
    import synth
    probs = [synth.nnls_gaussian(2500, 1500, 100 + k) for k in range(count)]
    ref = [_device_solve(lb, p) for p in probs]
    hs = [_host(p) for p in probs]
    s = lb.Solver(1500, 5, lower=torch.zeros(1500, dtype=torch.float64, device="cuda"))
    for rep in range(2):                                   # second call reuses buffers and graphs
        for h in hs:
            h[2][:] = 0.0
        rs = s.solve_lsq_host_batch([h[0] for h in hs], [h[1] for h in hs], [h[2] for h in hs])
        for (xd, rd), h, r in zip(ref, hs, rs):
            assert r.status == lb.CONVERGED
            assert np.array_equal(h[2], xd) and r.f == rd.f and r.iters == rd.iters


def test_solve_lsq_host_batch_shape_checks(lb):
    s = lb.Solver(10, 5)
    M = np.asfortranarray(np.zeros((4, 9)))
    x = np.zeros(9)
    with pytest.raises(lb.LbfgsbError):
        s.solve_lsq_host_batch([M], None, [x])
    assert s.solve_lsq_host_batch([], None, []) == []
