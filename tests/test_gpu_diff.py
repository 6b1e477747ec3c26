"""GPU parity of the difference-form Armijo test (reading R29)
against the oracle's own difference form (-m gpu), and the tolerances it makes
reachable: the plain test f(x_t) <= f + c1 a g^T p cannot resolve decreases
below ~eps|f| (hard part 4); the expansion can."""
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


def _cuda(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _gpu_solve(lb, prob, opts, m_hist=5):
    obj = lb.LSQObjective(lb.colmajor(prob.M), b=_cuda(prob.b), c=_cuda(prob.c), delta=prob.delta,
                          split=prob.split)
    s = lb.Solver(prob.nvars, m_hist, lower=_cuda(prob.lower), upper=_cuda(prob.upper), opts=opts)
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    return s.solve(obj, x), x.cpu().numpy()


def test_diff_nnls_parity(lb, orc):
    import synth
    prob = synth.nnls_gaussian(1500, 800, 93)
    r, x = _gpu_solve(lb, prob, lb.Options(armijo_diff=True, max_iters=20000))
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower,
                          opts=orc.Options(armijo_diff=True, max_iters=20000))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.pg_inf <= 1e-6 and abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    assert np.all(x >= 0)


def test_diff_nnls_tight_tolerance(lb):
    """tol 1e-10: converges and matches scipy's active-set NNLS optimum."""
    import synth
    from scipy.optimize import nnls
    prob = synth.nnls_gaussian(600, 300, 94)
    r, x = _gpu_solve(lb, prob, lb.Options(tol=1e-10, armijo_diff=True, max_iters=50000))
    xs, _ = nnls(prob.M, prob.b)
    assert r.status == lb.CONVERGED and r.pg_inf <= 1e-10
    assert np.allclose(x, xs, atol=1e-8)


def test_diff_lasso_split_parity(lb, orc):
    import synth
    prob = synth.lasso_split(400, 900, 95, alpha=0.7)
    r, x = _gpu_solve(lb, prob, lb.Options(armijo_diff=True, max_iters=50000))
    P = orc.LSQ(prob.M, b=prob.b, c=prob.c, delta=prob.delta, split=True)
    ro = orc.minimize_lsq(P, l=prob.lower, opts=orc.Options(armijo_diff=True, max_iters=50000))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)


def test_diff_box_qp_parity(lb, orc):
    rng = np.random.default_rng(4)
    n = 1200
    B = rng.standard_normal((n, n // 2)) / np.sqrt(n)
    Q = B @ B.T + 0.05 * np.eye(n)
    c = rng.standard_normal(n)
    obj = lb.QPObjective(lb.colmajor(Q), c=_cuda(c))
    s = lb.Solver(n, 5, lower=_cuda(np.zeros(n)), upper=_cuda(np.full(n, 2.0)),
                  opts=lb.Options(tol=1e-9, armijo_diff=True, max_iters=50000))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    ro = orc.minimize_lsq(orc.LSQ(Q, c=c, qp=True), l=np.zeros(n), u=np.full(n, 2.0),
                          opts=orc.Options(tol=1e-9, armijo_diff=True, max_iters=50000))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.pg_inf <= 1e-9 and abs(r.f - ro.f) <= 1e-10 * abs(ro.f)


def test_diff_kernel_svm_al_tight(lb, orc):
    """Alg. 4 on the Gaussian-kernel dual at tol = feas_tol = 1e-9: below the
    plain test's floor (test_gpu_qp uses 1e-6 for that reason)."""
    import synth
    prob = synth.svm_dual_kernel(600, 5, 7, gamma=1.0, C=1.0)
    Kd = lb.op_gaussian_kernel(_cuda(prob.meta["X"]), 1.0)
    obj = lb.QPObjective(Kd, c=_cuda(prob.c), colscale=_cuda(prob.colscale))
    s = lb.Solver(prob.nvars, 5, lower=_cuda(prob.lower), upper=_cuda(prob.upper),
                  opts=lb.Options(tol=1e-9, armijo_diff=True, max_iters=100000))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, E=_cuda(prob.E), e=prob.e, al_opts=lb.ALOptions(feas_tol=1e-9))
    P = orc.LSQ(prob.M, c=prob.c, colscale=prob.colscale, qp=True, E=prob.E, e=prob.e)
    ro = orc.al_solve(P, l=prob.lower, u=prob.upper,
                      opts=orc.Options(tol=1e-9, armijo_diff=True, max_iters=100000),
                      al_opts=orc.ALOptions(feas_tol=1e-9))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.violation_inf <= 1e-9
    assert abs(r.f - ro.f) <= 1e-9 * abs(ro.f)
    a = x.cpu().numpy()
    assert np.all(a >= 0) and np.all(a <= 1.0)


def test_diff_loopback_sharded(lb):
    """Sharded protocol (3 logical ranks, loopback) with the difference form:
    the r^T q, q^T q and separable sums travel in the same packs."""
    import synth
    from paper_2203_16340_b200.sharded import column_range
    prob = synth.lasso_split(300, 600, 96, alpha=0.5)
    r1, x1 = _gpu_solve(lb, prob, lb.Options(armijo_diff=True, max_iters=50000))
    sv, ob, xs, keep = [], [], [], []
    Pn = 3
    for k in range(Pn):
        c0, c1 = column_range(prob.ncols, Pn, k)
        vsl = np.r_[c0:c1, prob.ncols + c0:prob.ncols + c1]
        Mr = lb.colmajor(prob.M[:, c0:c1])
        o = lb.LSQObjective(Mr, b=_cuda(prob.b), c=_cuda(prob.c[vsl]), delta=prob.delta, split=True)
        s = lb.Solver(len(vsl), 5, lower=_cuda(prob.lower[vsl]),
                      opts=lb.Options(armijo_diff=True, max_iters=50000))
        sv.append(s); ob.append(o); xs.append(torch.zeros(len(vsl), dtype=torch.float64, device="cuda"))
        keep.append(Mr)
    r = lb.solve_loopback(sv, ob, xs)
    assert r.status == lb.CONVERGED and r1.status == lb.CONVERGED
    assert abs(r.f - r1.f) <= 1e-8 * abs(r1.f)
