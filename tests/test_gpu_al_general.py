"""GPU parity of the general Alg. 4 (al_solve's general path: many linear
constraints on the GEMV kernels, nonlinear constraints through hg / jtv
callbacks, callback objectives, warm start -- PAPER.md:204-208, 212-220,
536-552) against the oracle's orc_al_general on the same seeded inputs
(-m gpu).

Tolerances: both sides stop at feasibility 1e-6 and inner KKT 1e-6; the
objective agrees to 1e-7 relative (a feasibility gap of 1e-6 moves f by
~|lambda| 1e-6 at most; on these instances |lambda| ~ 1e-1), x to 1e-4, and
the returned point satisfies the constraints and the box exactly / to 1e-6."""
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
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _affine(rng, n, k):
    E = rng.standard_normal((n, k)) / np.sqrt(n)
    return E


def _problem(seed, m=300, n=150):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    b = rng.standard_normal(m)
    return rng, A, b


@pytest.mark.parametrize("k", [16, 64])
def test_many_linear_equalities_vs_oracle(lb, orc, k):
    """NNLS objective, k >> 4 linear equalities (the general path: E^T x and E w
    on the GEMV kernels), x >= 0."""
    rng, A, b = _problem(100 + k)
    n = A.shape[1]
    E = _affine(rng, n, k)
    e = E.T @ np.abs(rng.standard_normal(n))                  # feasible with x >= 0
    ro = orc.al_general(n, base=orc.LSQ(A, b=b), E=E, e=e, l=0.0)
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"))
    obj = lb.LSQObjective(lb.colmajor(A), b=_cuda(b))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, E=_cuda(E), e=e)
    xg = x.cpu().numpy()
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert np.all(xg >= 0.0)
    assert np.max(np.abs(E.T @ xg - e)) <= 1e-6
    assert abs(r.f - ro.f) <= 1e-7 * abs(ro.f)
    assert np.max(np.abs(xg - ro.x)) <= 1e-4
    assert np.max(np.abs(np.array(r.lam) - ro.lam)) <= 1e-3 * max(1.0, np.max(np.abs(ro.lam)))


def test_many_linear_inequalities_vs_oracle(lb, orc):
    """32 linear inequalities G^T x <= hv (some active) and a two-sided box."""
    rng, A, b = _problem(7)
    n = A.shape[1]
    G = _affine(rng, n, 32)
    x_ref = orc.minimize_lsq(orc.LSQ(A, b=b), l=-0.5, u=0.5).x
    hv = G.T @ x_ref - 0.05 * np.abs(rng.standard_normal(32))     # the box optimum violates them
    ro = orc.al_general(n, base=orc.LSQ(A, b=b), G=G, hv=hv, l=-0.5, u=0.5)
    s = lb.Solver(n, 5, lower=torch.full((n,), -0.5, dtype=torch.float64, device="cuda"),
                  upper=torch.full((n,), 0.5, dtype=torch.float64, device="cuda"))
    obj = lb.LSQObjective(lb.colmajor(A), b=_cuda(b))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, G=_cuda(G), hv=hv)
    xg = x.cpu().numpy()
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert np.all(np.abs(xg) <= 0.5)
    assert np.max(G.T @ xg - hv) <= 1e-6
    assert abs(r.f - ro.f) <= 1e-7 * abs(ro.f)
    assert np.all(np.array(r.mu) >= 0.0)


def test_nonlinear_sphere_lsq_base(lb, orc):
    """min 1/2||x - c||^2 (LSQ: M = I, b = c) s.t. ||x||^2 = 1 through the
    nonlinear callbacks (torch on the device): x* = c/||c|| (closed form) and
    the oracle's orc_al_general with numpy callbacks."""
    rng = np.random.default_rng(3)
    n = 40
    c = 3.0 * rng.standard_normal(n) / np.sqrt(n)
    s = lb.Solver(n, 5)
    obj = lb.LSQObjective(lb.colmajor(np.eye(n)), b=_cuda(c))

    def hg(x, h, g):
        h[0] = torch.dot(x, x) - 1.0

    def jtv(x, ve, vi, out):
        out.copy_(2.0 * ve[0] * x)
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, hg=hg, jtv=jtv, m_nl=1)
    ro = orc.al_general(n, base=orc.LSQ(np.eye(n), b=c), m_nl=1,
                        hg=lambda x: (np.array([x @ x - 1.0]), np.zeros(0)), jtv=lambda x, ve, vi: 2.0 * ve[0] * x)
    xg = x.cpu().numpy()
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert np.max(np.abs(xg - c / np.linalg.norm(c))) <= 1e-5
    assert abs(r.f - ro.f) <= 1e-7 * abs(ro.f)
    assert abs(r.lam[0] - ro.lam[0]) <= 1e-4 * max(1.0, abs(ro.lam[0]))


def test_callback_objective_with_linear_and_nonlinear_constraints(lb, orc):
    """A callback objective (log-sum-exp + ridge, torch) with 8 linear
    equalities, one nonlinear inequality ||x||^2 <= R and a box: GPU general
    path vs the oracle with the numpy twin of the objective."""
    rng = np.random.default_rng(11)
    n, k = 30, 50
    A = rng.standard_normal((k, n))
    c = rng.standard_normal(n)
    E = _affine(rng, n, 8)
    x0 = 0.2 * rng.random(n)
    e = E.T @ x0
    R = 1.5 * float(x0 @ x0)
    At, ct = _cuda(A), _cuda(c)

    def fg_t(x, g):
        z = At @ x
        zm = z.max()
        w = torch.exp(z - zm)
        sw = w.sum()
        g.copy_(At.T @ (w / sw) + x + ct)
        return float(zm + torch.log(sw) + 0.5 * torch.dot(x, x) + torch.dot(ct, x))

    def fg_n(x):
        z = A @ x
        zm = z.max()
        w = np.exp(z - zm)
        return zm + np.log(w.sum()) + 0.5 * x @ x + c @ x, A.T @ (w / w.sum()) + x + c
    obj = lb.CallbackObjective(fg_t, n)
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")

    def hg(x, h, g):
        g[0] = torch.dot(x, x) - R

    def jtv(x, ve, vi, out):
        out.copy_(2.0 * vi[0] * x)
    r = s.al_solve(obj, x, E=_cuda(E), e=e, hg=hg, jtv=jtv, p_nl=1)
    ro = orc.al_general(n, fun=fg_n, E=E, e=e, p_nl=1, hg=lambda x: (np.zeros(0), np.array([x @ x - R])),
                        jtv=lambda x, ve, vi: 2.0 * vi[0] * x, l=0.0)
    xg = x.cpu().numpy()
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert np.all(xg >= 0.0) and xg @ xg <= R + 1e-6
    assert np.max(np.abs(E.T @ xg - e)) <= 1e-6
    assert abs(r.f - ro.f) <= 1e-7 * max(1.0, abs(ro.f))


def test_general_path_equals_fused_path_optimum(lb):
    """The linear SVM dual (one equality) through the fused path (LSQ objective,
    <= 4 constraints) and through the general path (the same objective as a
    callback) reach the same optimum."""
    import synth
    p = synth.svm_dual_linear(600, 10, 12)
    n = p.nvars
    M = lb.colmajor(p.M)
    y = _cuda(p.colscale)
    cvec = _cuda(p.c)
    lo = torch.zeros(n, dtype=torch.float64, device="cuda")
    up = _cuda(p.upper)
    s = lb.Solver(n, 5, lower=lo, upper=up)
    x1 = torch.zeros(n, dtype=torch.float64, device="cuda")
    r1 = s.al_solve(lb.LSQObjective(M, colscale=y, c=cvec), x1, E=y.reshape(-1, 1), e=np.zeros(1))
    Mt = _cuda(p.M)

    def fg(a, g):
        w = Mt @ (a * y)
        g.copy_(y * (Mt.T @ w) + cvec)
        return float(0.5 * torch.dot(w, w) + torch.dot(cvec, a))
    x2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    r2 = s.al_solve(lb.CallbackObjective(fg, n), x2, E=y.reshape(-1, 1), e=np.zeros(1))
    assert r1.status == r2.status == lb.CONVERGED
    assert abs(r1.f - r2.f) <= 1e-7 * abs(r1.f)


@pytest.mark.parametrize("general", [False, True])
def test_warm_start_reentry(lb, general):
    """Re-entering Alg. 4 with the converged x, multipliers and penalty stops
    after one outer iteration at the same point (SURVEY.md 5 checkpoint /
    resume), in the fused path (1 equality) and the general path (8)."""
    rng, A, b = _problem(21)
    n = A.shape[1]
    k = 8 if general else 1
    E = _affine(rng, n, k)
    e = E.T @ np.abs(rng.standard_normal(n))
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"))
    obj = lb.LSQObjective(lb.colmajor(A), b=_cuda(b))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r1 = s.al_solve(obj, x, E=_cuda(E), e=e)
    x1 = x.clone()
    r2 = s.al_solve(obj, x, E=_cuda(E), e=e, lam0=r1.lam, warm_start=True,
                    al_opts=lb.ALOptions(rho0=r1.rho))
    assert r1.status == r2.status == lb.CONVERGED
    assert r2.outer_iters == 1
    assert float(torch.max(torch.abs(x - x1))) <= 1e-6


def test_constraint_callback_error_is_reported(lb):
    n = 5
    s = lb.Solver(n, 5)
    obj = lb.LSQObjective(lb.colmajor(np.eye(n)), b=_cuda(np.ones(n)))

    def hg(x, h, g):
        raise ValueError("boom")
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    with pytest.raises(lb.LbfgsbError):
        s.al_solve(obj, x, hg=hg, jtv=lambda *a: None, m_nl=1)
