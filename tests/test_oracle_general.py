"""Pins of the oracle's generic-objective Alg. 1 (orc_minimize_fg) and the
general Alg. 4 (orc_al_general: many linear constraints, nonlinear
constraints through value / J^T v callbacks, warm start) -- PAPER.md:204-208
(problem class), 210-222 (Eq. 3), 536-552 (Alg. 4) -- against closed forms,
scipy and KKT conditions (-m "not gpu")."""
import numpy as np
import pytest


def _kkt_box(grad, x, l, u, tol):
    """Projected-gradient KKT residual of a box problem."""
    pg = np.clip(x - grad, l, u) - x
    return np.max(np.abs(pg)) <= tol


@pytest.mark.parametrize("seed", range(4))
def test_minimize_fg_vs_scipy_lbfgsb(orc, seed):
    """A non-quadratic convex objective (log-sum-exp + ridge) on a box: the
    optimum agrees with scipy's Fortran L-BFGS-B (library) and satisfies KKT."""
    from scipy.optimize import minimize
    rng = np.random.default_rng(seed)
    n, k = 12, 30
    A = rng.standard_normal((k, n))
    c = rng.standard_normal(n)

    def fun(x):
        z = A @ x
        zm = z.max()
        w = np.exp(z - zm)
        f = zm + np.log(w.sum()) + 0.5 * x @ x + c @ x
        g = A.T @ (w / w.sum()) + x + c
        return f, g
    l, u = -0.3 * np.ones(n), 0.5 * np.ones(n)
    r = orc.minimize_fg(fun, n, l=l, u=u, opts=orc.Options(tol=1e-7))
    assert r.status == orc.CONVERGED
    ref = minimize(lambda x: fun(x)[0], np.zeros(n), jac=lambda x: fun(x)[1], method="L-BFGS-B",
                   bounds=list(zip(l, u)), options={"ftol": 1e-15, "gtol": 1e-12, "maxiter": 10000})
    assert abs(r.f - ref.fun) <= 1e-10 * max(1.0, abs(ref.fun))
    assert _kkt_box(fun(r.x)[1], r.x, l, u, 1e-7)


def test_minimize_fg_lsq_same_optimum(orc):
    """On the NNLS objective the generic path (evaluated trial values) and the
    LSQ path (carried residual, R13) reach the same optimum (Corollary,
    PAPER.md:198 -- unique optimal value of a convex problem)."""
    import synth
    p = synth.nnls_gaussian(120, 60, 3)
    P = orc.LSQ(p.M, b=p.b)
    r1 = orc.minimize_lsq(P, l=p.lower)
    r2 = orc.minimize_fg(lambda x: (P.value(x), P.grad(x)), 60, l=p.lower)
    assert r1.status == r2.status == orc.CONVERGED
    assert abs(r1.f - r2.f) <= 1e-10 * abs(r1.f)


@pytest.mark.parametrize("seed", range(5))
def test_al_sphere_projection(orc, seed):
    """min 1/2||x - c||^2 s.t. ||x||^2 = 1 (one NONLINEAR equality through the
    callbacks): x* = c / ||c|| (closed form), lambda* = (||c|| - 1)/2... from
    x - c + 2 lambda x = 0."""
    rng = np.random.default_rng(seed)
    n = 7
    c = rng.standard_normal(n) * (0.3 + 2 * seed)
    r = orc.al_general(n, fun=lambda x: (0.5 * np.sum((x - c) ** 2), x - c), m_nl=1,
                       hg=lambda x: (np.array([x @ x - 1.0]), np.zeros(0)),
                       jtv=lambda x, ve, vi: 2.0 * x * ve[0],
                       opts=orc.Options(tol=1e-7, max_iters=3000), al_opts=orc.ALOptions(feas_tol=1e-8))
    nc = np.linalg.norm(c)
    assert r.status == orc.CONVERGED
    assert np.max(np.abs(r.x - c / nc)) <= 1e-5
    assert abs(r.lam[0] - (nc - 1.0) / 2.0) <= 1e-4 * max(1.0, nc)


@pytest.mark.parametrize("scale", [0.4, 3.0])
def test_al_ball_projection(orc, scale):
    """min 1/2||x - c||^2 s.t. ||x||^2 <= 1 (one nonlinear inequality):
    x* = c / max(1, ||c||); mu* = 0 when c is inside."""
    rng = np.random.default_rng(1)
    n = 9
    c = rng.standard_normal(n)
    c = scale * c / np.linalg.norm(c)
    r = orc.al_general(n, fun=lambda x: (0.5 * np.sum((x - c) ** 2), x - c), p_nl=1,
                       hg=lambda x: (np.zeros(0), np.array([x @ x - 1.0])),
                       jtv=lambda x, ve, vi: 2.0 * x * vi[0],
                       opts=orc.Options(tol=1e-7, max_iters=3000), al_opts=orc.ALOptions(feas_tol=1e-8))
    assert r.status == orc.CONVERGED
    assert np.max(np.abs(r.x - c / max(1.0, scale))) <= 1e-5
    assert r.mu[0] >= 0.0
    if scale < 1:
        assert r.mu[0] == 0.0


def _affine(rng, n, k):
    E = rng.standard_normal((n, k)) / np.sqrt(n)
    e = 0.1 * rng.standard_normal(k)
    b = rng.standard_normal(n)
    return E, e, b


@pytest.mark.parametrize("k", [8, 64])
def test_al_many_linear_equalities_closed_form(orc, k):
    """min 1/2||x - b||^2 s.t. E^T x = e with k LINEAR equalities, no box:
    x* = b - E (E^T E)^{-1} (E^T b - e), lambda* = (E^T E)^{-1}(E^T b - e)."""
    rng = np.random.default_rng(k)
    n = 200
    E, e, b = _affine(rng, n, k)
    P = orc.LSQ(np.eye(n), b=b)
    r = orc.al_general(n, base=P, E=E, e=e, opts=orc.Options(max_iters=3000))
    lam = np.linalg.solve(E.T @ E, E.T @ b - e)
    assert r.status == orc.CONVERGED
    assert np.max(np.abs(r.x - (b - E @ lam))) <= 1e-5
    assert np.max(np.abs(r.lam - lam)) <= 1e-4 * max(1.0, np.max(np.abs(lam)))


def test_al_linear_equalities_box_kkt(orc):
    """NNLS-type objective, 64 equalities and x >= 0: the KKT conditions of
    the constrained problem hold with the returned multipliers (stationarity
    of f + lam^T h on the box, feasibility), and the optimum equals the one
    the LSQ-family AL path (orc_al_solve, carried residual) reaches."""
    rng = np.random.default_rng(5)
    n, k = 150, 64
    E, e, b = _affine(rng, n, k)
    A = rng.standard_normal((300, n)) / np.sqrt(300)
    P = orc.LSQ(A, b=rng.standard_normal(300))
    e = E.T @ np.abs(rng.standard_normal(n))              # feasible with x >= 0
    r = orc.al_general(n, base=P, E=E, e=e, l=0.0, opts=orc.Options(max_iters=3000))
    assert r.status == orc.CONVERGED
    grad = P.grad(r.x) + E @ r.lam
    assert _kkt_box(grad, r.x, 0.0, np.inf, 1e-5)
    assert np.max(np.abs(E.T @ r.x - e)) <= 1e-6
    P2 = orc.LSQ(A, b=P.b, E=E, e=e)
    r2 = orc.al_solve(P2, l=0.0, opts=orc.Options(max_iters=3000))
    assert abs(r.f - r2.f) <= 1e-8 * abs(r2.f)


def test_al_linear_through_callbacks_equals_linear_block(orc):
    """The same 16 affine equalities given as E (linear block) or through the
    nonlinear callbacks (h = E^T x - e, J^T v = E v) give the same optimum."""
    rng = np.random.default_rng(9)
    n, k = 80, 16
    E, e, b = _affine(rng, n, k)
    P = orc.LSQ(np.eye(n), b=b)
    r1 = orc.al_general(n, base=P, E=E, e=e, l=-0.2)
    r2 = orc.al_general(n, base=P, m_nl=k, hg=lambda x: (E.T @ x - e, np.zeros(0)),
                        jtv=lambda x, ve, vi: E @ ve, l=-0.2)
    assert r1.status == r2.status == orc.CONVERGED
    assert abs(r1.f - r2.f) <= 1e-8 * abs(r1.f)
    assert np.max(np.abs(r1.x - r2.x)) <= 1e-5


def test_al_general_warm_start_reentry(orc):
    """Re-entering with the multipliers and x of a converged run stops after
    one outer iteration at the same point (checkpoint/resume)."""
    rng = np.random.default_rng(2)
    n = 10
    c = rng.standard_normal(n) * 3
    kw = dict(fun=lambda x: (0.5 * np.sum((x - c) ** 2), x - c), m_nl=1,
              hg=lambda x: (np.array([x @ x - 1.0]), np.zeros(0)), jtv=lambda x, ve, vi: 2.0 * x * ve[0],
              opts=orc.Options(max_iters=3000))
    r1 = orc.al_general(n, **kw)
    r2 = orc.al_general(n, x0=r1.x, lam0=r1.lam, al_opts=orc.ALOptions(rho0=r1.rho), **kw)
    assert r2.status == orc.CONVERGED and r2.outer_iters == 1
    assert np.max(np.abs(r2.x - r1.x)) <= 1e-6


def test_al_general_callback_failure_is_reported(orc):
    def bad(x):
        raise ValueError("boom")
    with pytest.raises(RuntimeError):
        orc.al_general(3, fun=bad)
