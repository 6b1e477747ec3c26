"""Pins of the oracle's QP objective (f = 1/2 x^T D Q D x + c^T x,
the kernel dual SVM of PAPER.md:349-352) against closed forms, brute force
and a library solver."""
import itertools

import numpy as np
import pytest


def _spd(rng, n, cond=10.0):
    U, _ = np.linalg.qr(rng.standard_normal((n, n)))
    return U @ np.diag(np.linspace(1.0, cond, n)) @ U.T


def test_unconstrained_qp_closed_form(orc):
    rng = np.random.default_rng(1)
    n = 25
    Q = _spd(rng, n)
    c = rng.standard_normal(n)
    r = orc.minimize_lsq(orc.LSQ(Q, c=c, qp=True), opts=orc.Options(tol=1e-12))
    assert np.allclose(r.x, -np.linalg.solve(Q, c), atol=1e-9)
    assert r.f == pytest.approx(-0.5 * c @ np.linalg.solve(Q, c), rel=1e-12)


def _box_qp_bruteforce(Q, c, u):
    """min 1/2 x^T Q x + c^T x on [0, u]: enumerate (free / lower / upper) per variable."""
    n = len(c)
    best = None
    for st in itertools.product((0, 1, 2), repeat=n):
        x = np.zeros(n)
        up = [i for i in range(n) if st[i] == 2]
        fr = [i for i in range(n) if st[i] == 0]
        x[up] = u[up]
        if fr:
            rhs = -(c[fr] + Q[np.ix_(fr, up)] @ x[up])
            x[fr] = np.linalg.solve(Q[np.ix_(fr, fr)], rhs)
            if np.any(x[fr] < 0) or np.any(x[fr] > u[fr]):
                continue
        g = Q @ x + c
        ok = all((st[i] != 1 or g[i] >= -1e-10) and (st[i] != 2 or g[i] <= 1e-10) for i in range(n))
        if ok:
            f = 0.5 * x @ Q @ x + c @ x
            if best is None or f < best[1]:
                best = (x, f)
    return best


@pytest.mark.parametrize("seed", range(15))
def test_box_qp_bruteforce(orc, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(2, 7))
    Q = _spd(rng, n, cond=20.0)
    c = rng.standard_normal(n) * 2
    u = 0.2 + rng.random(n)
    x_bf, f_bf = _box_qp_bruteforce(Q, c, u)
    r = orc.minimize_lsq(orc.LSQ(Q, c=c, qp=True), l=np.zeros(n), u=u,
                         opts=orc.Options(tol=1e-11, max_iters=5000))
    assert r.status == orc.CONVERGED
    assert abs(r.f - f_bf) <= 1e-10 * max(1.0, abs(f_bf))
    assert np.allclose(r.x, x_bf, atol=1e-7)


def test_qp_equals_lsq_normal_equations(orc):
    """Q = M^T M, c = -M^T b: same minimiser as 1/2||Mx - b||^2, f offset 1/2||b||^2."""
    rng = np.random.default_rng(3)
    M = rng.standard_normal((60, 30)) / np.sqrt(60)
    b = rng.standard_normal(60)
    r1 = orc.minimize_lsq(orc.LSQ(M, b=b), l=np.zeros(30), opts=orc.Options(tol=1e-10))
    r2 = orc.minimize_lsq(orc.LSQ(M.T @ M, c=-(M.T @ b), qp=True), l=np.zeros(30),
                          opts=orc.Options(tol=1e-10))
    assert r2.f + 0.5 * b @ b == pytest.approx(r1.f, rel=1e-10)
    assert np.allclose(r1.x, r2.x, atol=1e-7)


def test_qp_colscale_is_DQD(orc):
    rng = np.random.default_rng(4)
    n = 12
    K = _spd(rng, n)
    y = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    c = -np.ones(n)
    r1 = orc.minimize_lsq(orc.LSQ(K, c=c, colscale=y, qp=True), l=np.zeros(n), u=np.ones(n),
                          opts=orc.Options(tol=1e-11))
    r2 = orc.minimize_lsq(orc.LSQ(np.diag(y) @ K @ np.diag(y), c=c, qp=True), l=np.zeros(n),
                          u=np.ones(n), opts=orc.Options(tol=1e-11))
    assert np.allclose(r1.x, r2.x, atol=1e-9) and r1.f == pytest.approx(r2.f, rel=1e-12)


def test_kernel_svm_dual_vs_scipy(orc):
    """Gaussian-kernel dual SVM (gamma = 1, c = 1) on 40 points,
    via Alg. 4, against scipy's SLSQP on the same QP."""
    from scipy.optimize import minimize
    import synth
    X, y = synth.blobs(40, 2, seed=5)
    K = synth.gaussian_kernel(X, 1.0)
    n = len(y)
    Q = (y[:, None] * K) * y[None, :]
    P = orc.LSQ(K, c=-np.ones(n), colscale=y, qp=True, E=y.reshape(n, 1), e=[0.0])
    # tol 1e-7: tighter inner tolerances hit the Armijo cancellation floor (|f| ~ 6)
    r = orc.al_solve(P, l=np.zeros(n), u=np.ones(n), opts=orc.Options(tol=1e-7),
                     al_opts=orc.ALOptions(feas_tol=1e-8))
    res = minimize(lambda a: 0.5 * a @ Q @ a - a.sum(), np.zeros(n), jac=lambda a: Q @ a - 1,
                   bounds=[(0, 1)] * n, constraints=[{"type": "eq", "fun": lambda a: y @ a,
                                                      "jac": lambda a: y}],
                   method="SLSQP", options={"ftol": 1e-14, "maxiter": 1000})
    assert r.status == orc.CONVERGED
    assert abs(y @ r.x) <= 1e-8
    assert abs(r.f - res.fun) <= 1e-6 * abs(res.fun)
