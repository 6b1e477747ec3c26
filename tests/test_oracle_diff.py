"""Pins of the oracle's difference-form Armijo test (reading R29, SURVEY 8(f)
N4): f(x + alpha p) - f(x) expanded exactly for the quadratic-plus-separable
objective with AL terms (Eq. (3)).

The expansion is pinned against the objective's DEFINITION evaluated in exact
rational arithmetic (fractions.Fraction: every float converts exactly), so a
dropped or mis-signed term of the expansion, a transposed operand or a wrong
(.)_+ branch fails; the solver-level pins check that the variant reaches the
paper's KKT tolerance where the plain f(x_t) <= f + c1 alpha g^T p test hits
its cancellation floor."""
from fractions import Fraction as F

import numpy as np
import pytest
import scipy.optimize


def _exact_delta(P, x, p, alpha):
    """f(x + alpha p) - f(x) with x + alpha p formed exactly."""
    xs = [F(float(a)) + F(float(alpha)) * F(float(b)) for a, b in zip(x, p)]
    return _exact_f_rat(P, xs) - _exact_f_rat(P, [F(float(a)) for a in x])


def _exact_f_rat(P, xs):
    """f of oracle.LSQ by its definition on exact rationals xs."""
    nv = P.nvars
    cs = [F(float(v)) for v in P.colscale] if P.colscale is not None else [F(1)] * P.ncols
    v = [xs[j] - xs[P.ncols + j] for j in range(P.ncols)] if P.split else list(xs)
    v = [cs[j] * v[j] for j in range(P.ncols)]
    M = [[F(float(P.M[i, j])) for j in range(P.ncols)] for i in range(P.m)]
    Mv = [sum(M[i][j] * v[j] for j in range(P.ncols)) for i in range(P.m)]
    if P.qp:
        quad = F(1, 2) * sum(v[i] * Mv[i] for i in range(P.m))
    else:
        b = [F(float(t)) for t in P.b] if P.b is not None else [F(0)] * P.m
        quad = F(1, 2) * sum((Mv[i] - b[i]) ** 2 for i in range(P.m))
    f = quad
    if P.c is not None:
        f += sum(F(float(P.c[j])) * xs[j] for j in range(nv))
    f += F(float(P.delta)) / 2 * sum(t * t for t in xs)
    rho = F(float(P.rho))
    for k in range(P.n_eq):
        h = sum(F(float(P.E[j, k])) * xs[j] for j in range(nv)) - F(float(P.e[k]))
        t = h + F(float(P.lam[k])) / rho
        f += rho / 2 * t * t
    for k in range(P.n_in):
        g = sum(F(float(P.G[j, k])) * xs[j] for j in range(nv)) - F(float(P.hv[k]))
        t = g + F(float(P.mu[k])) / rho
        if t > 0:
            f += rho / 2 * t * t
    return f


def _problem(orc, kind, rng):
    m, nc = 7, 5
    M = rng.standard_normal((m, nc))
    if kind == "lsq":
        P = orc.LSQ(M, b=rng.standard_normal(m))
    elif kind == "lsq_sep":
        P = orc.LSQ(M, b=rng.standard_normal(m), c=rng.standard_normal(nc), delta=0.3,
                    colscale=rng.uniform(0.5, 2.0, nc))
    elif kind == "split":
        P = orc.LSQ(M, b=rng.standard_normal(m), c=np.full(2 * nc, 0.2), split=True, delta=0.1)
    elif kind == "qp":
        A = rng.standard_normal((nc, nc))
        P = orc.LSQ(A @ A.T, c=rng.standard_normal(nc), qp=True, colscale=np.sign(rng.standard_normal(nc)),
                    delta=0.05)
    elif kind == "al":
        P = orc.LSQ(M, b=rng.standard_normal(m), c=rng.standard_normal(nc), delta=0.2,
                    E=rng.standard_normal((nc, 2)), e=rng.standard_normal(2),
                    G=rng.standard_normal((nc, 2)), hv=rng.standard_normal(2))
        P.lam[:] = rng.standard_normal(2)
        P.mu[:] = np.abs(rng.standard_normal(2))
        P.rho = 3.5
    else:
        raise ValueError(kind)
    return P


@pytest.mark.parametrize("kind", ["lsq", "lsq_sep", "split", "qp", "al"])
@pytest.mark.parametrize("alpha", [1.0, 0.37, 1.0 / 1024])
def test_delta_matches_exact_definition(orc, kind, alpha):
    seed = ["lsq", "lsq_sep", "split", "qp", "al"].index(kind) * 10 + int(alpha * 1024) % 7
    rng = np.random.default_rng(seed)
    P = _problem(orc, kind, rng)
    for trial in range(3):
        x = rng.standard_normal(P.nvars)
        p = rng.standard_normal(P.nvars)
        got = P.armijo_delta(x, p, alpha)
        want = _exact_delta(P, x, p, alpha)
        # scale of the terms that are summed in fp64
        scale = 1.0 + abs(float(_exact_f_rat(P, [F(float(v)) for v in x])))
        assert abs(got - float(want)) <= 1e-13 * scale, (kind, alpha, got, float(want))


def test_delta_inequality_branch_crossing(orc):
    """(.)_+ branches: t0 > 0 > t1, t0 < 0 < t1, both negative."""
    rng = np.random.default_rng(5)
    nc = 4
    M = rng.standard_normal((6, nc))
    Gc = np.zeros((nc, 1)); Gc[0, 0] = 1.0
    for x0, p0 in [(0.5, -1.0), (-0.5, 1.0), (-0.5, -1.0), (0.5, 1.0)]:
        P = orc.LSQ(M, b=rng.standard_normal(6), G=Gc, hv=[0.0])
        P.mu[:] = 0.0
        P.rho = 2.0
        x = rng.standard_normal(nc); x[0] = x0
        p = rng.standard_normal(nc); p[0] = p0
        got = P.armijo_delta(x, p, 1.0)
        want = float(_exact_delta(P, x, p, 1.0))
        assert got == pytest.approx(want, rel=1e-12, abs=1e-13), (x0, p0)


def test_delta_linear_term_is_gradient(orc):
    """d/dalpha of the expansion at 0 equals g^T p (orc_lsq_grad), the
    first-order term of the Armijo test: small alpha, Delta/alpha -> g^T p."""
    rng = np.random.default_rng(9)
    P = _problem(orc, "al", rng)
    x = rng.standard_normal(P.nvars); p = rng.standard_normal(P.nvars)
    g = P.grad(x)
    a = 1e-7
    assert P.armijo_delta(x, p, a) / a == pytest.approx(g @ p, rel=1e-5)


def test_diff_mode_same_iterates_at_loose_tol(orc):
    """In exact arithmetic the two Armijo forms take the same decisions; at a
    tolerance far above the cancellation floor the two runs agree."""
    rng = np.random.default_rng(2)
    A = rng.standard_normal((80, 40)); b = rng.standard_normal(80)
    P = orc.LSQ(A, b=b)
    r0 = orc.minimize_lsq(P, l=np.zeros(40), opts=orc.Options(tol=1e-5))
    r1 = orc.minimize_lsq(P, l=np.zeros(40), opts=orc.Options(tol=1e-5, armijo_diff=True))
    assert r0.status == r1.status == 0
    assert r0.iters == r1.iters
    assert np.allclose(r0.x, r1.x, atol=1e-9)
    assert r1.f == pytest.approx(r0.f, rel=1e-12)


def test_diff_mode_reaches_tight_tolerance_nnls(orc):
    """tol 1e-10 on an NNLS whose optimum scipy's active-set nnls gives
    exactly: the difference form converges (pg <= 1e-10) and matches."""
    rng = np.random.default_rng(3)
    A = rng.standard_normal((300, 150)) / np.sqrt(300); b = rng.standard_normal(300)
    xs, _ = scipy.optimize.nnls(A, b)
    P = orc.LSQ(A, b=b)
    r = orc.minimize_lsq(P, l=np.zeros(150), opts=orc.Options(tol=1e-10, armijo_diff=True,
                                                             max_iters=50000))
    assert r.status == 0, r.status
    assert r.pg_inf <= 1e-10
    assert np.allclose(r.x, xs, atol=1e-8)
