"""Pins of the oracle's joint-probability / regularised-OT objective (SURVEY
8(f) N2):  min <M, P> + lam r(P)  s.t.  P 1 = u, P^T 1 = v,
P >= 0, solved with Alg. 4 around Alg. 1.

Pins (none re-types the oracle's own arithmetic):
  * entropy r = sum P log P: the exact solution is the Sinkhorn scaling
    P* = diag(a) exp(-M/lam) diag(b) (stationarity M + lam(log P + 1) +
    alpha_i + beta_j = 0 with P > 0), computed here by Sinkhorn's iteration;
  * Gaussian r = 1/2 ||P||^2: brute force over the faces {P_ij = 0, ij in Z}
    (equality-constrained QP per face by its KKT system), and the smooth
    Lagrange dual maximised with scipy BFGS;
  * the gradient against central finite differences of the value (pins the
    row / column broadcast of the marginal multipliers);
  * the difference-form Armijo expansion with the entropy term (R29 + R30)
    against a direct evaluation of f(x_t) - f(x), including trial points
    clipped to the lower bound."""
import itertools

import numpy as np
import pytest
import scipy.optimize

import synth

LENT = 1e-300   # entropy lower bound (reading R30)


def _sinkhorn(M, u, v, lam, iters=20000):
    K = np.exp(-M / lam)
    a = np.ones(len(u)); b = np.ones(len(v))
    for _ in range(iters):
        a = u / (K @ b)
        b = v / (K.T @ a)
    return a[:, None] * K * b[None, :]


def _al(orc, P, l, tol=1e-10):
    return orc.al_solve(P, l=l, opts=orc.Options(tol=tol, armijo_diff=True, max_iters=200000),
                        al_opts=orc.ALOptions(feas_tol=tol))


@pytest.mark.parametrize("case", ["ds2_8", "ds2_15", "ds1_12", "rect"])
def test_entropy_matches_sinkhorn(orc, case):
    if case.startswith("ds2"):
        t = synth.transport_ds2(int(case.split("_")[1]), 3)
        M, u, v, lam = t.cost, t.u, t.v, t.lam
    elif case == "ds1_12":
        t = synth.transport_ds1(12)
        M, u, v, lam = t.cost, t.u, t.v, t.lam
    else:
        rng = np.random.default_rng(4)
        M = rng.uniform(size=(5, 9)) * 3.0
        u = rng.uniform(size=5); u /= u.sum(); v = rng.uniform(size=9); v /= v.sum()
        lam = 0.7
    m, n = M.shape
    Ps = _sinkhorn(M, u, v, lam)
    P = orc.LSQ.transport(M, u, v, "entropy", lam)
    r = _al(orc, P, np.full(m * n, LENT))
    assert r.status == orc.CONVERGED
    X = r.x.reshape(m, n, order="F")
    assert np.max(np.abs(X - Ps)) <= 1e-8 * Ps.max()
    fstar = np.sum(M * Ps) + lam * np.sum(Ps * np.log(Ps))
    assert r.f == pytest.approx(fstar, rel=1e-9)
    assert r.violation_inf <= 1e-10


def _gauss_faces(M, u, v, lam):
    """min <M,P> + lam/2 ||P||^2, marginals, P >= 0, by enumerating the zero set."""
    m, n = M.shape
    N = m * n
    A = np.zeros((m + n, N))
    for j in range(n):
        for i in range(m):
            A[i, i + j * m] = 1.0
            A[m + j, i + j * m] = 1.0
    bvec = np.r_[u, v]
    c = M.reshape(-1, order="F")
    best = None
    for Z in itertools.product((0, 1), repeat=N):
        free = np.array([z == 0 for z in Z])
        if not free.any():
            continue
        Af = A[:, free]
        # KKT: lam x_f + c_f + Af^T nu = 0, Af x_f = b
        nf = int(free.sum())
        K = np.block([[lam * np.eye(nf), Af.T], [Af, np.zeros((m + n, m + n))]])
        rhs = np.r_[-c[free], bvec]
        sol, *_ = np.linalg.lstsq(K, rhs, rcond=None)
        x = np.zeros(N); x[free] = sol[:nf]
        if np.min(x) < -1e-12 or np.max(np.abs(A @ x - bvec)) > 1e-10:
            continue
        f = c @ x + 0.5 * lam * x @ x
        if best is None or f < best[0]:
            best = (f, x)
    return best


@pytest.mark.parametrize("shape,seed", [((2, 3), 1), ((3, 3), 2), ((2, 4), 3)])
def test_gaussian_bruteforce(orc, shape, seed):
    rng = np.random.default_rng(seed)
    m, n = shape
    M = rng.uniform(size=(m, n))
    u = rng.uniform(size=m); u /= u.sum(); v = rng.uniform(size=n); v /= v.sum()
    lam = 0.5
    fb, xb = _gauss_faces(M, u, v, lam)
    P = orc.LSQ.transport(M, u, v, "gaussian", lam)
    r = _al(orc, P, np.zeros(m * n))
    assert r.status == orc.CONVERGED
    assert np.allclose(r.x, xb, atol=1e-8)
    assert r.f == pytest.approx(fb, rel=1e-9, abs=1e-12)


@pytest.mark.parametrize("n", [6, 10])
def test_gaussian_vs_dual_ds2(orc, n):
    """Larger than brute force: the Lagrange dual of the Gaussian case,
    max -a.u - b.v - 1/(2 lam) sum (-(M_ij + a_i + b_j))_+^2, is smooth and
    unconstrained; P_ij = (-(M_ij + a_i + b_j))_+ / lam at its maximiser
    (scipy BFGS, then semismooth Newton steps on the support)."""
    t = synth.transport_ds2(n, 7)
    m, lam = t.m, t.lam
    M = t.cost

    def negdual(z):
        a, b = z[:m], z[m:]
        Z = np.maximum(-(M + a[:, None] + b[None, :]), 0.0)
        P = Z / lam
        val = a @ t.u + b @ t.v + 0.5 / lam * np.sum(Z * Z)
        grad = np.r_[t.u - P.sum(1), t.v - P.sum(0)]
        return val, grad

    z = np.zeros(m + n)
    for _ in range(5):
        res = scipy.optimize.minimize(negdual, z, jac=True, method="BFGS",
                                      options={"gtol": 1e-14, "maxiter": 20000})
        z = res.x
    for _ in range(8):                   # semismooth Newton polish on the support
        a, b = z[:m], z[m:]
        S = (M + a[:, None] + b[None, :] < 0).astype(float)
        _, g = negdual(z)
        J = np.block([[np.diag(S.sum(1)), S], [S.T, np.diag(S.sum(0))]]) / lam
        z = z - np.linalg.lstsq(J, g, rcond=None)[0]
    a, b = z[:m], z[m:]
    Pd = np.maximum(-(M + a[:, None] + b[None, :]), 0.0) / lam
    assert np.max(np.abs(np.r_[Pd.sum(1) - t.u, Pd.sum(0) - t.v])) <= 1e-11
    P = orc.LSQ.transport(t.cost, t.u, t.v, "gaussian", lam)
    r = _al(orc, P, np.zeros(m * n))
    assert r.status == orc.CONVERGED
    assert np.allclose(r.x.reshape(m, n, order="F"), Pd, atol=1e-8)


@pytest.mark.parametrize("reg", ["entropy", "gaussian"])
def test_gradient_finite_differences(orc, reg):
    rng = np.random.default_rng(11)
    m, n = 4, 6
    M = rng.uniform(size=(m, n))
    u = rng.uniform(size=m); u /= u.sum(); v = rng.uniform(size=n); v /= v.sum()
    P = orc.LSQ.transport(M, u, v, reg, 0.5)
    P.lam[:] = rng.standard_normal(m + n)
    P.rho = 2.5
    x = rng.uniform(0.05, 0.2, m * n)
    g = P.grad(x)
    h = 1e-6
    for j in range(m * n):
        e = np.zeros(m * n); e[j] = h
        fd = (P.value(x + e) - P.value(x - e)) / (2 * h)
        assert g[j] == pytest.approx(fd, rel=1e-6, abs=1e-7), j


def _f_direct(M, u, v, lam, reg, lmul, rho, x):
    m, n = M.shape
    X = x.reshape(m, n, order="F")
    if reg == "entropy":
        r = np.sum(np.where(X > 0, X * np.log(np.where(X > 0, X, 1.0)), 0.0))
    else:
        r = 0.5 * np.sum(X * X)
    h = np.r_[X.sum(1) - u, X.sum(0) - v]
    return np.sum(M * X) + lam * r + 0.5 * rho * np.sum((h + lmul / rho) ** 2)


@pytest.mark.parametrize("reg", ["entropy", "gaussian"])
@pytest.mark.parametrize("alpha", [1.0, 0.3, 1e-3])
def test_delta_entropy_direct(orc, reg, alpha):
    rng = np.random.default_rng(12)
    m, n = 5, 4
    M = rng.uniform(size=(m, n))
    u = rng.uniform(size=m); u /= u.sum(); v = rng.uniform(size=n); v /= v.sum()
    P = orc.LSQ.transport(M, u, v, reg, 0.5)
    P.lam[:] = 0.1 * rng.standard_normal(m + n)
    P.rho = 3.0
    lo = LENT if reg == "entropy" else 0.0
    x = rng.uniform(0.01, 0.1, m * n)
    p = rng.standard_normal(m * n) * 0.05
    p[:3] = -1.0                     # these elements clip to the lower bound
    got = P.armijo_delta(x, p, alpha, l=np.full(m * n, lo))
    xt = np.maximum(x + alpha * p, lo)
    # the expansion treats the smooth terms on x + alpha p and the entropy on
    # the clipped point: build the same reference from the definition
    f0 = _f_direct(M, u, v, 0.5, reg, P.lam, P.rho, x)
    if reg == "entropy":
        fl = _f_direct(M, u, v, 0.0, reg, P.lam, P.rho, x + alpha * p)
        fl0 = _f_direct(M, u, v, 0.0, reg, P.lam, P.rho, x)
        ent = lambda z: np.sum(z * np.log(z))
        want = (fl - fl0) + 0.5 * (ent(xt) - ent(x))
    else:
        want = _f_direct(M, u, v, 0.5, reg, P.lam, P.rho, x + alpha * p) - f0
    assert got == pytest.approx(want, rel=1e-10, abs=1e-13)
