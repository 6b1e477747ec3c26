"""Pins of the CPU oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a worked example
(tests/golden/spec_examples.json, with citations), a closed form, a library
routine (scipy / numpy.linalg), brute force on tiny inputs, or an invariant
of the paper (Theorem 1, Corollary).
"""
import itertools
import json
import os

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _bnd(v):
    if v is None:
        return None
    a = np.array([np.nan if t is None else t for t in v], dtype=float)
    return None if np.all(np.isnan(a)) else a


# ---------------------------------------------------------------- examples
def test_clip_examples(orc):
    for ex in GOLD["clip"]:
        out = orc.clip(ex["x"], _bnd(ex["l"]), _bnd(ex["u"]))
        assert np.array_equal(out, np.array(ex["out"], float)), ex["cite"]


def test_clip_idempotent(orc):
    rng = np.random.default_rng(0)
    x = rng.standard_normal(1000) * 3
    l = rng.standard_normal(1000) - 1
    u = l + rng.random(1000) * 2
    c1 = orc.clip(x, l, u)
    assert np.array_equal(orc.clip(c1, l, u), c1)
    assert np.array_equal(c1, np.minimum(np.maximum(x, l), u))   # numpy's clip


def test_masked_dot_examples(orc):
    for ex in GOLD["masked_dot"]:
        assert orc.masked_dot(ex["u"], ex["v"], ex["free"]) == ex["out"], ex["cite"]
    rng = np.random.default_rng(1)
    u, v = rng.standard_normal(64), rng.standard_normal(64)
    s = rng.random(64) < 0.5
    assert orc.masked_dot(u, v, s) == pytest.approx(float(np.dot(u[s], v[s])), rel=1e-14)
    # full mask equals the plain dot with the same (sequential) order
    assert orc.masked_dot(u, v, np.ones(64, bool)) == orc.masked_dot(u, v, None)


def test_matvec_examples(orc):
    for ex in GOLD["matvec"]:
        A = np.array(ex["A"], float)
        if "out" in ex:
            assert np.array_equal(orc.matvec(A, ex["x"]), np.array(ex["out"], float)), ex["cite"]
        if "out_t" in ex:
            assert np.array_equal(orc.matvec_t(A, ex["x"]), np.array(ex["out_t"], float)), ex["cite"]


def test_matvec_unit_vectors_and_blas(orc):
    rng = np.random.default_rng(2)
    A = np.asfortranarray(rng.standard_normal((37, 23)))
    for i in range(23):
        e = np.zeros(23); e[i] = 1.0
        assert np.array_equal(orc.matvec(A, e), A[:, i])          # A e_i = column i exactly
    x, r = rng.standard_normal(23), rng.standard_normal(37)
    assert np.allclose(orc.matvec(A, x), A @ x, rtol=0, atol=1e-13)     # BLAS
    assert np.allclose(orc.matvec_t(A, r), A.T @ r, rtol=0, atol=1e-13)


def test_working_set_examples(orc):
    for ex in GOLD["working_set"]:
        fr = orc.working_set(ex["x"], ex["g"], ex["l"], ex["u"], ex["eps"])
        assert list(fr.astype(int)) == ex["free"], ex["cite"]


def test_working_set_unbounded_and_degenerate(orc):
    rng = np.random.default_rng(3)
    x, g = rng.standard_normal(50), rng.standard_normal(50)
    assert orc.working_set(x, g, None, None, 1e-9).all()          # nothing can be eps-active
    # l == u: every coordinate is fixed whatever the gradient sign (R17)
    l = rng.standard_normal(50)
    assert not orc.working_set(l, g, l, l, 1e-9).any()
    # gradient exactly 0 at a bound counts as fixed (Eq. 1 uses >= / <=)
    assert not orc.working_set([0.0], [0.0], [0.0], None, 1e-9)[0]


def test_check_convergence_examples(orc):
    for ex in GOLD["check_convergence"]:
        assert orc.check_convergence(ex["g"], ex["free"], ex["tol"]) == ex["out"], ex["cite"]


# ---------------------------------------------------------------- Alg. 3
def test_two_loop_examples(orc):
    for ex in GOLD["two_loop"]:
        d = orc.two_loop(ex["g"], ex["free"], ex["S"], ex["Y"])
        assert np.allclose(d, ex["d"], rtol=0, atol=1e-15), ex["cite"]


def _dense_inverse_bfgs(S, Y, free, gamma):
    """Closed form of the L-BFGS inverse Hessian on the free set:
    H0 = gamma I, H <- (I - rho s y^T) H (I - rho y s^T) + rho s s^T (Nocedal & Wright 7.19)."""
    idx = np.flatnonzero(free)
    k = len(idx)
    H = gamma * np.eye(k)
    for s, y in zip(S, Y):
        s, y = s[idx], y[idx]
        rho = 1.0 / (s @ y)
        V = np.eye(k) - rho * np.outer(y, s)
        H = V.T @ H @ V + rho * np.outer(s, s)
    return idx, H


@pytest.mark.parametrize("seed", range(120))
def test_two_loop_equals_dense_inverse_bfgs(orc, seed):
    """Alg. 3 with every pair passing the screen equals the explicit
    inverse-BFGS matrix recursion restricted to S."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 9)); nh = int(rng.integers(1, 5))
    free = rng.random(n) < 0.75
    free[0] = True
    B = rng.standard_normal((n, n)); Q = B @ B.T + n * np.eye(n)     # SPD => y = Q s
    # s supported on S, so <s[S], y[S]> = s^T Q s > 0 and every pair passes the screen
    S = [np.where(free, rng.standard_normal(n), 0.0) for _ in range(nh)]
    Y = [Q @ s for s in S]
    g = rng.standard_normal(n)
    for screen_full in (False, True):
        d = orc.two_loop(g, free, S, Y, eps=1e-12, screen_full_norm=screen_full)
        sN, yN = S[-1][free], Y[-1][free]
        nuN = (Y[-1] @ Y[-1]) if screen_full else (yN @ yN)
        idx, H = _dense_inverse_bfgs(S, Y, free, (sN @ yN) / nuN)
        ref = -(H @ g[idx])
        assert np.allclose(d[idx], ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max())
        assert np.all(d[~free] == 0.0)                                # d[S-bar] = 0


@pytest.mark.parametrize("seed", range(30))
def test_two_loop_secant_equation(orc, seed):
    """H_k y_{k-1} = s_{k-1} on S when every pair passes (quasi-Newton secant condition):
    feeding g := y_{k-1} must return d = -s_{k-1}."""
    rng = np.random.default_rng(100 + seed)
    n = 12; nh = 4
    free = np.ones(n, bool); free[rng.integers(0, n, 3)] = False
    B = rng.standard_normal((n, n)); Q = B @ B.T + np.eye(n)
    S = [np.where(free, rng.standard_normal(n), 0.0) for _ in range(nh)]
    Y = [Q @ s for s in S]
    Sm = [np.where(free, s, 0) for s in S]; Ym = [np.where(free, y, 0) for y in Y]
    d = orc.two_loop(Ym[-1], free, Sm, Ym, eps=1e-12)
    assert np.allclose(d, -Sm[-1], rtol=1e-9, atol=1e-11)


def test_two_loop_screen_soundness(orc):
    """a pair with <s[S],y[S]> <= eps ||y[S]||^2 never influences d
    (removing an OLDER screened pair gives the same output bit for bit)."""
    rng = np.random.default_rng(7)
    for _ in range(50):
        n = 10
        free = rng.random(n) < 0.8
        S = [rng.standard_normal(n) for _ in range(3)]
        Y = [rng.standard_normal(n) for _ in range(3)]
        s0, y0 = S[0], Y[0]
        Y[0] = -y0 if (s0[free] @ y0[free]) > 0 else y0   # pair 0 fails the screen
        g = rng.standard_normal(n)
        d_all = orc.two_loop(g, free, S, Y)
        d_wo = orc.two_loop(g, free, S[1:], Y[1:])
        assert np.array_equal(d_all, d_wo)


def test_two_loop_descent_on_free_set(orc):
    """SPEC.md:192 / PAPER.md:151: <g[S], d[S]> < 0 whenever the screen is passed."""
    rng = np.random.default_rng(8)
    for _ in range(100):
        n = 20
        free = rng.random(n) < 0.6; free[0] = True
        S = [rng.standard_normal(n) for _ in range(5)]
        Y = [rng.standard_normal(n) for _ in range(5)]
        g = rng.standard_normal(n)
        d = orc.two_loop(g, free, S, Y, eps=1e-9)
        assert g[free] @ d[free] < 0


# ---------------------------------------------------------------- Alg. 2 / step
def test_project_direction_examples(orc):
    for ex in GOLD["project_direction"]:
        p, br = orc.project_direction(ex["x"], ex["g"], ex["d"], ex["l"], ex["u"], ex["eps"])
        assert br == ex["projected"], ex["cite"]
        assert np.allclose(p, ex["p"], rtol=0, atol=1e-15), ex["cite"]


def test_project_direction_properties(orc):
    """truncated p has ||p|| <= ||d|| and
    <p, g> <= <d, g>; projected p keeps x + p feasible."""
    rng = np.random.default_rng(9)
    for _ in range(500):
        n = 16
        l = np.zeros(n); u = np.ones(n)
        x = np.clip(rng.random(n) * 1.4 - 0.2, 0, 1)
        g = rng.standard_normal(n)
        eps = 1e-6
        fr = orc.working_set(x, g, l, u, eps)
        d = np.where(fr, -g * rng.random(n) * 2, 0.0)
        p, br = orc.project_direction(x, g, d, l, u, eps)
        if br:
            assert np.all(x + p >= 0) and np.all(x + p <= 1)
            assert p @ g <= -eps * (p @ p)
        else:
            assert np.linalg.norm(p) <= np.linalg.norm(d)
            assert p @ g <= d @ g + 1e-15


def test_max_step_examples(orc):
    for ex in GOLD["max_step"]:
        out = orc.max_step(ex["x"], ex["p"], _bnd(ex["l"]), _bnd(ex["u"]))
        exp = np.inf if ex["out"] == "inf" else ex["out"]
        assert out == exp, ex["cite"]


def test_armijo_examples(orc):
    for ex in GOLD["armijo"]:
        assert orc.armijo_scalar_quadratic(ex["x"], ex["p"]) == ex["alpha"], ex["cite"]


# ---------------------------------------------------------------- Alg. 1 (NNLS)
def test_minimize_example(orc):
    ex = GOLD["minimize"][0]
    P = orc.LSQ(np.array(ex["A"], float), b=ex["b"])
    r = orc.minimize_lsq(P, l=np.zeros(2))
    assert r.status == orc.CONVERGED
    assert np.allclose(r.x, ex["x"], atol=1e-12) and r.f == pytest.approx(ex["f"], abs=1e-14)


def _nnls_bruteforce(A, b):
    """Enumerate every support F; the unique KKT point of the strictly convex
    NNLS (A full column rank) is the minimiser (PAPER.md:198 Corollary)."""
    m, n = A.shape
    best = None
    for k in range(n + 1):
        for F in itertools.combinations(range(n), k):
            x = np.zeros(n)
            if F:
                sol, *_ = np.linalg.lstsq(A[:, F], b, rcond=None)
                if np.any(sol <= 0):
                    continue
                x[list(F)] = sol
            g = A.T @ (A @ x - b)
            mask = np.ones(n, bool); mask[list(F)] = False
            if np.all(g[mask] >= -1e-10):
                f = 0.5 * np.sum((A @ x - b) ** 2)
                if best is None or f < best[1]:
                    best = (x, f)
    return best


@pytest.mark.parametrize("seed", range(40))
def test_nnls_bruteforce_active_set(orc, seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 11)); m = n + int(rng.integers(0, 8))
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    b = rng.standard_normal(m)
    x_bf, f_bf = _nnls_bruteforce(A, b)
    r = orc.minimize_lsq(orc.LSQ(A, b=b), l=np.zeros(n),
                         opts=orc.Options(tol=1e-11, max_iters=5000))
    assert r.status == orc.CONVERGED
    assert np.all(r.x >= 0)                                             # feasible (Thm. 1)
    assert abs(r.f - f_bf) <= 1e-10 * max(1.0, abs(f_bf))
    assert np.allclose(r.x, x_bf, atol=1e-7)


@pytest.mark.parametrize("seed", range(6))
def test_nnls_vs_scipy(orc, seed):
    from scipy.optimize import nnls
    rng = np.random.default_rng(2000 + seed)
    m, n = 300, 150
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    b = rng.standard_normal(m)
    xs, rn = nnls(A, b, maxiter=5000)
    # tol 1e-6 (the north-star KKT tolerance): tighter tolerances hit the Armijo
    # cancellation floor f(x+ap)-f(x) ~ ulp(f) (hard part 4)
    r = orc.minimize_lsq(orc.LSQ(A, b=b), l=np.zeros(n), opts=orc.Options(tol=1e-6))
    assert r.status == orc.CONVERGED
    assert r.f == pytest.approx(0.5 * rn ** 2, rel=1e-10)
    assert r.pg_inf <= 1e-6


def test_nnls_inactive_bounds_closed_form(orc):
    """b = A x_true with x_true >= 1: bounds inactive, x* = (A^T A)^{-1} A^T b."""
    rng = np.random.default_rng(11)
    m, n = 80, 30
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    xt = 1.0 + rng.random(n)
    b = A @ xt
    r = orc.minimize_lsq(orc.LSQ(A, b=b), l=np.zeros(n), opts=orc.Options(tol=1e-12))
    x_ls = np.linalg.solve(A.T @ A, A.T @ b)
    assert np.allclose(r.x, x_ls, atol=1e-9) and r.f <= 1e-20


def test_unconstrained_quadratic(orc):
    """f = 1/2||x - c||^2 with no bounds => x* = c."""
    rng = np.random.default_rng(12)
    c = rng.standard_normal(40)
    r = orc.minimize_lsq(orc.LSQ(np.eye(40), b=c), opts=orc.Options(tol=1e-12))
    assert np.allclose(r.x, c, atol=1e-12)


def test_monotone_and_feasible_iterates(orc):
    """Theorem 1: f decreases every iteration and every
    iterate is feasible.  Checked by re-running with max_iters = k."""
    rng = np.random.default_rng(13)
    A = rng.standard_normal((60, 40)) / np.sqrt(60)
    b = rng.standard_normal(60)
    P = orc.LSQ(A, b=b)
    fs = []
    for k in range(0, 25):
        r = orc.minimize_lsq(P, l=np.zeros(40), opts=orc.Options(max_iters=k))
        assert np.all(r.x >= 0)
        fs.append(r.f)
    assert all(fs[i + 1] <= fs[i] for i in range(len(fs) - 1))


def test_nnls_free_fraction_binomial(orc):
    """Gaussian A (m >= n), Gaussian b: #nonzeros of x* ~ Binomial(n, 1/2)
    (SURVEY.md 8(c) pin (vi)).  Mean over 40 draws of n=60 must be near 30."""
    nz = []
    for s in range(40):
        rng = np.random.default_rng(3000 + s)
        A = rng.standard_normal((120, 60)) / np.sqrt(120)
        b = rng.standard_normal(120)
        r = orc.minimize_lsq(orc.LSQ(A, b=b), l=np.zeros(60), opts=orc.Options(tol=1e-10))
        nz.append(int(np.sum(r.x > 0)))
    mean = np.mean(nz)
    assert abs(mean - 30) < 4 * np.sqrt(15 / 40)   # 4 sigma of the mean


# ---------------------------------------------------------------- lasso split
@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_lasso_orthonormal_closed_form(orc, alpha):
    """A^T A = I: x* = soft(A^T b, lam*alpha) / (1 + lam(1-alpha)); u * v = 0."""
    rng = np.random.default_rng(14)
    m, n = 50, 20
    Q, _ = np.linalg.qr(rng.standard_normal((m, n)))
    b = rng.standard_normal(m)
    lam = 0.3
    P = orc.LSQ(Q, b=b, c=np.full(2 * n, lam * alpha), delta=lam * (1 - alpha), split=True)
    r = orc.minimize_lsq(P, l=np.zeros(2 * n), opts=orc.Options(tol=1e-12))
    z = Q.T @ b
    xs = np.sign(z) * np.maximum(np.abs(z) - lam * alpha, 0) / (1 + lam * (1 - alpha))
    assert np.allclose(r.x[:n] - r.x[n:], xs, atol=1e-9)
    assert np.max(r.x[:n] * r.x[n:]) <= 1e-12


# ---------------------------------------------------------------- Alg. 4
def test_al_scalar_equality(orc):
    """min x^2 s.t. x = 1 => x = 1, lambda = -2 (KKT by hand)."""
    P = orc.LSQ(np.array([[np.sqrt(2.0)]]), b=[0.0], E=np.ones((1, 1)), e=[1.0])
    r = orc.al_solve(P, opts=orc.Options(tol=1e-10))
    assert r.status == orc.CONVERGED
    assert r.x[0] == pytest.approx(1.0, abs=1e-6)
    assert r.lam[0] == pytest.approx(-2.0, abs=1e-5)


def _simplex_proj(c):
    """Euclidean projection onto the probability simplex (sort-based closed form)."""
    u = np.sort(c)[::-1]
    css = np.cumsum(u)
    k = np.nonzero(u * np.arange(1, len(c) + 1) > (css - 1))[0][-1]
    tau = (css[k] - 1) / (k + 1)
    return np.maximum(c - tau, 0)


def test_al_simplex_example(orc):
    ex = GOLD["al"][1]
    P = orc.LSQ(np.eye(2), b=ex["b"], E=np.ones((2, 1)), e=[1.0])
    r = orc.al_solve(P, l=np.zeros(2))
    assert np.allclose(r.x, ex["x"], atol=1e-6)


@pytest.mark.parametrize("seed", range(8))
def test_al_simplex_projection(orc, seed):
    rng = np.random.default_rng(4000 + seed)
    n = 30
    c = rng.standard_normal(n) * 0.5
    P = orc.LSQ(np.eye(n), b=c, E=np.ones((n, 1)), e=[1.0])
    r = orc.al_solve(P, l=np.zeros(n), opts=orc.Options(tol=1e-9))
    assert r.status == orc.CONVERGED
    assert np.allclose(r.x, _simplex_proj(c), atol=1e-6)
    assert abs(r.x.sum() - 1) <= 1e-6


@pytest.mark.parametrize("seed", range(6))
def test_al_inequality_capped_simplex(orc, seed):
    """min 1/2||x-c||^2 s.t. 1^T x <= 1, x >= 0: x = c_+ if sum(c_+) <= 1 else
    the simplex projection; mu >= 0 always."""
    rng = np.random.default_rng(5000 + seed)
    n = 20
    c = rng.standard_normal(n) * (0.1 if seed % 2 else 0.6)
    P = orc.LSQ(np.eye(n), b=c, G=np.ones((n, 1)), hv=[1.0])
    r = orc.al_solve(P, l=np.zeros(n), opts=orc.Options(tol=1e-9))
    cp = np.maximum(c, 0)
    ref = cp if cp.sum() <= 1 else _simplex_proj(c)
    assert np.allclose(r.x, ref, atol=1e-6)
    assert np.all(r.mu >= 0)


def test_al_without_constraints_is_one_inner_solve(orc):
    """with m = p = 0 the AL loop is one box solve, bit for bit."""
    rng = np.random.default_rng(15)
    A = rng.standard_normal((40, 20)); b = rng.standard_normal(40)
    P = orc.LSQ(A, b=b)
    r1 = orc.al_solve(P, l=np.zeros(20))
    r2 = orc.minimize_lsq(P, l=np.zeros(20), x0=np.zeros(20))
    assert np.array_equal(r1.x, r2.x) and r1.outer_iters == 1


def test_svm_two_point_example(orc):
    """two points, y = [+1,-1], K = I, c = 1 => a = [1, 1], f = -1."""
    ex = GOLD["al"][2]
    y = np.array([1.0, -1.0])
    P = orc.LSQ(np.eye(2), c=-np.ones(2), colscale=y, E=y.reshape(2, 1), e=[0.0])
    r = orc.al_solve(P, l=np.zeros(2), u=np.ones(2), opts=orc.Options(tol=1e-10))
    assert np.allclose(r.x, ex["a"], atol=1e-6) and r.f == pytest.approx(ex["f"], abs=1e-6)


@pytest.mark.parametrize("seed", range(3))
def test_svm_duality_gap(orc, seed):
    """Linear-kernel SVM: primal 1/2||w||^2 + C sum hinge equals minus the dual
    optimum (strong duality), with w = X^T (a*y) and b from the free SVs."""
    import synth
    p = synth.svm_dual_linear(300, 5, 6000 + seed, sep=1.5)
    P = orc.LSQ(p.M, c=p.c, colscale=p.colscale, E=p.E, e=p.e)
    r = orc.al_solve(P, l=p.lower, u=p.upper, opts=orc.Options(tol=1e-9),
                     al_opts=orc.ALOptions(feas_tol=1e-9))
    a, y, X = r.x, p.colscale, p.M.T
    C = p.upper[0]
    assert np.all(a >= 0) and np.all(a <= C)
    assert abs(y @ a) <= 1e-8
    w = X.T @ (a * y)
    fsv = (a > 1e-6) & (a < C - 1e-6)
    b0 = np.median(y[fsv] - X[fsv] @ w)
    primal = 0.5 * w @ w + C * np.sum(np.maximum(0, 1 - y * (X @ w + b0)))
    dual = r.f
    assert abs(primal + dual) <= 1e-5 * abs(dual)


# ---------------------------------------------------------------- paper replay
@pytest.mark.slow
def test_ds2_iteration_count_loose(orc):
    """NNLS reaches absolute error 1e-10 in 30-40 iterations.
    Loosely pinned on data set (ii) at t = 0.25 (33-34 f/g evals)."""
    import synth
    from scipy.optimize import nnls
    p = synth.nnls_ds2(0.25, 12)
    _, rn = nnls(p.M, p.b, maxiter=10000)
    fstar = 0.5 * rn ** 2
    for k in range(10, 80):
        r = orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower,
                             opts=orc.Options(tol=0.0, max_iters=k))
        if r.f - fstar <= 1e-10:
            break
    assert 15 <= k <= 60, k


@pytest.mark.parametrize("seed", range(10))
def test_no_projection_variant_same_optimum(orc, seed):
    """skipping Alg. 2's projection branch keeps the convergence
    guarantee -- the variant reaches the brute-force NNLS optimum too."""
    rng = np.random.default_rng(7000 + seed)
    n = int(rng.integers(3, 10)); m = n + 4
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    b = rng.standard_normal(m)
    x_bf, f_bf = _nnls_bruteforce(A, b)
    r = orc.minimize_lsq(orc.LSQ(A, b=b), l=np.zeros(n),
                         opts=orc.Options(tol=1e-11, max_iters=20000, no_projection=True))
    assert r.status == orc.CONVERGED and r.last_branch == 0
    assert abs(r.f - f_bf) <= 1e-10 * max(1.0, abs(f_bf))
