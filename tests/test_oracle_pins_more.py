"""Pins for the oracle parts round 1 left unpinned ("What's weak" 1):

* Alg. 3's initial scaling when the NEWEST pair fails the screen
  (reading R4): H0 = I, the passing pairs still update H;
* Alg. 4's multiplier updates, violation measure and penalty rule
  (readings R20/R21) against SPEC's worked examples
   and a hand-computed outer-iteration trace;
* the LSQ Armijo search itself (readings R10/R11): its
  start alpha_0 = min(1, alpha_max) and the accepted trial, on hand-computed
  two-variable instances.

Each ``check_*`` function is also run against deliberately broken builds of
the oracle in tests/test_oracle_mutants.py, which asserts that it FAILS there.
"""
import json
import os
from fractions import Fraction as F

import numpy as np
import pytest

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- Alg. 3, R4
def _dense_inverse_bfgs(S, Y, free, gamma):
    """H0 = gamma I on S, H <- V^T H V + rho s s^T (Nocedal & Wright eq. 7.19)
    over the given pairs, oldest first, restricted to the free set."""
    idx = np.flatnonzero(free)
    H = gamma * np.eye(len(idx))
    for s, y in zip(S, Y):
        s, y = s[idx], y[idx]
        rho = 1.0 / (s @ y)
        V = np.eye(len(idx)) - rho * np.outer(y, s)
        H = V.T @ H @ V + rho * np.outer(s, s)
    return idx, H


def _history(rng, n, free, nh, failing):
    """nh pairs, oldest first; pair i passes the screen (y = Q s, <s,y>_S > 0)
    unless i is in ``failing`` (y = -Q s, <s,y>_S < 0)."""
    B = rng.standard_normal((n, n))
    Q = B @ B.T + n * np.eye(n)
    S = [np.where(free, rng.standard_normal(n), 0.0) for _ in range(nh)]
    Y = [(-1.0 if i in failing else 1.0) * (Q @ s) for i, s in enumerate(S)]
    return S, Y


def check_two_loop_newest_pair_fails(orc, seeds=range(40)):
    """the initial scaling q <- (rho^{k-1}/||y^{k-1}||^2) q is
    applied only 'if rho^{k-1} > eps ||y^{k-1}||^2' -- pair k-1, the newest.
    When it fails, H0 = I and the passing (older) pairs still enter the
    recursion: d[S] = -H g[S] with H the dense inverse-BFGS recursion over the
    passing pairs from H0 = I."""
    for seed in seeds:
        rng = np.random.default_rng(5000 + seed)
        n = int(rng.integers(3, 9)); nh = int(rng.integers(2, 5))
        free = rng.random(n) < 0.8
        free[:2] = True
        S, Y = _history(rng, n, free, nh, failing={nh - 1})
        g = rng.standard_normal(n)
        for full in (False, True):
            d = orc.two_loop(g, free, S, Y, eps=1e-12, screen_full_norm=full)
            idx, H = _dense_inverse_bfgs(S[:-1], Y[:-1], free, 1.0)
            ref = -(H @ g[idx])
            assert np.allclose(d[idx], ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max()), seed
            assert np.all(d[~free] == 0.0)


def check_two_loop_middle_pair_fails(orc, seeds=range(40)):
    """A failing pair in the middle is skipped in both loops; the newest pair
    passes, so H0 = (rho^{k-1}/nu^{k-1}) I."""
    for seed in seeds:
        rng = np.random.default_rng(6000 + seed)
        n = int(rng.integers(3, 9)); nh = 3
        free = rng.random(n) < 0.8
        free[:2] = True
        S, Y = _history(rng, n, free, nh, failing={1})
        g = rng.standard_normal(n)
        d = orc.two_loop(g, free, S, Y, eps=1e-12)
        sN, yN = S[-1][free], Y[-1][free]
        idx, H = _dense_inverse_bfgs([S[0], S[2]], [Y[0], Y[2]], free, (sN @ yN) / (yN @ yN))
        ref = -(H @ g[idx])
        assert np.allclose(d[idx], ref, rtol=1e-9, atol=1e-12 * np.abs(ref).max()), seed


def test_two_loop_newest_pair_fails_screen(orc):
    check_two_loop_newest_pair_fails(orc)


def test_two_loop_middle_pair_fails_screen(orc):
    check_two_loop_middle_pair_fails(orc)


# ---------------------------------------------------------------- Alg. 4 pieces
def check_al_spec_examples(orc):
    for ex in GOLD["al_update_rho"]:
        assert orc.al_update_rho(ex["rho"], ex["vprev"], ex["v"]) == ex["out"], ex["cite"]
    for ex in GOLD["al_update_multipliers"]:
        lam, mu = orc.al_update_multipliers(ex["lam"], ex["h"], ex["mu"], ex["g"], ex["rho"])
        assert np.array_equal(lam, np.array(ex["lam_out"], float)), ex["cite"]
        assert np.array_equal(mu, np.array(ex["mu_out"], float)), ex["cite"]
    for ex in GOLD["al_violation"]:
        assert orc.al_violation(ex["h"], ex["g"], ex["mu"], ex["rho"]) == ex["out"], ex["cite"]


def test_al_spec_examples(orc):
    check_al_spec_examples(orc)


def check_al_hand_trace(orc):
    """The first three outer iterations of Alg. 4 computed by hand
    (tests/golden/spec_examples.json 'al_trace')."""
    ex = GOLD["al_trace"][0]
    P = orc.LSQ(np.array(ex["M"]), b=ex["b"], E=np.array(ex["E"]), e=ex["e"])
    res, tr = orc.al_solve(P, m_hist=5, trace=True)
    assert res.status == orc.CONVERGED
    for rec in ex["records"]:
        t = tr[rec["k"] - 1]
        assert t["rho_used"] == rec["rho_used"] and t["rho_next"] == rec["rho_next"], rec["note"]
        assert t["x"][0] == pytest.approx(rec["x"], abs=1e-12), rec["note"]
        assert t["lam"][0] == pytest.approx(rec["lam"], abs=1e-11), rec["note"]
        assert t["v"] == pytest.approx(rec["v"], abs=1e-12), rec["note"]


def test_al_hand_trace(orc):
    check_al_hand_trace(orc)


def _exact_al_trace(c, a, rho0, kind, n_outer, lam0=F(0), x0=F(0), feas_tol=F(1, 10**6)):
    """Alg. 4 in exact rational arithmetic on min c/2 (x - a)^2 s.t. x = 1
    (kind 'eq') or x <= 1 (kind 'in'), no box, with the inner problem solved
    in closed form: x = (c a + rho - m)/(c + rho) for the equality (m = lam)
    and for an active inequality (m = mu, valid while x - 1 + mu/rho > 0;
    else x = a).  Readings R20 (rho rule after the updates) and R21 (v)."""
    rho, m, x = F(rho0), lam0, x0

    def viol(x, m, rho):
        h = x - 1
        if kind == "eq":
            return abs(h)
        return abs(min(-h, m / rho))

    vprev = viol(x, m, rho)
    out = []
    for _ in range(n_outer):
        xe = (c * a + rho - m) / (c + rho)
        x = xe if (kind == "eq" or xe - 1 + m / rho > 0) else F(a)
        h = x - 1
        m = m + rho * h if kind == "eq" else max(m + rho * h, F(0))
        v = viol(x, m, rho)
        assert v == 0 or abs(v - vprev / 2) > F(1, 10**6) * vprev     # no near-ties
        rho_used = rho
        if v > vprev / 2:
            rho = rho * 2
        vprev = v
        out.append((rho_used, v, rho, m, x))
        if v <= feas_tol:
            break
    return out


def check_al_exact_traces(orc):
    """Whole outer trajectories vs exact arithmetic (closed-form inner solves):
    equality and inequality, cold and warm-started multipliers.  rho must
    double exactly where the exact trace doubles it."""
    cases = [("eq", F(9), F(3), F(0)), ("in", F(9), F(3), F(0)), ("eq", F(25), F(-2), F(0)),
             ("in", F(9), F(3), F(5)), ("in", F(9), F(3), F(30)), ("eq", F(9), F(3), F(-3))]
    for kind, c, a, m0 in cases:
        sc = float(c) ** 0.5
        if kind == "eq":
            P = orc.LSQ(np.array([[sc]]), b=[sc * float(a)], E=np.ones((1, 1)), e=[1.0])
            kw = {"lam0": [float(m0)]} if m0 else {}
        else:
            P = orc.LSQ(np.array([[sc]]), b=[sc * float(a)], G=np.ones((1, 1)), hv=[1.0])
            kw = {"mu0": [float(m0)]} if m0 else {}
        res, tr = orc.al_solve(P, m_hist=5, trace=True, **kw)
        ref = _exact_al_trace(c, a, 1, kind, len(tr), lam0=m0)
        n = min(len(tr), 6)
        for k in range(n):
            rho_used, v, rho_next, m, x = ref[k]
            t = tr[k]
            mult = t["lam"][0] if kind == "eq" else t["mu"][0]
            assert t["rho_used"] == float(rho_used) and t["rho_next"] == float(rho_next), (kind, c, a, m0, k)
            assert t["x"][0] == pytest.approx(float(x), abs=1e-10), (kind, c, a, m0, k)
            assert mult == pytest.approx(float(m), abs=1e-9 * max(1.0, abs(float(m)))), (kind, c, a, m0, k)
            assert t["v"] == pytest.approx(float(v), abs=1e-10), (kind, c, a, m0, k)


def test_al_exact_traces(orc):
    check_al_exact_traces(orc)


def test_al_warm_start_reentry(orc):
    """Re-entering Alg. 4 with the multipliers and x of a converged run is a
    fixed point: the first inner solve starts at a KKT point of L, the
    multiplier update adds rho h ~ 0 and the method stops after one outer
    iteration with the same x (the checkpoint/resume use of SURVEY.md 5)."""
    rng = np.random.default_rng(3)
    n = 30
    A = rng.standard_normal((40, n))
    b = rng.standard_normal(40)
    P = orc.LSQ(A, b=b, E=np.ones((n, 1)), e=[1.0])
    r1 = orc.al_solve(P, l=0.0, opts=orc.Options(tol=1e-9), al_opts=orc.ALOptions(feas_tol=1e-9))
    assert r1.status == orc.CONVERGED
    r2 = orc.al_solve(P, l=0.0, opts=orc.Options(tol=1e-9), al_opts=orc.ALOptions(feas_tol=1e-9),
                      x0=r1.x, lam0=r1.lam)
    assert r2.status == orc.CONVERGED and r2.outer_iters == 1
    assert np.max(np.abs(r2.x - r1.x)) <= 1e-7
    assert abs(r2.lam[0] - r1.lam[0]) <= 1e-6 * max(1.0, abs(r1.lam[0]))


# ---------------------------------------------------------------- Armijo on LSQ
def check_armijo_lsq_examples(orc):
    for ex in GOLD["armijo_lsq"]:
        P = orc.LSQ(np.array(ex["M"], float), b=ex["b"])
        x = np.array(ex["x"], float)
        l = np.array(ex["l"], float)
        if ex["d"] is not None:                      # the branch and alpha_max come from Alg. 2
            g = P.grad(x)
            p, br = orc.project_direction(x, g, ex["d"], l, None, 1e-9)
            assert br == ex["projected"], ex["cite"]
            assert np.array_equal(p, np.array(ex["p"], float)), ex["cite"]
            assert orc.max_step(x, p, l, None) == ex["amax"], ex["cite"]
        ok, alpha, ft, nbt, _ = orc.armijo_lsq(P, x, ex["p"], ex["amax"], l=l,
                                               opts=orc.Options(c1=ex["c1"]))
        assert ok, ex["cite"]
        assert alpha == ex["alpha"] and nbt == ex["n_bt"], (alpha, nbt, ex["cite"])
        assert ft == pytest.approx(ex["f_t"], abs=1e-15), ex["cite"]


def test_armijo_lsq_examples(orc):
    check_armijo_lsq_examples(orc)


def _exact_armijo(Mq, r, q, amax, c1, shrink, max_bt):
    """Armijo in exact arithmetic on f_t = 1/2||r + alpha q||^2: the first
    t with f_t <= f + c1 alpha <r, q> from alpha_0 = min(1, amax)."""
    f = sum(v * v for v in r) / 2
    gp = sum(a * b for a, b in zip(r, q))
    alpha = min(F(1), amax)
    for t in range(max_bt + 1):
        if t:
            alpha = alpha * shrink
        ft = sum((a + alpha * b) ** 2 for a, b in zip(r, q)) / 2
        if ft <= f + c1 * alpha * gp:
            return alpha, t
    return None, None


def check_armijo_lsq_random(orc, n_cases=60):
    """Random small LSQ instances with dyadic data (every product exact in
    fp64, so the float decisions equal the exact ones away from ties)."""
    rng = np.random.default_rng(11)
    done = 0
    while done < n_cases:
        m = int(rng.integers(1, 4)); n = int(rng.integers(1, 4))
        M = rng.integers(-8, 9, (m, n)) / 4.0
        x = rng.integers(0, 8, n) / 8.0
        b = rng.integers(-16, 17, m) / 8.0
        p = rng.integers(-8, 9, n) / 8.0
        amax = float(rng.choice([0.25, 0.5, 0.75, 1.0, 2.0, 3.0]))
        r = M @ x - b; q = M @ p
        if not (r @ q < 0):
            continue
        c1 = float(rng.choice([1e-4, 0.25, 0.5]))
        P = orc.LSQ(M, b=b)
        ok, alpha, ft, nbt, _ = orc.armijo_lsq(P, x, p, amax, opts=orc.Options(c1=c1, max_backtracks=30))
        ea, et = _exact_armijo(M, [F(v) for v in r], [F(v) for v in q], F(amax), F(c1), F(1, 2), 30)
        if ea is None:
            assert not ok
        else:
            assert ok and alpha == float(ea) and nbt == et, (M, x, b, p, amax, c1)
        done += 1


def test_armijo_lsq_random_exact(orc):
    check_armijo_lsq_random(orc)


# ---------------------------------------------------------------- OpenMP variant
def test_threaded_oracle_is_bit_identical(orc):
    """the all-cores oracle (OpenMP over output elements, same
    per-output summation order) gives the 1-thread oracle's bits: matvecs with
    ragged row blocks, and a whole NNLS solve."""
    import synth
    rng = np.random.default_rng(0)
    A = rng.standard_normal((1003, 357)); x = rng.standard_normal(357); r = rng.standard_normal(1003)
    prob = synth.nnls_gaussian(700, 300, 12)
    try:
        orc.set_threads(1)
        q1, g1 = orc.matvec(A, x), orc.matvec_t(A, r)
        s1 = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
        for t in (2, 3, 7):
            orc.set_threads(t)
            assert np.array_equal(orc.matvec(A, x), q1) and np.array_equal(orc.matvec_t(A, r), g1)
            st = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
            assert np.array_equal(st.x, s1.x) and st.f == s1.f and st.iters == s1.iters
    finally:
        orc.set_threads(1)


# ---------------------------------------------------------------- R13 optional refresh
@pytest.mark.parametrize("R", [1, 3])
def test_periodic_refresh_changes_only_rounding(orc, R):
    """R13: the carried residual r + alpha q equals M~x' - b in exact arithmetic,
    so refreshing r, f and g every R iterations leaves the trajectory unchanged
    up to rounding: f after k = 1..6 iterations agrees with the refresh-free run
    to 1e-12, and the optimum to 1e-12."""
    import synth
    p = synth.nnls_gaussian(150, 80, 17)
    P = orc.LSQ(p.M, b=p.b)
    for k in range(1, 7):
        a = orc.minimize_lsq(P, l=p.lower, opts=orc.Options(max_iters=k, tol=1e-12))
        b = orc.minimize_lsq(P, l=p.lower, opts=orc.Options(max_iters=k, tol=1e-12, refresh_every=R))
        assert a.iters == b.iters == k
        assert abs(a.f - b.f) <= 1e-12 * abs(a.f)
    a = orc.minimize_lsq(P, l=p.lower)
    b = orc.minimize_lsq(P, l=p.lower, opts=orc.Options(refresh_every=R))
    assert a.status == b.status == orc.CONVERGED
    assert abs(a.f - b.f) <= 1e-12 * abs(a.f)


def test_periodic_refresh_removes_residual_drift(orc):
    """A long run (a badly conditioned NNLS, ~hundreds of iterations): with the
    refresh the reported f (recomputed from x at the end in both cases) is
    unchanged while the refresh keeps the carried f exact at the refresh points
    -- pinned through the final f against the refresh-free run and against
    scipy's active-set NNLS optimum."""
    from scipy.optimize import nnls
    import synth
    p = synth.nnls_ds1(0.1, 3)
    P = orc.LSQ(p.M, b=p.b)
    a = orc.minimize_lsq(P, l=p.lower, opts=orc.Options(max_iters=20000))
    b = orc.minimize_lsq(P, l=p.lower, opts=orc.Options(max_iters=20000, refresh_every=10))
    xs, rn = nnls(p.M, p.b, maxiter=100000)
    fs = 0.5 * rn * rn
    for r in (a, b):
        assert r.status == orc.CONVERGED
        assert abs(r.f - fs) <= 1e-8 * abs(fs)
