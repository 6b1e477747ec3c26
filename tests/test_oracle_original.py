"""Pins of the oracle's ORIGINAL L-BFGS-B (SURVEY 8(f) N3 baseline, Byrd et al.
1995: generalized Cauchy point + direct primal subspace minimisation;
PAPER.md:436-457) against library solvers: scipy's active-set NNLS
(Lawson-Hanson) and scipy's L-BFGS-B (the Fortran code of the same authors)
on box-constrained least squares."""
import numpy as np
import pytest
import scipy.optimize


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_nnls_matches_lawson_hanson(orc, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((240, 120)) / np.sqrt(240); b = rng.standard_normal(240)
    xs, rn = scipy.optimize.nnls(A, b)
    r, tcp = orc.minimize_lsq_original(orc.LSQ(A, b=b), l=np.zeros(120),
                                       opts=orc.Options(tol=1e-7, max_iters=5000))
    assert r.status == orc.CONVERGED and r.pg_inf <= 1e-7
    assert r.f == pytest.approx(0.5 * rn ** 2, rel=1e-10)
    assert np.allclose(r.x, xs, atol=1e-6)
    assert tcp > 0.0


@pytest.mark.parametrize("seed", [4, 5])
def test_two_sided_box_matches_fortran_lbfgsb(orc, seed):
    rng = np.random.default_rng(seed)
    m, n = 150, 90
    A = rng.standard_normal((m, n)) / np.sqrt(m); b = 3.0 * rng.standard_normal(m)
    lo = -rng.uniform(0.0, 0.5, n); up = rng.uniform(0.0, 0.5, n)
    fg = lambda x: (0.5 * np.sum((A @ x - b) ** 2), A.T @ (A @ x - b))
    ref = scipy.optimize.minimize(fg, np.zeros(n), jac=True, method="L-BFGS-B", bounds=list(zip(lo, up)),
                                  options=dict(maxcor=5, gtol=1e-10, ftol=1e-16, maxiter=10000))
    r, _ = orc.minimize_lsq_original(orc.LSQ(A, b=b), l=lo, u=up, opts=orc.Options(tol=1e-7, max_iters=5000))
    assert r.status == orc.CONVERGED
    assert r.f == pytest.approx(ref.fun, rel=1e-9)
    assert np.all(r.x >= lo) and np.all(r.x <= up)


def test_same_solution_as_modified_method(orc):
    """Both methods reach the same KKT point on the paper's data set (ii)."""
    import synth
    p = synth.nnls_ds2(0.25, 12)
    P = orc.LSQ(p.M, b=p.b)
    o = orc.Options(tol=1e-8, max_iters=5000, armijo_diff=True)       # below the plain test's floor (R29)
    r1, _ = orc.minimize_lsq_original(P, l=p.lower, opts=o)
    r2 = orc.minimize_lsq(P, l=p.lower, opts=o)
    assert r1.status == r2.status == orc.CONVERGED
    assert r1.f == pytest.approx(r2.f, rel=1e-9)
