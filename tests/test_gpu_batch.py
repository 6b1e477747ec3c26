"""GPU parity of the batched small-problem mode (SURVEY 8(f) N4 "replicas",
one CTA per problem; lbfgsb_solve_batched_lsq) against the oracle, problem by
problem, and against the single-problem path (-m gpu)."""
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


def _batch(B, m, n, seed0):
    import synth
    probs = [synth.nnls_gaussian(m, n, seed0 + k) for k in range(B)]
    A = np.stack([p.M for p in probs]); b = np.stack([p.b for p in probs])
    return probs, A, b


@pytest.mark.parametrize("B,m,n,mh", [(24, 200, 100, 5), (7, 50, 31, 3), (5, 400, 200, 5), (3, 1, 9, 5)])
def test_batched_nnls_vs_oracle(lb, orc, B, m, n, mh):
    probs, A, b = _batch(B, m, n, 1000 + m)
    M = lb.colmajor_batch(A)
    bd = torch.from_numpy(b).cuda()
    x = torch.zeros(B, n, dtype=torch.float64, device="cuda")
    lo = torch.zeros(B, n, dtype=torch.float64, device="cuda")
    res = lb.solve_batched_lsq(M, bd, x, lower=lo, m_hist=mh)
    xs = x.cpu().numpy()
    for k, p in enumerate(probs):
        ro = orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower, m_hist=mh)
        r = res[k]
        assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED, (k, r)
        assert r.pg_inf <= 1e-6
        fl = max(abs(ro.f), 1e-12)
        assert abs(r.f - ro.f) <= 1e-8 * fl, (k, r.f, ro.f)
        assert np.all(xs[k] >= 0)


def test_batched_two_sided_box_matches_single_path(lb):
    """Each CTA takes the decisions lbfgsb_solve takes on the same problem
    alone (same device decision functions; sums in a different order)."""
    import synth
    B, m, n = 6, 120, 80
    probs, A, b = _batch(B, m, n, 77)
    rng = np.random.default_rng(3)
    lo = -rng.uniform(0.0, 0.3, (B, n)); up = rng.uniform(0.0, 0.3, (B, n))
    x = torch.zeros(B, n, dtype=torch.float64, device="cuda")
    res = lb.solve_batched_lsq(lb.colmajor_batch(A), torch.from_numpy(b).cuda(), x,
                               lower=torch.from_numpy(lo).cuda(), upper=torch.from_numpy(up).cuda())
    for k, p in enumerate(probs):
        obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda())
        s = lb.Solver(n, 5, lower=torch.from_numpy(lo[k]).cuda(), upper=torch.from_numpy(up[k]).cuda())
        xk = torch.zeros(n, dtype=torch.float64, device="cuda")
        r1 = s.solve(obj, xk)
        assert res[k].status == r1.status == lb.CONVERGED
        assert abs(res[k].f - r1.f) <= 1e-10 * abs(r1.f)
        assert abs(res[k].iters - r1.iters) <= 2
        assert np.allclose(x[k].cpu().numpy(), xk.cpu().numpy(), atol=1e-6)


def test_batched_empty_and_stationary(lb):
    res = lb.solve_batched_lsq(torch.zeros(0, 3, 2, dtype=torch.float64, device="cuda"),
                               torch.zeros(0, 2, dtype=torch.float64, device="cuda"),
                               torch.zeros(0, 3, dtype=torch.float64, device="cuda"))
    assert res == []
    # A = I, b <= 0: x* = 0 at x^0, S^0 empty -> converged with 0 iterations
    A = np.stack([np.eye(4)] * 3); b = -np.ones((3, 4))
    x = torch.zeros(3, 4, dtype=torch.float64, device="cuda")
    res = lb.solve_batched_lsq(lb.colmajor_batch(A), torch.from_numpy(b).cuda(), x,
                               lower=torch.zeros(3, 4, dtype=torch.float64, device="cuda"))
    assert all(r.status == lb.CONVERGED and r.iters == 0 for r in res)
    assert torch.all(x == 0)


def _scaled(B, m, n, seed0, scale):
    import synth
    probs = [synth.nnls_gaussian(m, n, seed0 + k) for k in range(B)]
    for p in probs:
        p.M = p.M * scale
        p.b = p.b * scale
    return probs


def test_batched_long_backtracking_vs_oracle(lb, orc):
    """A badly scaled A (x1000) needs > 16 Armijo trials in its first
    iteration, so the batched kernel goes through its LS_CONT continuation
    (a second batch of trials) -- the stall path of ADVICE r1; results must
    still match the oracle.  tol = 1e-6 * scale^2 (the gradient scales with
    scale^2; an absolute 1e-6 sits below the fp64 cancellation floor of the
    plain Armijo test at f ~ 1e7, R29)."""
    probs = _scaled(6, 60, 30, 5, 1000.0)
    A = np.stack([p.M for p in probs]); b = np.stack([p.b for p in probs])
    x = torch.zeros(6, 30, dtype=torch.float64, device="cuda")
    res = lb.solve_batched_lsq(lb.colmajor_batch(A), torch.from_numpy(b).cuda(), x,
                               lower=torch.zeros(6, 30, dtype=torch.float64, device="cuda"), tol=1.0)
    for k, p in enumerate(probs):
        first = orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower, opts=orc.Options(max_iters=1))
        assert first.n_backtracks > 16                # the first search alone needs > 16 trials
        ro = orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower, opts=orc.Options(tol=1.0))
        r = res[k]
        assert r.status == ro.status == lb.CONVERGED, (k, r)
        assert r.n_backtracks > 16
        assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f), (k, r.f, ro.f)


def test_batched_fallback_paths_vs_oracle(lb, orc):
    """The R14 fallback in the batched kernel (the FALLBACK stall path of
    ADVICE r1).  max_backtracks = 0 (one Armijo trial per search): on these
    seeds the L-BFGS step is sometimes rejected, the fallback (empty ring,
    steepest descent) is accepted, and the solve converges -- as in the
    oracle.  On a x10-scaled problem with max_backtracks = 3 the very first
    search fails twice (the fallback cannot help with an empty ring):
    LINESEARCH_FAILURE at iteration 0 with one fallback, as in the oracle."""
    seeds = [5, 7, 8, 9]
    import synth
    probs = [synth.nnls_gaussian(60, 30, s) for s in seeds]
    A = np.stack([p.M for p in probs]); b = np.stack([p.b for p in probs])
    x = torch.zeros(len(seeds), 30, dtype=torch.float64, device="cuda")
    res = lb.solve_batched_lsq(lb.colmajor_batch(A), torch.from_numpy(b).cuda(), x,
                               lower=torch.zeros(len(seeds), 30, dtype=torch.float64, device="cuda"),
                               opts=lb.Options(max_backtracks=0))
    nfb = 0
    for k, p in enumerate(probs):
        ro = orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower, opts=orc.Options(max_backtracks=0))
        r = res[k]
        assert r.status == ro.status == lb.CONVERGED, (k, r, ro.status)
        assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
        nfb += r.n_fallbacks
    assert nfb >= 1
    probs = _scaled(3, 60, 30, 5, 10.0)
    A = np.stack([p.M for p in probs]); b = np.stack([p.b for p in probs])
    x = torch.zeros(3, 30, dtype=torch.float64, device="cuda")
    res = lb.solve_batched_lsq(lb.colmajor_batch(A), torch.from_numpy(b).cuda(), x,
                               lower=torch.zeros(3, 30, dtype=torch.float64, device="cuda"),
                               opts=lb.Options(max_backtracks=3, tol=1e-4))
    for k, p in enumerate(probs):
        ro = orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower, opts=orc.Options(max_backtracks=3, tol=1e-4))
        assert ro.status == orc.LINESEARCH_FAILURE and ro.iters == 0 and ro.n_fallbacks == 1
        r = res[k]
        assert r.status == lb.LINESEARCH_FAILURE and r.iters == 0 and r.n_fallbacks == 1, (k, r)


def test_batched_rejects_bad_options_and_bounds(lb):
    A = np.stack([np.eye(4)] * 2); b = np.ones((2, 4))
    M = lb.colmajor_batch(A); bd = torch.from_numpy(b).cuda()
    x = torch.zeros(2, 4, dtype=torch.float64, device="cuda")
    with pytest.raises(lb.LbfgsbError):
        lb.solve_batched_lsq(M, bd, x, opts=lb.Options(c1=1.5))
    with pytest.raises(lb.LbfgsbError):
        lb.solve_batched_lsq(M, bd, x, opts=lb.Options(eps=-1.0))
    lo = torch.zeros(2, 4, dtype=torch.float64, device="cuda")
    up = torch.zeros(2, 4, dtype=torch.float64, device="cuda")
    up[1, 2] = -1.0                                   # l > u
    with pytest.raises(lb.LbfgsbError):
        lb.solve_batched_lsq(M, bd, x, lower=lo, upper=up)
    up[1, 2] = float("nan")
    with pytest.raises(lb.LbfgsbError):
        lb.solve_batched_lsq(M, bd, x, lower=lo, upper=up)
