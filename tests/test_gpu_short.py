"""Short-column backward GEMV variants against the CPU oracle (-m gpu), and the
split / colscale forms of the long-column k_bwd_s.

m < 2048 rows selects the short-column kernels (bwd.cu launch_bwd):
  * k_bwd_wo when a CTA owns >= 64 columns (C4's 1000 x 100000 operator):
    dynamic 4-column units per warp, the epilogue in 32-column mini-tiles run
    by the warp that completes them, Gram partials summed in mini-tile order;
  * k_bwd_wd below that (C1).
The unit -> warp and mini-tile -> warp assignments are dynamic (shared-memory
counters), so besides oracle parity these tests check that the results are
bitwise reproducible run to run.  Tolerances are those of test_gpu_parity.py
(DESIGN.md section 6)."""
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


def _solve(lb, prob, opts=None, m_hist=5):
    M = lb.colmajor(prob.M)
    b = None if prob.b is None else _cuda(prob.b)
    c = None if prob.c is None else _cuda(prob.c)
    cs = None if prob.colscale is None else _cuda(prob.colscale)
    obj = lb.LSQObjective(M, b=b, c=c, delta=prob.delta, colscale=cs, split=prob.split)
    lo = None if prob.lower is None else _cuda(prob.lower)
    up = None if prob.upper is None else _cuda(prob.upper)
    s = lb.Solver(prob.nvars, m_hist, lower=lo, upper=up, opts=opts or lb.Options())
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    return r, x.cpu().numpy()


def _nnls_pos(m, n, seed):
    """Box-constrained LSQ 0 <= x <= 0.05 on the NNLS Gaussian data: with n >> m
    the plain NNLS fits b exactly (f* = 0, where a relative f test is void); the
    upper bound keeps f* > 0 and puts variables on both bounds."""
    import synth
    prob = synth.nnls_gaussian(m, n, seed)
    prob.upper = np.full(n, 0.05)
    return prob


def _oracle(orc, prob, opts=None, m_hist=5):
    P = orc.LSQ(prob.M, b=prob.b, c=prob.c, delta=prob.delta, colscale=prob.colscale, split=prob.split)
    return orc.minimize_lsq(P, l=prob.lower, u=prob.upper, m_hist=m_hist, opts=opts or orc.Options())


@pytest.mark.parametrize("m,n", [(1000, 30000), (999, 25001), (63, 40000), (2047, 20000)])
def test_gemvt_parity_short_columns(lb, orc, m, n):
    """g = M^T r (BWD_PLAIN through k_bwd_wo) element by element, ragged m and n."""
    rng = np.random.default_rng(m + 3 * n)
    A = rng.standard_normal((m, n))
    r = rng.standard_normal(m)
    obj = lb.LSQObjective(lb.colmajor(A))
    g = torch.empty(n, dtype=torch.float64, device="cuda")
    lb.op_gemvt(obj, _cuda(r), g)
    ref = orc.matvec_t(A, r)
    assert np.all(np.abs(g.cpu().numpy() - ref) <= 1e-12 * (np.abs(A).T @ np.abs(r)))


def test_gemvt_short_columns_split_and_colscale(lb, orc):
    rng = np.random.default_rng(77)
    m, n = 700, 26000
    A = rng.standard_normal((m, n))
    r = rng.standard_normal(m)
    bound = np.abs(A).T @ np.abs(r)
    gt = orc.matvec_t(A, r)
    obj = lb.LSQObjective(lb.colmajor(A), split=True)
    g = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    lb.op_gemvt(obj, _cuda(r), g)
    gg = g.cpu().numpy()
    assert np.array_equal(gg[:n], -gg[n:])
    assert np.all(np.abs(gg[:n] - gt) <= 1e-12 * bound)
    w = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    obj2 = lb.LSQObjective(lb.colmajor(A), colscale=_cuda(w))
    g2 = torch.empty(n, dtype=torch.float64, device="cuda")
    lb.op_gemvt(obj2, _cuda(r), g2)
    assert np.all(np.abs(g2.cpu().numpy() - w * gt) <= 1e-12 * bound)


@pytest.mark.parametrize("m,n,seed", [(700, 40000, 61), (1000, 30011, 62)])
def test_nnls_end_to_end_short_columns(lb, orc, m, n, seed):
    prob = _nnls_pos(m, n, seed)
    r, x = _solve(lb, prob)
    ro = _oracle(orc, prob)
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.pg_inf <= 1e-6 and ro.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    assert np.all(x >= 0.0)


def test_first_iterations_match_oracle_short_columns(lb, orc):
    """Trajectory parity on k_bwd_wo (1000 x 30000): f to 1e-12 and x to 1e-10
    of its magnitude after k = 1..4 iterations."""
    prob = _nnls_pos(1000, 30000, 63)
    for k in range(1, 5):
        r, x = _solve(lb, prob, opts=lb.Options(max_iters=k, tol=1e-12))
        ro = _oracle(orc, prob, opts=orc.Options(max_iters=k, tol=1e-12))
        assert r.iters == ro.iters == k
        assert abs(r.f - ro.f) <= 1e-12 * abs(ro.f)
        assert np.max(np.abs(x - ro.x)) <= 1e-10 * max(np.max(np.abs(ro.x)), 1e-300)


def test_lasso_split_short_columns(lb, orc):
    """Split operator [A, -A] on k_bwd_wo (both halves of a mini-tile's columns):
    the first 10 iterations against the oracle's (a full lasso solve takes the
    oracle minutes at this size)."""
    import synth
    prob = synth.lasso_split(400, 20000, 64)
    r, x = _solve(lb, prob, opts=lb.Options(max_iters=10, tol=1e-12))
    ro = _oracle(orc, prob, opts=orc.Options(max_iters=10, tol=1e-12))
    assert r.iters == ro.iters == 10
    assert abs(r.f - ro.f) <= 1e-10 * abs(ro.f)
    assert np.max(np.abs(x - ro.x)) <= 1e-8 * max(np.max(np.abs(ro.x)), 1e-300)
    n = prob.ncols
    assert np.max(x[:n] * x[n:]) <= 1e-12


@pytest.mark.parametrize("m_hist", [1, 5, 9])
def test_short_columns_bitwise_reproducible(lb, m_hist):
    """Dynamic unit / mini-tile scheduling: repeated solves (graph and eager,
    history lengths whose Gram entries span one to four per-lane registers and
    beyond) are bitwise identical."""
    import synth
    prob = synth.nnls_gaussian(800, 33000, 65)
    out = []
    for opts in (lb.Options(), lb.Options(), lb.Options(use_graph=False)):
        r, x = _solve(lb, prob, opts=opts, m_hist=m_hist)
        out.append((x, r.f, r.iters))
    for x, f, it in out[1:]:
        assert np.array_equal(x, out[0][0]) and f == out[0][1] and it == out[0][2]


@pytest.mark.parametrize("m,n", [(16, 2_000_000), (16, 6_500_000)])
def test_short_column_fallbacks(lb, orc, m, n):
    """Very many short columns: the mini-tile partials of k_bwd_wo no longer fit
    shared memory (2 M columns: k_bwd_wd), then neither do k_bwd_wd's column
    dots (6.5 M columns: k_bwd_w, round 1's per-warp-epilogue kernel).  GEMV^T
    element by element, and the first 3 iterations against the oracle."""
    import synth
    rng = np.random.default_rng(m + n)
    A = np.asfortranarray(rng.standard_normal((m, n)) / np.sqrt(m))
    r = rng.standard_normal(m)
    obj = lb.LSQObjective(lb.colmajor(A))
    g = torch.empty(n, dtype=torch.float64, device="cuda")
    lb.op_gemvt(obj, _cuda(r), g)
    assert np.all(np.abs(g.cpu().numpy() - orc.matvec_t(A, r)) <= 1e-12 * (np.abs(A).T @ np.abs(r)))
    prob = synth.Problem("nnls", "fallback", A, b=rng.standard_normal(m), lower=np.zeros(n),
                         upper=np.full(n, 0.05))
    r3, x = _solve(lb, prob, opts=lb.Options(max_iters=3, tol=1e-12))
    ro = _oracle(orc, prob, opts=orc.Options(max_iters=3, tol=1e-12))
    assert r3.iters == ro.iters == 3
    # f falls by ~10 orders of magnitude in 3 steps here (16 rows, millions of columns): its rounding
    # floor is that of the carried residual, eps * f(x0) = eps * ||b||^2 / 2, so compare on that scale
    f0 = 0.5 * float(prob.b @ prob.b)
    assert abs(r3.f - ro.f) <= 1e-12 * f0
    assert np.max(np.abs(x - ro.x)) <= 1e-10 * max(np.max(np.abs(ro.x)), 1e-300)


@pytest.mark.parametrize("P", [2, 4])
def test_sharded_loopback_short_columns(lb, orc, P):
    """Column sharding on the short-column kernel (>= 64 columns per CTA in every shard: k_bwd_wo, whose
    Gram tail then writes the sharded pack): P logical ranks with the P2P exchange equal the copy exchange
    bitwise, and reach the oracle's optimum."""
    from test_gpu_sharded import _gather_x, _shards
    prob = _nnls_pos(700, 80000, 66)
    out = []
    for p2p in (False, True):
        sv, ob, xs, keep = _shards(lb, prob, P)
        if p2p:
            lb.p2p_connect_local(sv, prob.M.shape[0])
        r = lb.solve_loopback(sv, ob, xs)
        out.append((r, _gather_x(prob, P, xs)))
    (r0, x0), (r1, x1) = out
    assert r1.status == lb.CONVERGED and r1.pg_inf <= 1e-6
    assert np.array_equal(x0, x1) and r0.f == r1.f and r0.iters == r1.iters
    ro = _oracle(orc, prob)
    assert ro.pg_inf <= 1e-6
    # 80000 columns under the 0.05 bound still fit b almost exactly (f* ~ 1e-11): compare f on the scale of
    # its rounding floor, that of the carried residual, eps * f(x0) = eps * ||b||^2 / 2
    assert abs(r1.f - ro.f) <= 1e-12 * 0.5 * float(prob.b @ prob.b)


# ---- the long-column k_bwd_s (m >= 2048) with the split and colscale operators (C3 / SVM forms)
def test_gemvt_kbwd_s_split_and_colscale(lb, orc):
    rng = np.random.default_rng(91)
    m, n = 3000, 5001
    A = rng.standard_normal((m, n))
    r = rng.standard_normal(m)
    bound = np.abs(A).T @ np.abs(r)
    gt = orc.matvec_t(A, r)
    g = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    lb.op_gemvt(lb.LSQObjective(lb.colmajor(A), split=True), _cuda(r), g)
    gg = g.cpu().numpy()
    assert np.array_equal(gg[:n], -gg[n:])
    assert np.all(np.abs(gg[:n] - gt) <= 1e-12 * bound)
    w = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    g2 = torch.empty(n, dtype=torch.float64, device="cuda")
    lb.op_gemvt(lb.LSQObjective(lb.colmajor(A), colscale=_cuda(w)), _cuda(r), g2)
    assert np.all(np.abs(g2.cpu().numpy() - w * gt) <= 1e-12 * bound)


def test_lasso_split_kbwd_s_first_iterations(lb, orc):
    """The C3 form on k_bwd_s: a split operator whose CTAs own 2 x 135 variables (two epilogue tiles);
    10 iterations against the oracle's."""
    import synth
    prob = synth.lasso_split(3000, 20000, 92)
    r, x = _solve(lb, prob, opts=lb.Options(max_iters=10, tol=1e-12))
    ro = _oracle(orc, prob, opts=orc.Options(max_iters=10, tol=1e-12))
    assert r.iters == ro.iters == 10
    assert abs(r.f - ro.f) <= 1e-10 * abs(ro.f)
    assert np.max(np.abs(x - ro.x)) <= 1e-8 * max(np.max(np.abs(ro.x)), 1e-300)
    n = prob.ncols
    assert np.max(x[:n] * x[n:]) <= 1e-12


def test_svm_dual_al_short_columns(lb, orc):
    """The C4 form (linear-SVM dual: colscale = y, 0 <= a <= C, y^T a = 0 through Alg. 4) on k_bwd_wo:
    20000 samples, so the fused AL path's epilogue (ccoef E_k terms) runs in the mini-tiles."""
    import synth
    prob = synth.svm_dual_linear(20000, 20, 93)
    M = lb.colmajor(prob.M)
    obj = lb.LSQObjective(M, c=_cuda(prob.c), colscale=_cuda(prob.colscale))
    s = lb.Solver(prob.nvars, 5, lower=_cuda(prob.lower), upper=_cuda(prob.upper), opts=lb.Options(tol=1e-6))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, E=_cuda(prob.E), e=prob.e)
    P = orc.LSQ(prob.M, c=prob.c, colscale=prob.colscale, E=prob.E, e=prob.e)
    ro = orc.al_solve(P, l=prob.lower, u=prob.upper, opts=orc.Options(tol=1e-6))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.violation_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-6 * abs(ro.f)
    a = x.cpu().numpy()
    assert np.all(a >= 0) and np.all(a <= 1.0)
