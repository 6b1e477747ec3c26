"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle
(-m gpu; run on a B200 via gpurun).

Tolerances:
  * elementwise / index / min-max outputs: bit-exact;
  * sums and GEMV outputs: |delta| <= 1e-12 * sum_j |terms_j| (condition-
    normalised reading of the north star's "1e-12 relative");
  * direction d: ||delta d||_inf <= 1e-10 ||d||_inf on well-conditioned pairs;
  * end to end: |f_gpu - f_orc| <= 1e-8 |f_orc|, pg <= 1e-6 on both.
"""
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


def _gemv_bound(A, p):
    return np.abs(A) @ np.abs(p)


# ------------------------------------------------------------------ a1 / a3 GEMVs
@pytest.mark.parametrize("m,n", [(200, 100), (1037, 77), (2050, 1500), (513, 8), (1, 5), (7000, 333),
                                 (30000, 64), (100000, 40), (30001, 37)])
def test_gemv_parity(lb, orc, m, n):
    rng = np.random.default_rng(m * 7 + n)
    A = rng.standard_normal((m, n))
    p = rng.standard_normal(n)
    p[rng.random(n) < 0.4] = 0.0                     # skipped (inactive) columns
    obj = lb.LSQObjective(lb.colmajor(A))
    q = torch.empty(m, dtype=torch.float64, device="cuda")
    lb.op_gemv(obj, _cuda(p), q)
    ref = orc.matvec(A, p)
    assert np.all(np.abs(q.cpu().numpy() - ref) <= 1e-12 * _gemv_bound(A, p) + 1e-300)


@pytest.mark.parametrize("m,n", [(200, 100), (1037, 77), (2050, 1500), (513, 8), (1, 5), (7000, 333),
                                 (30000, 64), (100000, 40), (30001, 37)])
def test_gemvt_parity(lb, orc, m, n):
    rng = np.random.default_rng(m * 11 + n)
    A = rng.standard_normal((m, n))
    r = rng.standard_normal(m)
    obj = lb.LSQObjective(lb.colmajor(A))
    g = torch.empty(n, dtype=torch.float64, device="cuda")
    lb.op_gemvt(obj, _cuda(r), g)
    ref = orc.matvec_t(A, r)
    assert np.all(np.abs(g.cpu().numpy() - ref) <= 1e-12 * (np.abs(A).T @ np.abs(r)))


def test_gemv_split_and_colscale(lb, orc):
    rng = np.random.default_rng(5)
    m, n = 300, 120
    A = rng.standard_normal((m, n))
    w = np.where(rng.random(n) < 0.5, 1.0, -1.0)
    p2 = rng.standard_normal(2 * n)
    # split: M~ = [A, -A]
    obj = lb.LSQObjective(lb.colmajor(A), split=True)
    q = torch.empty(m, dtype=torch.float64, device="cuda")
    lb.op_gemv(obj, _cuda(p2), q)
    pe = p2[:n] - p2[n:]
    assert np.all(np.abs(q.cpu().numpy() - orc.matvec(A, pe)) <= 1e-12 * _gemv_bound(A, pe))
    g = torch.empty(2 * n, dtype=torch.float64, device="cuda")
    r = rng.standard_normal(m)
    lb.op_gemvt(obj, _cuda(r), g)
    gt = orc.matvec_t(A, r)
    gg = g.cpu().numpy()
    assert np.array_equal(gg[:n], -gg[n:])
    assert np.all(np.abs(gg[:n] - gt) <= 1e-12 * (np.abs(A).T @ np.abs(r)))
    # colscale: M~ = A diag(w)
    obj2 = lb.LSQObjective(lb.colmajor(A), colscale=_cuda(w))
    p = rng.standard_normal(n)
    lb.op_gemv(obj2, _cuda(p), q)
    assert np.all(np.abs(q.cpu().numpy() - orc.matvec(A, w * p)) <= 1e-12 * _gemv_bound(A, p))


# ------------------------------------------------------------------ a4 + a5 + a6
def _rand_state(rng, n, nh, box=True):
    l = np.zeros(n) if box else np.full(n, -np.inf)
    u = np.where(rng.random(n) < 0.5, np.inf, 1.0) if box else np.full(n, np.inf)
    x = np.clip(rng.random(n) * 1.5 - 0.25, l, u)
    x[rng.random(n) < 0.2] = 0.0 if box else x[0]
    g = rng.standard_normal(n)
    B = rng.standard_normal((n, 8)) / np.sqrt(n)
    S = [rng.standard_normal(n) for _ in range(nh)]
    Y = [s + 0.1 * (B @ (B.T @ s)) for s in S]        # y = (I + B B^T) s: curvature > 0
    return l, u, x, g, S, Y


@pytest.mark.parametrize("n,nh", [(100, 0), (1000, 0), (37, 3), (1000, 5), (4099, 5), (257, 16)])
def test_direction_parity(lb, orc, n, nh):
    rng = np.random.default_rng(n + nh)
    l, u, x, g, S, Y = _rand_state(rng, n, nh)
    lo, up = _cuda(l), _cuda(u)
    s = lb.Solver(n, max(nh, 1) if nh <= 16 else 16, lower=lo, upper=up)
    out = s.op_direction(_cuda(x), _cuda(g), _cuda(np.array(S)) if nh else None,
                         _cuda(np.array(Y)) if nh else None)
    free = orc.working_set(x, g, l, u, 1e-9)
    assert np.array_equal(out["free"].cpu().numpy(), free)                  # Eq. (1) bit-exact
    d_ref = orc.two_loop(g, free, S, Y, eps=1e-9)
    d = out["d"].cpu().numpy()
    if nh == 0:
        assert np.array_equal(d, d_ref)                                      # d = -g[S] exactly
    else:
        assert np.max(np.abs(d - d_ref)) <= 1e-10 * np.max(np.abs(d_ref))
    assert np.all(d[~free] == 0.0)
    # Alg. 2 on the GPU's own d must equal the oracle's Alg. 2 on that d, bit for bit
    p_ref, br_ref = orc.project_direction(x, g, d, l, u, 1e-9)
    assert out["projected"] == br_ref
    assert np.array_equal(out["p"].cpu().numpy(), p_ref)
    gp_ref = float(np.sum(g * p_ref))
    assert abs(out["gp"] - gp_ref) <= 1e-12 * np.sum(np.abs(g * p_ref))
    if not br_ref:
        assert out["amax"] == orc.max_step(x, p_ref, l, u)                   # min: exact


def test_direction_screen_full_norm(lb, orc):
    rng = np.random.default_rng(77)
    n, nh = 500, 4
    l, u, x, g, S, Y = _rand_state(rng, n, nh)
    Y[1] = -Y[1]                                                             # screened-out pair
    s = lb.Solver(n, 5, lower=_cuda(l), upper=_cuda(u), opts=lb.Options(screen_full_norm=True))
    out = s.op_direction(_cuda(x), _cuda(g), _cuda(np.array(S)), _cuda(np.array(Y)))
    free = orc.working_set(x, g, l, u, 1e-9)
    d_ref = orc.two_loop(g, free, S, Y, eps=1e-9, screen_full_norm=True)
    d = out["d"].cpu().numpy()
    assert np.max(np.abs(d - d_ref)) <= 1e-10 * np.max(np.abs(d_ref))


def test_direction_unbounded_all_free(lb, orc):
    rng = np.random.default_rng(78)
    n = 300
    l, u, x, g, S, Y = _rand_state(rng, n, 3, box=False)
    s = lb.Solver(n, 3)
    out = s.op_direction(_cuda(x), _cuda(g), _cuda(np.array(S)), _cuda(np.array(Y)))
    assert out["free"].all()
    d_ref = orc.two_loop(g, np.ones(n, bool), S, Y, eps=1e-9)
    assert np.max(np.abs(out["d"].cpu().numpy() - d_ref)) <= 1e-10 * np.max(np.abs(d_ref))
    assert out["projected"]


# ------------------------------------------------------------------ a2 trials
def test_trials_parity(lb, orc):
    rng = np.random.default_rng(9)
    m, n = 400, 150
    A = rng.standard_normal((m, n)) / np.sqrt(m)
    b = rng.standard_normal(m)
    c = rng.standard_normal(n) * 0.1
    x = np.abs(rng.standard_normal(n))
    p = rng.standard_normal(n)
    P = orc.LSQ(A, b=b, c=c, delta=0.3)
    r = orc.matvec(A, x) - b
    q = orc.matvec(A, p)
    s = lb.Solver(n, 5, lower=_cuda(np.zeros(n)))
    obj = lb.LSQObjective(lb.colmajor(A), b=_cuda(b), c=_cuda(c), delta=0.3)
    f = s.op_trials(obj, _cuda(r), _cuda(q), _cuda(x), _cuda(p), 1.0, 16)
    a = 1.0
    for t in range(16):
        xt = np.maximum(x + a * p, 0.0)
        rt = r + a * q
        ref = 0.5 * rt @ rt + c @ xt + 0.15 * xt @ xt
        scale = 0.5 * rt @ rt + np.abs(c) @ np.abs(xt) + 0.15 * xt @ xt
        assert abs(f[t] - ref) <= 1e-12 * scale, t
        a *= 0.5


# ------------------------------------------------------------------ end to end (Alg. 1)
def _solve_both(lb, orc, prob, m_hist=5, tol=1e-6, opts=None, oopts=None):
    M = lb.colmajor(prob.M)
    b = None if prob.b is None else _cuda(prob.b)
    c = None if prob.c is None else _cuda(prob.c)
    cs = None if prob.colscale is None else _cuda(prob.colscale)
    obj = lb.LSQObjective(M, b=b, c=c, delta=prob.delta, colscale=cs, split=prob.split)
    lo = None if prob.lower is None else _cuda(prob.lower)
    up = None if prob.upper is None else _cuda(prob.upper)
    s = lb.Solver(prob.nvars, m_hist, lower=lo, upper=up, opts=opts or lb.Options(tol=tol))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    P = orc.LSQ(prob.M, b=prob.b, c=prob.c, delta=prob.delta, colscale=prob.colscale,
                split=prob.split)
    ro = orc.minimize_lsq(P, l=prob.lower, u=prob.upper, m_hist=m_hist,
                          opts=oopts or orc.Options(tol=tol))
    return r, ro, x.cpu().numpy()


@pytest.mark.parametrize("m,n,seed", [(200, 100, 1), (50, 30, 2), (2000, 1000, 3), (999, 1501, 4),
                                      (4000, 2000, 5)])
def test_nnls_end_to_end(lb, orc, m, n, seed):
    import synth
    prob = synth.nnls_gaussian(m, n, seed)
    r, ro, x = _solve_both(lb, orc, prob)
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.pg_inf <= 1e-6 and ro.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    assert np.all(x >= 0.0)                                             # feasible (Thm. 1)


def test_nnls_first_iterations_match_oracle(lb, orc):
    """Trajectory parity: x after k = 1..4 iterations agrees with the oracle."""
    import synth
    prob = synth.nnls_gaussian(300, 120, 21)
    for k in range(1, 5):
        r, ro, x = _solve_both(lb, orc, prob, opts=lb.Options(max_iters=k, tol=1e-12),
                               oopts=orc.Options(max_iters=k, tol=1e-12))
        assert r.iters == ro.iters == k
        assert abs(r.f - ro.f) <= 1e-12 * abs(ro.f)


def test_nnls_first_iterations_match_oracle_kbwd_s(lb, orc):
    """Trajectory parity on the C2 kernels (m = 4000 >= 2048: k_bwd_s, the
    long-column k_fwd): after k = 1..4 iterations f agrees to 1e-12 and x to
    1e-10 of its magnitude (the same decisions step by step)."""
    import synth
    prob = synth.nnls_gaussian(4000, 2000, 22)
    for k in range(1, 5):
        r, ro, x = _solve_both(lb, orc, prob, opts=lb.Options(max_iters=k, tol=1e-12),
                               oopts=orc.Options(max_iters=k, tol=1e-12))
        assert r.iters == ro.iters == k
        assert abs(r.f - ro.f) <= 1e-12 * abs(ro.f)
        xo = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower,
                              opts=orc.Options(max_iters=k, tol=1e-12)).x
        assert np.max(np.abs(x - xo)) <= 1e-10 * max(np.max(np.abs(xo)), 1e-300)


@pytest.mark.parametrize("m,n,seed", [(40000, 2000, 41), (30001, 1203, 42)])
def test_nnls_end_to_end_tall(lb, orc, m, n, seed):
    """C5-shaped columns (m >= 30000: the generic persistent k_bwd and the tall
    k_fwd geometry) end to end against the oracle."""
    import synth
    prob = synth.nnls_gaussian(m, n, seed)
    r, ro, x = _solve_both(lb, orc, prob)
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.pg_inf <= 1e-6 and ro.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    assert np.all(x >= 0.0)


@pytest.mark.parametrize("R,check", [(3, 8), (5, 2), (1, 4)])
def test_periodic_refresh_matches_oracle(lb, orc, R, check):
    """opts.refresh_every (R13's optional refresh: exact r, f, g at the top of
    every R-th iteration) against the oracle's refresh at the same iterations:
    f after k = 1..6 iterations to 1e-12, the converged f to 1e-8; the chunks
    of the replayed graph end at the multiples of R whatever check_every is."""
    import synth
    prob = synth.nnls_gaussian(2000, 1000, 23)
    for k in range(1, 7):
        r, ro, x = _solve_both(lb, orc, prob, opts=lb.Options(max_iters=k, tol=1e-12, refresh_every=R,
                                                              check_every=check),
                               oopts=orc.Options(max_iters=k, tol=1e-12, refresh_every=R))
        assert r.iters == ro.iters == k
        assert abs(r.f - ro.f) <= 1e-12 * abs(ro.f)
    r, ro, x = _solve_both(lb, orc, prob, opts=lb.Options(refresh_every=R, check_every=check),
                           oopts=orc.Options(refresh_every=R))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f) and r.pg_inf <= 1e-6


def test_trials_per_pass_does_not_change_the_trajectory(lb):
    """opts.trials_per_pass moves only the batch boundaries of the Armijo
    trials (the trials are sequential, alpha_t = alpha_0 beta^t by repeated
    multiplication): x is bitwise the same at 1, 3 and 16 trials per pass on a
    x300-scaled NNLS whose searches need several backtracks (so the host
    continuation runs at 1 and 3)."""
    import synth
    p = synth.nnls_gaussian(400, 200, 24)
    M = lb.colmajor(p.M * 300.0)
    obj = lb.LSQObjective(M, b=_cuda(p.b * 300.0))
    out = []
    for tpp in (1, 3, 16):
        s = lb.Solver(p.nvars, 5, lower=_cuda(p.lower), opts=lb.Options(trials_per_pass=tpp, tol=0.09))
        x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
        r = s.solve(obj, x)
        out.append((x.cpu().numpy(), r))
    assert out[0][1].n_backtracks > 0 and out[0][1].status == lb.CONVERGED
    for x, r in out[1:]:
        assert np.array_equal(x, out[0][0]) and r.f == out[0][1].f and r.iters == out[0][1].iters
    with pytest.raises(lb.LbfgsbError):
        lb.Solver(p.nvars, 5, opts=lb.Options(trials_per_pass=17))


def test_determinism_graph_vs_eager(lb):
    """Deterministic reductions: graph replay, eager launches and different
    host-check chunks give bit-identical results."""
    import synth
    prob = synth.nnls_gaussian(3000, 1500, 31)
    M, b = lb.colmajor(prob.M), _cuda(prob.b)
    obj = lb.LSQObjective(M, b=b)
    xs = []
    for opts in (lb.Options(), lb.Options(use_graph=False), lb.Options(check_every=3),
                 lb.Options(check_every=1, use_graph=False)):
        s = lb.Solver(prob.nvars, 5, lower=_cuda(prob.lower), opts=opts)
        x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
        r = s.solve(obj, x)
        xs.append((x.cpu().numpy(), r.f, r.iters))
    for x, f, it in xs[1:]:
        assert np.array_equal(x, xs[0][0]) and f == xs[0][1] and it == xs[0][2]


def test_edge_cases(lb, orc):
    import synth
    # all variables fixed at x0 = 0: b anti-correlated with every column -> S empty, 0 iterations
    rng = np.random.default_rng(3)
    A = np.abs(rng.standard_normal((50, 20)))
    b = -np.ones(50)
    obj = lb.LSQObjective(lb.colmajor(A), b=_cuda(b))
    s = lb.Solver(20, 5, lower=_cuda(np.zeros(20)))
    x = torch.zeros(20, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    assert r.iters == 0 and r.status == lb.CONVERGED and r.n_free == 0
    assert torch.all(x == 0)
    # n = 1
    prob = synth.nnls_gaussian(5, 1, 4)
    r, ro, _ = _solve_both(lb, orc, prob)
    assert abs(r.f - ro.f) <= 1e-12 * abs(ro.f)
    # unbounded: plain L-BFGS on a least-squares problem equals the normal equations
    A = rng.standard_normal((60, 25))
    b = rng.standard_normal(60)
    obj = lb.LSQObjective(lb.colmajor(A), b=_cuda(b))
    s = lb.Solver(25, 5, opts=lb.Options(tol=1e-10))
    x = torch.zeros(25, dtype=torch.float64, device="cuda")
    s.solve(obj, x)
    assert np.allclose(x.cpu().numpy(), np.linalg.lstsq(A, b, rcond=None)[0], atol=1e-8)
    # max_iters = 0 returns x0 clipped
    s = lb.Solver(25, 5, lower=_cuda(np.zeros(25)), opts=lb.Options(max_iters=0))
    x = _cuda(rng.standard_normal(25))
    r = s.solve(obj, x)
    assert r.iters == 0 and r.status == lb.MAX_ITERS and torch.all(x >= 0)
    # two-sided box with odd m (scalar path of the GEMVs)
    A = rng.standard_normal((101, 40))
    b = rng.standard_normal(101) * 3
    prob = synth.Problem("nnls", "box", A, b=b, lower=-np.ones(40) * 0.1, upper=np.ones(40) * 0.2)
    r, ro, x = _solve_both(lb, orc, prob)
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f) and r.pg_inf <= 1e-6
    assert np.all(x >= -0.1) and np.all(x <= 0.2)


def test_bad_bounds_rejected(lb):
    with pytest.raises(lb.LbfgsbError):
        lb.Solver(3, 5, lower=_cuda(np.array([0.0, 1.0, 0.0])), upper=_cuda(np.array([1.0, 0.0, 1.0])))


@pytest.mark.parametrize("alpha", [1.0, 0.5])
def test_lasso_split_end_to_end(lb, orc, alpha):
    import synth
    prob = synth.lasso_split(400, 1000, 7, alpha=alpha)
    r, ro, x = _solve_both(lb, orc, prob)
    assert r.pg_inf <= 1e-6 and ro.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    n = prob.ncols
    assert np.max(x[:n] * x[n:]) <= 1e-12


def test_callback_objective(lb, orc):
    """User objective through lbfgsb_objective_callback (f/grad on the device)."""
    import synth
    prob = synth.nnls_gaussian(300, 150, 12)
    A = torch.from_numpy(prob.M.copy()).cuda()
    b = _cuda(prob.b)

    def fg(x, g):
        r = A @ x - b
        g.copy_(A.T @ r)
        return 0.5 * float(r @ r)

    obj = lb.CallbackObjective(fg, prob.nvars)
    s = lb.Solver(prob.nvars, 5, lower=_cuda(prob.lower))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
    assert r.status == lb.CONVERGED and r.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)


# ------------------------------------------------------------------ Alg. 4 (AL)
def test_al_simplex(lb, orc):
    rng = np.random.default_rng(40)
    n = 50
    c = rng.standard_normal(n) * 0.5
    obj = lb.LSQObjective(lb.colmajor(np.eye(n)), b=_cuda(c))
    s = lb.Solver(n, 5, lower=_cuda(np.zeros(n)), opts=lb.Options(tol=1e-9))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, E=_cuda(np.ones((n, 1))), e=[1.0])
    ro = orc.al_solve(orc.LSQ(np.eye(n), b=c, E=np.ones((n, 1)), e=[1.0]), l=np.zeros(n),
                      opts=orc.Options(tol=1e-9))
    assert r.status == lb.CONVERGED
    assert np.allclose(x.cpu().numpy(), ro.x, atol=1e-7)
    assert abs(r.lam[0] - ro.lam[0]) <= 1e-6 * max(1, abs(ro.lam[0]))


def test_al_inequality(lb, orc):
    rng = np.random.default_rng(41)
    n = 40
    c = rng.standard_normal(n) * 0.6
    obj = lb.LSQObjective(lb.colmajor(np.eye(n)), b=_cuda(c))
    s = lb.Solver(n, 5, lower=_cuda(np.zeros(n)), opts=lb.Options(tol=1e-9))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, G=_cuda(np.ones((n, 1))), hv=[1.0])
    ro = orc.al_solve(orc.LSQ(np.eye(n), b=c, G=np.ones((n, 1)), hv=[1.0]), l=np.zeros(n),
                      opts=orc.Options(tol=1e-9))
    assert np.allclose(x.cpu().numpy(), ro.x, atol=1e-7)
    assert r.mu[0] >= 0


def test_svm_dual_al(lb, orc):
    import synth
    prob = synth.svm_dual_linear(2000, 20, 42)
    M = lb.colmajor(prob.M)
    obj = lb.LSQObjective(M, c=_cuda(prob.c), colscale=_cuda(prob.colscale))
    s = lb.Solver(prob.nvars, 5, lower=_cuda(prob.lower), upper=_cuda(prob.upper),
                  opts=lb.Options(tol=1e-6))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.al_solve(obj, x, E=_cuda(prob.E), e=prob.e)
    P = orc.LSQ(prob.M, c=prob.c, colscale=prob.colscale, E=prob.E, e=prob.e)
    ro = orc.al_solve(P, l=prob.lower, u=prob.upper, opts=orc.Options(tol=1e-6))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.violation_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-6 * abs(ro.f)
    a = x.cpu().numpy()
    assert np.all(a >= 0) and np.all(a <= 1.0)


# ------------------------------------------------------------------ full size (bench config)
@pytest.mark.slow
def test_c2_full_size_sampled_kkt(lb, orc):
    """BASELINE configs[1] (20000 x 10000) in the bench's launch configuration:
    the KKT residual is re-derived on the host for 200 sampled coordinates
    from r = A x - b computed by the oracle's matvec."""
    import synth
    prob = synth.CONFIGS["C2"]()
    M = lb.colmajor(prob.M)
    obj = lb.LSQObjective(M, b=_cuda(prob.b))
    s = lb.Solver(prob.nvars, 5, lower=_cuda(prob.lower))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    assert r.status == lb.CONVERGED and r.pg_inf <= 1e-6
    xh = x.cpu().numpy()
    assert np.all(xh >= 0)
    res = orc.matvec(prob.M, xh) - prob.b
    f = 0.5 * res @ res
    assert abs(r.f - f) <= 1e-10 * f
    idx = np.random.default_rng(0).choice(prob.nvars, 200, replace=False)
    gs = np.array([prob.M[:, j] @ res for j in idx])
    pg = np.abs(np.maximum(xh[idx] - gs, 0.0) - xh[idx])
    assert np.max(pg) <= 2e-6
