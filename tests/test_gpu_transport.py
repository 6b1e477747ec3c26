"""GPU parity of the joint-probability / regularised-OT path (SURVEY 8(f) N2,
PAPER.md:393-402) through the C ABI (al_solve_transport) against the CPU
oracle on the same seeded inputs, plus at larger sizes against the Sinkhorn
scaling (entropy) computed with plain torch ops in the test (-m gpu)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

LENT = 1e-300   # entropy lower bound (reading R30)


@pytest.fixture(scope="module")
def lb():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2203_16340_b200 as lb
    lb.load()
    return lb


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _gpu(lb, M, u, v, reg, lam, tol, max_outer=100, eps=1e-9):
    m, n = M.shape
    Md = _cuda(np.asfortranarray(M).reshape(-1, order="F")).reshape(n, m).T   # (m, n) column-major
    obj = lb.TransportObjective(Md, reg, lam)
    lo = torch.full((m * n,), LENT if reg == "entropy" else 0.0, dtype=torch.float64, device="cuda")
    s = lb.Solver(m * n, 5, lower=lo, opts=lb.Options(tol=tol, max_iters=200000, eps=eps))
    x = torch.zeros(m * n, dtype=torch.float64, device="cuda")
    lam_out = torch.zeros(m + n, dtype=torch.float64, device="cuda")
    r = s.al_solve_transport(obj, x, _cuda(u), _cuda(v), lam_out=lam_out,
                             al_opts=lb.ALOptions(feas_tol=tol, max_outer=max_outer))
    return r, x.cpu().numpy().reshape(m, n, order="F"), lam_out.cpu().numpy()


def _orc(orc, M, u, v, reg, lam, tol):
    m, n = M.shape
    P = orc.LSQ.transport(M, u, v, reg, lam)
    r = orc.al_solve(P, l=np.full(m * n, LENT if reg == "entropy" else 0.0),
                     opts=orc.Options(tol=tol, armijo_diff=True, max_iters=200000),
                     al_opts=orc.ALOptions(feas_tol=tol))
    return r, r.x.reshape(m, n, order="F")


def _rand(m, n, seed):
    rng = np.random.default_rng(seed)
    M = rng.uniform(size=(m, n))
    u = rng.uniform(size=m); u /= u.sum(); v = rng.uniform(size=n); v /= v.sum()
    return M, u, v


CASES = [("ds2", 20, None), ("ds1", 24, None), ("rand", 270, 21), ("rand", 17, 40), ("rand", 1, 7)]


@pytest.mark.parametrize("reg", ["entropy", "gaussian"])
@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}{c[1]}x{c[2]}")
def test_transport_parity(lb, orc, reg, case):
    import synth
    kind, a, b = case
    if kind == "ds2":
        t = synth.transport_ds2(a, 5); M, u, v = t.cost, t.u, t.v
    elif kind == "ds1":
        t = synth.transport_ds1(a); M, u, v = t.cost, t.u, t.v
    else:
        M, u, v = _rand(a, b, a * 100 + b)
    tol = 1e-9
    r, X, lamg = _gpu(lb, M, u, v, reg, 0.5, tol)
    ro, Xo = _orc(orc, M, u, v, reg, 0.5, tol)
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED, (r, ro.status)
    assert r.violation_inf <= tol
    # both sides stop at ||g[S]||_inf <= tol; the AL objective is lam-strongly
    # convex in the Gaussian case, so each x* is within tol / lam of the exact one
    scale = np.abs(Xo).max()
    assert np.max(np.abs(X - Xo)) <= 1e-7 * scale + 4 * tol / 0.5
    assert abs(r.f - ro.f) <= 1e-9 * max(abs(ro.f), 1.0)
    assert np.all(X >= 0)
    assert np.allclose(X.sum(1), u, atol=2 * tol) and np.allclose(X.sum(0), v, atol=2 * tol)


def _sinkhorn_torch(M, u, v, lam, iters=5000):
    K = torch.exp(-M / lam)
    a = torch.ones_like(u); b = torch.ones_like(v)
    for _ in range(iters):
        a = u / (K @ b)
        b = v / (K.T @ a)
    return a[:, None] * K * b[None, :]


@pytest.mark.parametrize("n,tol,prel", [(200, 1e-9, 1e-6), (400, 1e-8, 2e-5), (1000, 2e-6, 3e-3)])
def test_entropy_ds2_vs_sinkhorn(lb, n, tol, prel):
    """Full-scale invariants: the entropic optimum is the Sinkhorn scaling of
    exp(-M / lam) for any cost (stationarity with P > 0); DS2 n = 1000 is
    2 * 10^6 variables and 3000 constraints.  At n = 1000 the
    smallest marginals are ~1e-7, so the multiplier iteration of Alg. 4
    contracts by ~1 / (1 + rho u_min / lam) per outer step and rho ~ 5e5 makes
    the inner problems stiff: the test runs at tol = feas_tol = 2e-6
    (N2 notes).  The epsilon of Eq. (1) must sit below the scale of
    the entries (~1e-11 in the smallest rows): eps = 1e-20 (reading R30).
    The optimum is strictly interior: every entry must end above the R30
    lower bound 1e-300 with |gradient| <= 2 tol (no entry may sit on the
    bound), and P agrees with Sinkhorn to `prel` of max P (measured on B200:
    8.6e-11 / 3.0e-5 at n = 400, tol 1e-8; 5.3e-9 / 4.7e-6 at n = 1000, tol 2e-6)."""
    import synth
    t = synth.transport_ds2(n, 9)
    r, X, lamg = _gpu(lb, t.cost, t.u, t.v, "entropy", t.lam, tol, max_outer=60, eps=1e-20)
    assert r.status == lb.CONVERGED, r
    assert np.allclose(X.sum(1), t.u, atol=2 * tol) and np.allclose(X.sum(0), t.v, atol=2 * tol)
    # stationarity of the inner problem with the updated multipliers (Alg. 4 line 6):
    # |M + lam (log P + 1) + l_i + l_{m+j}| <= tol on EVERY entry (all entries are free)
    m = t.m
    assert np.all(X > 1e-290)
    G = t.cost + t.lam * (np.log(X) + 1.0) + lamg[:m, None] + lamg[None, m:]
    assert np.max(np.abs(G)) <= 2 * tol
    Ps = _sinkhorn_torch(_cuda(t.cost), _cuda(t.u), _cuda(t.v), t.lam, iters=20000).cpu().numpy()
    assert np.max(np.abs(X - Ps)) <= prel * Ps.max()
    fstar = float(np.sum(t.cost * Ps) + t.lam * np.sum(Ps * np.log(Ps)))
    # f at a point with marginal residual h is f* - lam^T h to first order (KKT of the
    # equality-constrained problem): bound |f - f*| by 2 |lam|^T |h| (+ rounding)
    h = np.concatenate([X.sum(1) - t.u, X.sum(0) - t.v])
    assert abs(r.f - fstar) <= 2.0 * float(np.abs(lamg) @ np.abs(h)) + 1e-9 * abs(fstar)


def test_gaussian_ds1_kkt(lb):
    """Gaussian regulariser at DS1 n = 500 (250000 variables): KKT of the
    original problem from the returned multipliers: P = (-(M + l_i + l_j))_+ / lam
    (stationarity of Eq. (3) at the inner optimum, with the multipliers after
    the update of Alg. 4 line 6), marginals within feas_tol."""
    import synth
    t = synth.transport_ds1(500)
    tol = 1e-9
    r, X, lamg = _gpu(lb, t.cost, t.u, t.v, "gaussian", t.lam, tol)
    assert r.status == lb.CONVERGED
    assert np.allclose(X.sum(1), t.u, atol=2 * tol) and np.allclose(X.sum(0), t.v, atol=2 * tol)
    m = t.m
    Z = -(t.cost + lamg[:m, None] + lamg[None, m:]) / t.lam
    # |g_ij| <= tol on free entries with g = M + lam P + lambda_i + lambda_j
    assert np.max(np.abs(X - np.maximum(Z, 0.0))) <= 4 * tol / t.lam
