"""GPU parity of the original L-BFGS-B's generalized Cauchy point (SURVEY 8(f)
N3, the baseline of PAPER.md:436-457) through lbfgsb_op_cauchy_point against
the oracle's Algorithm CP on the same seeded inputs (-m gpu)."""
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


def _case(n, h, seed, inf_frac=0.2):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(n)
    l = x - rng.uniform(0.0, 1.5, n)
    u = x + rng.uniform(0.0, 1.5, n)
    l[rng.random(n) < inf_frac] = -np.inf
    u[rng.random(n) < inf_frac] = np.inf
    at = (rng.random(n) < 0.2) & np.isfinite(l)
    x[at] = l[at]
    g = rng.standard_normal(n)
    S = rng.standard_normal((h, n)) / np.sqrt(n)
    Y = S + 0.3 * rng.standard_normal((h, n)) / np.sqrt(n)     # s^T y > 0 w.h.p.
    for i in range(h):
        if S[i] @ Y[i] <= 0:
            Y[i] = S[i]
    theta = float(Y[-1] @ Y[-1] / (S[-1] @ Y[-1])) if h else 1.0
    return x, g, l, u, S, Y, theta


@pytest.mark.parametrize("n,h,seed", [(1, 0, 1), (7, 2, 2), (1000, 0, 3), (1000, 3, 4), (5000, 5, 5),
                                      (20000, 5, 6), (12801, 4, 7)])
def test_cauchy_point_parity(lb, orc, n, h, seed):
    x, g, l, u, S, Y, theta = _case(n, h, seed)
    s = lb.Solver(n, 5, lower=_cuda(l), upper=_cuda(u))
    r = s.op_cauchy_point(_cuda(x), _cuda(g), _cuda(S) if h else None, _cuda(Y) if h else None, theta)
    xo, co, po = orc.cauchy_point(x, g, l, u, S if h else None, Y if h else None, theta)
    assert r["passed"] == po                       # integer trip count decided identically
    xg = r["xcp"].cpu().numpy()
    assert np.allclose(xg, xo, rtol=1e-10, atol=1e-12)
    if h:
        assert np.allclose(r["c"], co, rtol=1e-9, atol=1e-12)
    assert r["scan_ms"] >= 0.0


def test_cauchy_point_ties_by_index(lb, orc):
    """Equal breakpoints are passed in index order on both sides."""
    n = 64
    x = np.zeros(n); g = -np.ones(n); u = np.full(n, 0.5); l = np.full(n, -1.0)
    s = lb.Solver(n, 5, lower=_cuda(l), upper=_cuda(u))
    r = s.op_cauchy_point(_cuda(x), _cuda(g), None, None, 1e-3)
    xo, _, po = orc.cauchy_point(x, g, l, u, None, None, 1e-3)
    assert r["passed"] == po == n
    assert np.array_equal(r["xcp"].cpu().numpy(), xo)
