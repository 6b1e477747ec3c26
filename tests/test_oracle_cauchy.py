"""Pins of the oracle's generalized Cauchy point: Algorithm CP
of the original L-BFGS-B (Byrd, Lu, Nocedal, Zhu 1995), the sequential step the
paper removes.

Pinned against what the definition fixes, not against the formulas of the
algorithm:
  * the compact form B = theta I - W M W^T equals the dense BFGS recursion
    B <- B - B s s^T B / (s^T B s) + y y^T / (y^T s) started from theta I;
  * the Cauchy point is the FIRST local minimiser of the quadratic model
    m(x) = g^T (x - x0) + 1/2 (x - x0)^T B (x - x0) along the projected
    gradient path x(t) = P(x0 - t g), found here by walking the path's linear
    segments with the dense B (no breakpoint recurrences);
  * c = W^T (x_cp - x0)."""
import numpy as np
import pytest


def _pairs(rng, n, h):
    S, Y = [], []
    while len(S) < h:
        s = rng.standard_normal(n)
        A = rng.standard_normal((n, n)); A = A @ A.T + 0.5 * np.eye(n)
        y = A @ s
        if s @ y > 1e-3:
            S.append(s); Y.append(y)
    return np.array(S).reshape(h, n), np.array(Y).reshape(h, n)


def _dense_bfgs(S, Y, theta, n):
    B = theta * np.eye(n)
    for s, y in zip(S, Y):
        Bs = B @ s
        B = B - np.outer(Bs, Bs) / (s @ Bs) + np.outer(y, y) / (y @ s)
    return B


def _gcp_bruteforce(x, g, l, u, B):
    """First local minimiser of the model along P(x - t g), segment by segment."""
    n = len(x)
    t_i = np.full(n, np.inf)
    for i in range(n):
        if g[i] < 0 and np.isfinite(u[i]):
            t_i[i] = (x[i] - u[i]) / g[i]
        elif g[i] > 0 and np.isfinite(l[i]):
            t_i[i] = (x[i] - l[i]) / g[i]
    bps = np.unique(np.r_[0.0, t_i[np.isfinite(t_i) & (t_i > 0)]])
    bps = np.r_[bps, np.inf]
    xt = lambda t: np.clip(x - t * g, l, u)
    for a, b in zip(bps[:-1], bps[1:]):
        xa = xt(a)
        dseg = np.where(t_i > a, -g, 0.0)                  # components still moving on (a, b)
        z = xa - x
        mp = g @ dseg + dseg @ B @ z                        # m'(a+)
        curv = dseg @ B @ dseg
        if mp >= 0:
            return xa
        if curv > 0:
            tau = a - mp / curv
            if tau < b:
                return xt(tau) if np.isfinite(b) else xa + (tau - a) * dseg
    raise AssertionError("model unbounded along the path")


@pytest.mark.parametrize("h", [1, 2, 3])
def test_compact_form_equals_bfgs(orc, h):
    rng = np.random.default_rng(h)
    n = 7
    S, Y = _pairs(rng, n, h)
    theta = float(Y[-1] @ Y[-1] / (S[-1] @ Y[-1]))
    M = orc.compact_m(S, Y, theta)
    W = np.hstack([Y.T, theta * S.T])
    B = theta * np.eye(n) - W @ M @ W.T
    assert np.allclose(B, _dense_bfgs(S, Y, theta, n), rtol=1e-9, atol=1e-9)


@pytest.mark.parametrize("seed", range(60))
def test_cauchy_point_first_local_min(orc, seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(1, 9))
    h = int(rng.integers(0, 4))
    x = rng.standard_normal(n)
    l = x - rng.uniform(0.0, 1.5, n)
    u = x + rng.uniform(0.0, 1.5, n)
    l[rng.random(n) < 0.2] = -np.inf
    u[rng.random(n) < 0.2] = np.inf
    at_l = rng.random(n) < 0.2
    x[at_l] = l[at_l] = np.where(np.isfinite(l[at_l]), l[at_l], x[at_l])
    g = rng.standard_normal(n) * 2.0
    if h:
        S, Y = _pairs(rng, n, h)
        theta = float(Y[-1] @ Y[-1] / (S[-1] @ Y[-1]))
    else:
        S = Y = None
        theta = float(rng.uniform(0.3, 3.0))
    B = _dense_bfgs(S if h else [], Y if h else [], theta, n)
    want = _gcp_bruteforce(x, g, l, u, B)
    xcp, c, passed = orc.cauchy_point(x, g, l, u, S, Y, theta)
    assert np.allclose(xcp, want, rtol=1e-9, atol=1e-9), (xcp, want)
    assert np.all(xcp >= l - 1e-15) and np.all(xcp <= u + 1e-15)
    if h:
        W = np.hstack([Y.T, theta * S.T])
        assert np.allclose(c, W.T @ (xcp - x), rtol=1e-9, atol=1e-9)
    # the model decreases from x0
    z = xcp - x
    assert g @ z + 0.5 * z @ B @ z <= 1e-12


def test_cauchy_point_passes_breakpoints_in_order(orc):
    """theta small (flat model): the path runs through every breakpoint."""
    n = 50
    rng = np.random.default_rng(7)
    x = np.zeros(n); g = -rng.uniform(0.5, 2.0, n)
    u = rng.uniform(0.1, 1.0, n); l = np.full(n, -1.0)
    xcp, _, passed = orc.cauchy_point(x, g, l, u, None, None, 1e-6)
    assert passed == n and np.array_equal(xcp, u)
