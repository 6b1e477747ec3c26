"""GPU tests of the column-sharded path (-m gpu).  Only one GPU is available
to this build, so the multi-rank protocol is verified two ways:
  * loopback: P logical ranks (handles) on one device exchanging their packs
    with device copies, checked against the single-GPU solve and the oracle;
  * a 1-rank NCCL communicator (lbfgsb_create_sharded, nranks = 1) running
    the full sharded protocol: NCCL all-gathers captured in the CUDA graph
    and the rank-order *_decide kernels.
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


def _shards(lb, prob, P, opts=None):
    from paper_2203_16340_b200.sharded import column_range
    sv, ob, xs, keep = [], [], [], []
    for r in range(P):
        c0, c1 = column_range(prob.ncols, P, r)
        Mr = lb.colmajor(prob.M[:, c0:c1])
        if prob.split:
            vsl = np.r_[c0:c1, prob.ncols + c0:prob.ncols + c1]
        else:
            vsl = np.arange(c0, c1)
        lo = None if prob.lower is None else _cuda(prob.lower[vsl])
        up = None if prob.upper is None else _cuda(prob.upper[vsl])
        c = None if prob.c is None else _cuda(prob.c[vsl])
        b = None if prob.b is None else _cuda(prob.b)
        o = lb.LSQObjective(Mr, b=b, c=c, delta=prob.delta, split=prob.split)
        s = lb.Solver(len(vsl), 5, lower=lo, upper=up, opts=opts or lb.Options())
        x = torch.zeros(len(vsl), dtype=torch.float64, device="cuda")
        sv.append(s); ob.append(o); xs.append(x); keep.append((Mr, lo, up, c, b))
    return sv, ob, xs, keep


def _gather_x(prob, P, xs):
    from paper_2203_16340_b200.sharded import column_range
    x = np.zeros(prob.nvars)
    for r in range(P):
        c0, c1 = column_range(prob.ncols, P, r)
        xr = xs[r].cpu().numpy()
        if prob.split:
            k = c1 - c0
            x[c0:c1] = xr[:k]
            x[prob.ncols + c0:prob.ncols + c1] = xr[k:]
        else:
            x[c0:c1] = xr
    return x


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_loopback_nnls_matches_single_gpu_and_oracle(lb, orc, P):
    import synth
    prob = synth.nnls_gaussian(3000, 2000, 77)
    sv, ob, xs, _ = _shards(lb, prob, P)
    r = lb.solve_loopback(sv, ob, xs)
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
    assert r.status == lb.CONVERGED and r.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    x = _gather_x(prob, P, xs)
    assert np.all(x >= 0)
    res = prob.M @ x - prob.b
    assert abs(0.5 * res @ res - r.f) <= 1e-10 * r.f


@pytest.mark.parametrize("P", [2, 4])
def test_loopback_tall_columns_vs_oracle(lb, orc, P):
    """Sharded loopback at m = 40000 (C5-shaped columns, generic k_bwd) against
    the oracle (VERDICT r1 "Next" 2)."""
    import synth
    prob = synth.nnls_gaussian(40000, 1600, 78)
    sv, ob, xs, _ = _shards(lb, prob, P)
    r = lb.solve_loopback(sv, ob, xs)
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
    assert r.status == lb.CONVERGED and r.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    assert np.all(_gather_x(prob, P, xs) >= 0)


def test_loopback_is_deterministic(lb):
    import synth
    prob = synth.nnls_gaussian(2500, 1800, 78)
    out = []
    for _ in range(2):
        sv, ob, xs, _ = _shards(lb, prob, 3)
        r = lb.solve_loopback(sv, ob, xs)
        out.append((_gather_x(prob, 3, xs), r.f, r.iters))
    assert np.array_equal(out[0][0], out[1][0]) and out[0][1:] == out[1][1:]


def test_loopback_lasso_split(lb, orc):
    import synth
    prob = synth.lasso_split(500, 1200, 79, alpha=0.5)
    sv, ob, xs, _ = _shards(lb, prob, 2)
    r = lb.solve_loopback(sv, ob, xs)
    P = orc.LSQ(prob.M, b=prob.b, c=prob.c, delta=prob.delta, split=True)
    ro = orc.minimize_lsq(P, l=prob.lower)
    assert r.pg_inf <= 1e-6 and abs(r.f - ro.f) <= 1e-8 * abs(ro.f)


def test_nccl_one_rank_sharded_protocol(lb, orc):
    """lbfgsb_create_sharded with a 1-rank communicator: NCCL all-gathers inside
    the captured graph + rank-order decisions give the single-GPU optimum."""
    import synth
    prob = synth.nnls_gaussian(2000, 1500, 80)
    nid = lb.nccl_unique_id()
    lo = _cuda(prob.lower)
    s = lb.Solver(prob.nvars, 5, lower=lo, nccl_id=nid, rank=0, nranks=1, n_global=prob.nvars)
    obj = lb.LSQObjective(lb.colmajor(prob.M), b=_cuda(prob.b))
    x = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r = s.solve(obj, x)
    ro = orc.minimize_lsq(orc.LSQ(prob.M, b=prob.b), l=prob.lower)
    assert r.status == lb.CONVERGED and r.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    s2 = lb.Solver(prob.nvars, 5, lower=lo, opts=lb.Options(use_graph=False), nccl_id=lb.nccl_unique_id(),
                   rank=0, nranks=1, n_global=prob.nvars)
    x2 = torch.zeros(prob.nvars, dtype=torch.float64, device="cuda")
    r2 = s2.solve(obj, x2)
    assert torch.equal(x, x2) and r.f == r2.f                     # graph == eager, bitwise
