"""GPU parity of the original L-BFGS-B baseline (
lbfgsb_solve_original) against the oracle's original L-BFGS-B and against
the modified method's optimum (-m gpu)."""
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


@pytest.mark.parametrize("gen,arg,seed", [("gauss", (300, 150), 1), ("ds2", 0.25, 12), ("gauss", (41, 77), 3)])
def test_original_lbfgsb_parity(lb, orc, gen, arg, seed):
    import synth
    p = synth.nnls_gaussian(*arg, seed) if gen == "gauss" else synth.nnls_ds2(arg, seed)
    n = p.nvars
    obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda())
    s = lb.Solver(n, 5, lower=torch.zeros(n, dtype=torch.float64, device="cuda"),
                  opts=lb.Options(tol=1e-6, max_iters=5000))
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    r, cp_ms = s.solve_original(obj, x)
    ro, _ = orc.minimize_lsq_original(orc.LSQ(p.M, b=p.b), l=p.lower, opts=orc.Options(tol=1e-6, max_iters=5000))
    assert r.status == lb.CONVERGED and ro.status == orc.CONVERGED
    assert r.pg_inf <= 1e-6
    assert abs(r.f - ro.f) <= 1e-8 * abs(ro.f)
    assert abs(r.iters - ro.iters) <= max(3, ro.iters // 5)
    assert cp_ms > 0.0
    # the modified method reaches the same optimum
    x2 = torch.zeros(n, dtype=torch.float64, device="cuda")
    r2 = s.solve(obj, x2)
    assert abs(r2.f - r.f) <= 1e-7 * abs(r.f)
