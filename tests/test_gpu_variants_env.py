"""The opt-in backward-GEMV variants, each selected by
an environment variable read when the library loads, so every case runs in a
fresh process: k_bwd_t (register r', per-warp TMA pipelines; LBFGSB_BWD_T=1,
ring depths 2 and 3; and its lockstep whole-segment form, LBFGSB_TT_LOCK=1) and k_bwd_c (TMA + CTA pairs; LBFGSB_TMA=1).  Each must
solve the NNLS instance to the oracle's optimum, like the default k_bwd_s."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_2203_16340_b200 as lb, synth
p = synth.nnls_gaussian(6000, 3000, 95)
s = lb.Solver(p.nvars, 5, lower=torch.zeros(p.nvars, dtype=torch.float64, device="cuda"))
obj = lb.LSQObjective(lb.colmajor(p.M), b=torch.from_numpy(p.b).cuda())
x = torch.zeros(p.nvars, dtype=torch.float64, device="cuda")
r = s.solve(obj, x)
g = torch.empty(p.nvars, dtype=torch.float64, device="cuda")
rr = torch.from_numpy(p.M @ x.cpu().numpy() - p.b).cuda()
lb.op_gemvt(obj, rr, g)
ref = p.M.T @ rr.cpu().numpy()
err = float(np.max(np.abs(g.cpu().numpy() - ref) / (np.abs(p.M.T) @ np.abs(rr.cpu().numpy()) + 1e-300)))
print(json.dumps({"f": r.f, "pg": r.pg_inf, "status": r.status, "iters": r.iters, "gemvt_err": err}))
""" % ROOT


@pytest.fixture(scope="module")
def oracle_f(orc):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import synth
    p = synth.nnls_gaussian(6000, 3000, 95)
    return orc.minimize_lsq(orc.LSQ(p.M, b=p.b), l=p.lower).f


@pytest.mark.parametrize("env", [{}, {"LBFGSB_BWD_T": "1"}, {"LBFGSB_BWD_T": "1", "LBFGSB_TT_STAGES": "2"},
                                 {"LBFGSB_BWD_T": "1", "LBFGSB_TT_LOCK": "1", "LBFGSB_TT_STAGES": "4"},
                                 {"LBFGSB_TMA": "1"}])
def test_backward_variant_solves_to_the_oracle(env, oracle_f):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", CHILD], env=e, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["status"] == 0 and d["pg"] <= 1e-6
    assert abs(d["f"] - oracle_f) <= 1e-8 * abs(oracle_f)
    assert d["gemvt_err"] <= 1e-12
