"""A/B timing of the backward GEMV variants on C2 (20000 x 10000): op_gemvt
(BWD_PLAIN, the stream kernel without the epilogue) and full bench solves.
Each setting runs in its own process (the variant is picked from env vars at
library load).  python tools/bwd_sweep.py [--child]"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child():
    import torch
    import paper_2203_16340_b200 as lb
    torch.manual_seed(0)
    m, n = 20000, 10000
    M = torch.randn(n, m, dtype=torch.float64, device="cuda").t()   # column-major view
    r = torch.randn(m, dtype=torch.float64, device="cuda")
    g = torch.empty(n, dtype=torch.float64, device="cuda")
    obj = lb.LSQObjective(M, b=None)
    for _ in range(3):
        lb.op_gemvt(obj, r, g)
    torch.cuda.synchronize()
    ref = (M.t() @ r)
    err = (g - ref).abs().max().item() / (M.abs().t() @ r.abs()).max().item()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 50
    e0.record()
    for _ in range(K):
        lb.op_gemvt(obj, r, g)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / K
    print(json.dumps({"us": us, "gbs": 8 * m * n / us / 1e3, "relerr": err}))


if __name__ == "__main__":
    if "--child" in sys.argv:
        child()
        sys.exit(0)
    settings = [("k_bwd_s", {})] + \
        [(f"k_bwd_t stages={s}", {"LBFGSB_BWD_T": "1", "LBFGSB_TT_STAGES": str(s)}) for s in (3,)] + \
        [(f"k_bwd_t lock stages={s}", {"LBFGSB_BWD_T": "1", "LBFGSB_TT_LOCK": "1", "LBFGSB_TT_STAGES": str(s)})
         for s in (3, 4, 5, 6)]
    for name, env in settings:
        e = dict(os.environ, **env)
        out = subprocess.run([sys.executable, __file__, "--child"], env=e, capture_output=True, text=True)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
        print(f"{name:24s} {line}", flush=True)
        if "--bench" in sys.argv:
            out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline",
                                  "--steps", "10"], env=e, capture_output=True, text=True)
            try:
                d = json.loads(out.stdout.strip().splitlines()[-1])
                print(f"{'':24s} bench {d['value']:.1f} it/s  bwd {d['roofline']['avg_launch_us']:.1f} us",
                      flush=True)
            except Exception:
                print(out.stderr[-800:])
