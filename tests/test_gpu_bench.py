"""The bench's C5 path end to end on a shrunken C5 (bench.py --c5-shape,
smoke option; BASELINE configs[4] itself is 160 GB): N = 1 and N = 2 under
torch.distributed.run (both ranks on the test box's one GPU, CUDA-IPC
mailboxes) print valid JSON lines with the same iteration count, objective
and x checksum -- the P-invariant group through the very code path the
driver's SCALE run takes."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(out):
    lines = [l for l in out.splitlines() if l.startswith("{")]
    assert lines, out[-3000:]
    return json.loads(lines[-1])


def test_bench_c5_path_n1_n2(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    args = ["bench.py", "--c5-shape", "20000,4000", "--steps", "2", "--warmup", "3", "--no-c2",
            "--no-cpu-baseline"]
    p1 = subprocess.run([sys.executable] + args, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p1.returncode == 0, p1.stdout[-2000:] + p1.stderr[-3000:]
    d1 = _line(p1.stdout)
    port = 29800 + os.getpid() % 1000
    p2 = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                         "--master-addr=127.0.0.1", f"--master-port={port}"] + args + ["--gpus", "2"],
                        cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert p2.returncode == 0, p2.stdout[-2000:] + p2.stderr[-3000:]
    d2 = _line(p2.stdout)
    for d, n in ((d1, 1), (d2, 2)):
        assert d["n_gpus"] == n and d["scaling"] == "strong" and d["status"] == "converged"
        assert d["config"]["p_invariant"] and d["config"]["n_global"] == 4000
        assert d["roofline"]["achieved"] and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d1["iters_per_solve"] == d2["iters_per_solve"]
    assert d1["f"] == d2["f"] and d1["x_sum"] == d2["x_sum"]
