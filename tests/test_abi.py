"""CPU-side checks of the C ABI boundary (-m "not gpu"): the library builds for
sm_100a, loads, and exports every function include/*.h declares; calls that
need a device fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    names = set()
    for h in ("lbfgsb.h", "lbfgsb_ops.h"):
        src = open(os.path.join(ROOT, "include", h)).read()
        src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
        for m in re.finditer(r"\b(?:lbfgsb_err|void|const char\*)\s+\**\s*([a-z_][a-z0-9_]*)\s*\(", src):
            names.add(m.group(1))
    return names


@pytest.fixture(scope="module")
def lib():
    from paper_2203_16340_b200 import _build
    path = _build.build()
    return path


def test_declared_names_nonempty():
    names = _declared()
    for n in ("lbfgsb_create", "lbfgsb_solve", "al_solve", "lbfgsb_op_gemv", "lbfgsb_op_gemvt",
              "lbfgsb_op_direction", "lbfgsb_create_sharded"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    L = C.CDLL(lib)
    missing = [n for n in sorted(_declared()) if not hasattr(L, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    for n in _declared():
        assert re.search(rf"\bT {n}$", out, re.M), n


def test_library_is_sm100a(lib):
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_fails_loudly(lib):
    """Without a GPU, lbfgsb_create must return LBFGSB_ERR_CUDA (6), never a CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    L = C.CDLL(lib)
    L.lbfgsb_create.restype = C.c_int32
    L.lbfgsb_create.argtypes = [C.c_int64, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p, C.POINTER(C.c_void_p)]
    h = C.c_void_p()
    rc = L.lbfgsb_create(10, 5, None, None, None, None, C.byref(h))
    assert rc == 6 and not h.value
    L.lbfgsb_last_error.restype = C.c_char_p
    assert b"CUDA" in L.lbfgsb_last_error()


def test_argument_errors_without_device(lib):
    L = C.CDLL(lib)
    L.lbfgsb_objective_lsq.restype = C.c_int32
    L.lbfgsb_objective_lsq.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                       C.c_int32, C.c_void_p, C.c_void_p, C.c_double,
                                       C.POINTER(C.c_void_p)]
    h = C.c_void_p()
    assert L.lbfgsb_objective_lsq(None, 10, 10, 10, None, 0, None, None, 0.0, C.byref(h)) == 1
    assert L.lbfgsb_objective_lsq(C.c_void_p(16), 10, 10, 5, None, 0, None, None, 0.0, C.byref(h)) == 2
    assert L.lbfgsb_objective_lsq(C.c_void_p(16), 10, 10, 10, C.c_void_p(16), 1, None, None, 0.0,
                                  C.byref(h)) == 1


def test_python_binding_has_no_cpu_path():
    """The binding refuses CPU tensors instead of computing on the host."""
    import torch
    import paper_2203_16340_b200 as lb
    with pytest.raises(lb.LbfgsbError):
        lb._ptr(torch.zeros(3, dtype=torch.float64))


def test_oracle_independent_of_product():
    """The oracle and the product share no code: no imports either way."""
    imp = re.compile(r"^\s*(import|from)\s+(\S+)", re.M)
    inc = re.compile(r'^\s*#\s*include\s*[<"]([^>"]+)[>"]', re.M)
    for dirpath, _, files in os.walk(os.path.join(ROOT, "paper_2203_16340_b200")):
        for f in files:
            src = open(os.path.join(dirpath, f), errors="ignore").read() if f.endswith(
                (".py", ".cu", ".cuh", ".h", ".cpp")) else ""
            for m in imp.finditer(src):
                assert not m.group(2).startswith(("oracle", "synth")), (f, m.group(0))
            for m in inc.finditer(src):
                assert "oracle" not in m.group(1), (f, m.group(0))
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            src = open(os.path.join(ROOT, "oracle", f)).read()
            for m in imp.finditer(src):
                assert "paper_2203_16340_b200" not in m.group(2), (f, m.group(0))
            for m in inc.finditer(src):
                assert m.group(1) in ("math.h", "stdint.h", "stdlib.h", "string.h", "time.h"), (f, m.group(0))
