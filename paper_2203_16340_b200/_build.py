"""Build liblbfgsb.so in-tree with nvcc for sm_100a (no GPU needed to compile)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "liblbfgsb.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# -fmad=false: no implicit FMA contraction; fused ops are explicit fma() (reading R12)
NVCC_FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
              "-Xcompiler", "-O2", "--expt-relaxed-constexpr"]


def _nccl_dirs():
    try:
        import nvidia.nccl as nn  # torch-bundled NCCL 2.28
        base = os.path.dirname(nn.__file__) if nn.__file__ else list(nn.__path__)[0]
    except Exception:
        return None
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and glob.glob(os.path.join(lib, "libnccl.so*")):
        return inc, lib
    return None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build() -> bool:
    if os.environ.get("LBFGSB_NO_AUTOBUILD"):        # A/B runs against a prebuilt variant library
        return False
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cmd = [nvcc, *ARCH, *NVCC_FLAGS, "-shared", "-I", os.path.join(ROOT, "include"), *cu,
           "-o", LIB + ".tmp"]
    nccl = _nccl_dirs()
    if nccl:
        inc, lib = nccl
        cmd += ["-DLBFGSB_WITH_NCCL", "-I", inc, "-L", lib, "-l:libnccl.so.2",
                "-Xlinker", "-rpath", "-Xlinker", lib]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(LIB + ".tmp", LIB)
    return LIB


def build_variant(out: str, defines: list[str], verbose: bool = False) -> str:
    """A/B experiments only: the same sources with extra -D flags into `out`."""
    nvcc = os.environ.get("NVCC", "nvcc")
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    cmd = [nvcc, *ARCH, *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-shared", "-I", os.path.join(ROOT, "include"),
           *cu, "-o", out]
    nccl = _nccl_dirs()
    if nccl:
        inc, lib = nccl
        cmd += ["-DLBFGSB_WITH_NCCL", "-I", inc, "-L", lib, "-l:libnccl.so.2",
                "-Xlinker", "-rpath", "-Xlinker", lib]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    os.makedirs(os.path.dirname(os.path.abspath(out)), exist_ok=True)
    subprocess.check_call(cmd)
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
