"""Seeded synthetic workloads (inputs only).

This module is shared by the tests, ``bench.py`` and ``__graft_entry__.smoke``;
it holds NONE of the method's arithmetic (no working set, no two-loop, no
projection, no line search): it only draws the problem data with numpy's
seeded ``Generator`` and returns numpy arrays.  Both the oracle and the CUDA
path receive the same arrays.

Recipes follow SURVEY.md 8(d) and the paper's NNLS
generators.  Every matrix is returned column-major
(Fortran-ordered, shape (m, n)) because both implementations store A
column-major.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _gauss_colmajor(rng, m, n, scale=1.0):
    # draw an (n, m) C-ordered block and view it transposed: column-major (m, n)
    a = rng.standard_normal((n, m))
    if scale != 1.0:
        a *= scale
    return a.T


@dataclass
class Problem:
    """One synthetic instance.  ``kind`` in {"nnls", "lasso", "svm"}."""
    kind: str
    name: str
    M: np.ndarray                      # (m, ncols) column-major
    b: np.ndarray | None = None
    c: np.ndarray | None = None        # length nvars
    delta: float = 0.0
    colscale: np.ndarray | None = None
    split: bool = False
    lower: np.ndarray | None = None    # length nvars, None = -inf
    upper: np.ndarray | None = None    # length nvars, None = +inf
    E: np.ndarray | None = None        # (nvars, n_eq)
    e: np.ndarray | None = None
    meta: dict = field(default_factory=dict)

    @property
    def m(self):
        return self.M.shape[0]

    @property
    def ncols(self):
        return self.M.shape[1]

    @property
    def nvars(self):
        return 2 * self.ncols if self.split else self.ncols


def nnls_gaussian(m: int, n: int, seed: int, name: str = "") -> Problem:
    """C1/C2: A_ij ~ N(0,1)/sqrt(m), b ~ N(0,1), l = 0, u = +inf.

    The NNLS problem of PAPER.md:371 with the 1/2 scaling of reading R16.
    Expected: ~50% of the variables at the bound at the optimum.
    """
    rng = np.random.default_rng(seed)
    A = _gauss_colmajor(rng, m, n, 1.0 / np.sqrt(m))
    b = rng.standard_normal(m)
    return Problem("nnls", name or f"nnls_gaussian_{m}x{n}", A, b=b,
                   lower=np.zeros(n), upper=None, meta=dict(m=m, n=n, seed=seed))


def nnls_ds1(t: float, seed: int) -> Problem:
    """Paper data set (i): A in R^{2000t x 6000t} uniform [0,1),
    planted x with density 0.01 (half-normal, reading R23),
    b = sqrt(0.003) A x + 0.003 z."""
    rng = np.random.default_rng(seed)
    m, n = int(round(2000 * t)), int(round(6000 * t))
    A = rng.random((n, m)).T
    x = np.zeros(n)
    nz = rng.random(n) < 0.01
    x[nz] = np.abs(rng.standard_normal(int(nz.sum())))
    b = np.sqrt(0.003) * (A @ x) + 0.003 * rng.standard_normal(m)
    return Problem("nnls", f"ds1_t{t}", A, b=b, lower=np.zeros(n), meta=dict(t=t, seed=seed))


def nnls_ds2(t: float, seed: int) -> Problem:
    """Paper data set (ii): A in R^{6000t x 3000t} Gaussian,
    planted density 0.1 (half-normal, R23), b = sqrt(1/6000) A x + 0.003 z (R24)."""
    rng = np.random.default_rng(seed)
    m, n = int(round(6000 * t)), int(round(3000 * t))
    A = _gauss_colmajor(rng, m, n)
    x = np.zeros(n)
    nz = rng.random(n) < 0.1
    x[nz] = np.abs(rng.standard_normal(int(nz.sum())))
    b = np.sqrt(1.0 / 6000.0) * (A @ x) + 0.003 * rng.standard_normal(m)
    return Problem("nnls", f"ds2_t{t}", A, b=b, lower=np.zeros(n), meta=dict(t=t, seed=seed))


def lasso_split(m: int, n: int, seed: int, alpha: float = 1.0, lam_frac: float = 0.1) -> Problem:
    """C3: elastic-net / lasso via split variables x = u - v, u, v >= 0.

    A ~ N(0,1)/sqrt(m); x_true 1% nonzeros +-N(0,1); b = A x_true + 0.01 z;
    lam = lam_frac * ||A^T b||_inf;
    f(u,v) = 1/2||A(u-v) - b||^2 + lam*alpha*1^T(u+v) + lam(1-alpha)/2 (||u||^2+||v||^2).
    """
    rng = np.random.default_rng(seed)
    A = _gauss_colmajor(rng, m, n, 1.0 / np.sqrt(m))
    xt = np.zeros(n)
    nz = rng.random(n) < 0.01
    xt[nz] = rng.standard_normal(int(nz.sum()))
    b = A @ xt + 0.01 * rng.standard_normal(m)
    lam = lam_frac * float(np.max(np.abs(A.T @ b)))
    c = np.full(2 * n, lam * alpha)
    return Problem("lasso", f"lasso_{m}x{n}_a{alpha}", A, b=b, c=c, delta=lam * (1 - alpha),
                   split=True, lower=np.zeros(2 * n), upper=None,
                   meta=dict(m=m, n=n, seed=seed, alpha=alpha, lam=lam))


def svm_dual_linear(N: int, d: int, seed: int, C: float = 1.0, sep: float = 2.0) -> Problem:
    """C4: linear-kernel dual SVM (PAPER.md:349-352 with K = X X^T).

    y balanced +-1; x_i ~ N(y_i (sep/sqrt(d)) 1, I_d); C = 1.
    f(a) = 1/2 ||X^T (a*y)||^2 - 1^T a, s.t. y^T a = 0, 0 <= a <= C.
    Stored as M = X^T (d x N column-major == X row-major), colscale = y, c = -1.
    """
    rng = np.random.default_rng(seed)
    y = np.where(np.arange(N) % 2 == 0, 1.0, -1.0)
    rng.shuffle(y)
    X_T = _gauss_colmajor(rng, d, N)            # column i = sample i
    X_T += (y * (sep / np.sqrt(d)))[None, :]
    return Problem("svm", f"svm_{N}x{d}", X_T, b=None, c=-np.ones(N), colscale=y,
                   lower=np.zeros(N), upper=np.full(N, C), E=y.reshape(N, 1),
                   e=np.zeros(1), meta=dict(N=N, d=d, seed=seed, C=C))


def weak_shard(m: int, ncols_local: int, rank: int, seed: int):
    """Rank `rank`'s column block of the weak-scaled NNLS workload: the global
    A = [A_0 | ... | A_{N-1}] with A_r ~ N(0,1)/sqrt(m) drawn from
    default_rng([seed, 0xA11, r+1]) and b ~ N(0,1) from default_rng([seed, 0xB0B]) (replicated),
    so the global problem is a C2-distributed NNLS with n = N * ncols_local."""
    # distinct SeedSequence entropies for b and every block (note: numpy treats
    # [seed, 0] like [seed], so the rank is offset to keep the streams apart)
    b = np.random.default_rng([seed, 0xB0B]).standard_normal(m)
    rng = np.random.default_rng([seed, 0xA11, rank + 1])
    A = rng.standard_normal((ncols_local, m)).T / np.sqrt(m)
    return Problem("nnls", f"weak_shard_r{rank}", A, b=b, lower=np.zeros(ncols_local),
                         meta=dict(m=m, ncols_local=ncols_local, rank=rank, seed=seed))



# --------------------------------------------------------------------------- C5 (device-generated)
def _gen_lib():
    """synth/libsynth.so (nvcc, sm_100a): the device twin of synth/philox.py."""
    import ctypes, os, subprocess
    here = os.path.dirname(os.path.abspath(__file__))
    src, lib = os.path.join(here, "csrc", "gen.cu"), os.path.join(here, "libsynth.so")
    if not os.path.exists(lib) or os.path.getmtime(lib) < os.path.getmtime(src):
        subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                               "-Xcompiler", "-fPIC", "-shared", src, "-o", lib + ".tmp"])
        os.replace(lib + ".tmp", lib)
    L = ctypes.CDLL(lib)
    L.synth_fill_centered.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double,
                                      ctypes.c_void_p]
    L.synth_fill_centered.restype = ctypes.c_int
    return L


def c5_device(m: int = 100000, n: int = 200000, seed: int = 5, col0: int = 0, ncols: int | None = None,
              device="cuda", b_chunk: int = 2048):
    """C5: NNLS with A_ij = (u_ij - 1/2) sqrt(12/m) generated ON the
    device (Philox, bit-identical to synth.philox on the host); planted x (10%
    nonzeros |N(0,1)|, numpy seed) and b = A x_plant + 0.1 z with the product
    formed by torch GEMVs over column chunks (library routine, input synthesis).
    Returns (A (m, ncols) column-major torch tensor for columns [col0, col0+ncols), b (m,) numpy,
    x_plant (n,) numpy).  b always covers ALL n columns (replicated across shards)."""
    import torch
    L = _gen_lib()
    ncols = n - col0 if ncols is None else ncols
    scale = float(np.sqrt(12.0 / m))
    rng = np.random.default_rng(seed)
    xp = np.zeros(n)
    nz = rng.random(n) < 0.1
    xp[nz] = np.abs(rng.standard_normal(int(nz.sum())))
    z = rng.standard_normal(m)
    st = torch.cuda.current_stream().cuda_stream
    At = torch.empty((ncols, m), dtype=torch.float64, device=device)   # column-major (m, ncols)
    rc = L.synth_fill_centered(At.data_ptr(), m, ncols, m, col0, seed, 0, scale, st)
    if rc != 0:
        raise RuntimeError(f"synth_fill_centered failed: {rc}")
    # b = A x_plant + 0.1 z over ALL columns (chunks of the full matrix regenerated on the fly)
    bt = torch.zeros(m, dtype=torch.float64, device=device)
    tmp = torch.empty((b_chunk, m), dtype=torch.float64, device=device)
    for c0 in range(0, n, b_chunk):
        k = min(b_chunk, n - c0)
        xs = xp[c0:c0 + k]
        if not np.any(xs):
            continue
        L.synth_fill_centered(tmp.data_ptr(), m, k, m, c0, seed, 0, scale, st)
        bt += tmp[:k].T @ torch.from_numpy(xs).to(device)
    del tmp
    b = bt.cpu().numpy() + 0.1 * z
    return At.T, b, xp


def c5_planted(m: int = 100000, n: int = 200000, seed: int = 5):
    """The host-side draws of C5 (x_plant: 10% nonzeros |N(0,1)|, noise z), as in c5_device."""
    rng = np.random.default_rng(seed)
    xp = np.zeros(n)
    nz = rng.random(n) < 0.1
    xp[nz] = np.abs(rng.standard_normal(int(nz.sum())))
    z = rng.standard_normal(m)
    return xp, z


def c5_block(m: int, col0: int, ncols: int, seed: int = 5, out=None, stream=None):
    """Columns [col0, col0+ncols) of the C5 matrix, generated on the device
    (Philox; bit-identical to synth.philox.centered_block) into a fresh or
    given (ncols, m) row-major tensor = (m, ncols) column-major.  Returns the
    (m, ncols) column-major view."""
    import torch
    L = _gen_lib()
    scale = float(np.sqrt(12.0 / m))
    At = torch.empty((ncols, m), dtype=torch.float64, device="cuda") if out is None else out
    st = stream.cuda_stream if stream is not None else torch.cuda.current_stream().cuda_stream
    rc = L.synth_fill_centered(At.data_ptr(), m, ncols, m, col0, seed, 0, scale, st)
    if rc != 0:
        raise RuntimeError(f"synth_fill_centered failed: {rc}")
    return At.T


def c5_rhs(m: int = 100000, n: int = 200000, seed: int = 5, b_chunk: int = 2048):
    """b = A x_plant + 0.1 z of C5 over ALL n columns (the replicated right-hand
    side; same arithmetic as c5_device, so the same bits)."""
    import torch
    L = _gen_lib()
    xp, z = c5_planted(m, n, seed)
    scale = float(np.sqrt(12.0 / m))
    st = torch.cuda.current_stream().cuda_stream
    bt = torch.zeros(m, dtype=torch.float64, device="cuda")
    tmp = torch.empty((b_chunk, m), dtype=torch.float64, device="cuda")
    for c0 in range(0, n, b_chunk):
        k = min(b_chunk, n - c0)
        xs = xp[c0:c0 + k]
        if not np.any(xs):
            continue
        L.synth_fill_centered(tmp.data_ptr(), m, k, m, c0, seed, 0, scale, st)
        bt += tmp[:k].T @ torch.from_numpy(xs).to("cuda")
    del tmp
    return bt.cpu().numpy() + 0.1 * z


def blobs(N: int, d: int, seed: int, sep: float = 2.0, scale: float = 1.0):
    """Two Gaussian blobs, labels +-1 balanced: x_i ~ scale * N(y_i sep/sqrt(d) 1, I_d).
    scale = 1/sqrt(d) gives ||x_i - x_j||^2 ~ 2 (LibSVM-like feature scaling, so a
    gamma = 1 Gaussian kernel is far from the identity).  Returns (X (N, d), y (N,))."""
    rng = np.random.default_rng(seed)
    y = np.where(np.arange(N) % 2 == 0, 1.0, -1.0)
    rng.shuffle(y)
    X = rng.standard_normal((N, d)) + (y * (sep / np.sqrt(d)))[:, None]
    if scale != 1.0:
        X *= scale
    return X, y


def gaussian_kernel(X, gamma: float):
    """K_ij = exp(-gamma ||x_i - x_j||^2) ("standard Gaussian kernel"), numpy, by
    direct differences (no ||x||^2 expansion)."""
    X = np.asarray(X, dtype=np.float64)
    N = X.shape[0]
    K = np.empty((N, N))
    for i in range(N):
        d = X - X[i]
        K[:, i] = np.exp(-gamma * np.einsum("ij,ij->i", d, d))
    return np.asfortranarray(K)


def svm_dual_kernel(N: int, d: int, seed: int, gamma: float = 1.0, C: float = 1.0, sep: float = 2.0):
    """N1: Gaussian-kernel dual SVM on synthetic blobs (PAPER.md:349-355,
    gamma = 1, c = 1): min 1/2 (a*y)^T K (a*y) - 1^T a s.t. y^T a = 0, 0 <= a <= C.
    Returns the Problem with M = K (QP objective, colscale = y) and the raw X."""
    X, y = blobs(N, d, seed, sep)
    K = gaussian_kernel(X, gamma)
    p = Problem("svm_kernel", f"svmk_{N}x{d}", K, b=None, c=-np.ones(N), colscale=y,
                lower=np.zeros(N), upper=np.full(N, C), E=y.reshape(N, 1), e=np.zeros(1),
                meta=dict(N=N, d=d, seed=seed, gamma=gamma, C=C, X=X, qp=True))
    return p


@dataclass
class Transport:
    """Joint-probability / regularised OT instance:
    min <cost, P> + lam r(P) s.t. P 1 = u, P^T 1 = v, P >= 0."""
    name: str
    cost: np.ndarray                   # (m, n), column-major
    u: np.ndarray                      # (m,), sums to 1
    v: np.ndarray                      # (n,), sums to 1
    lam: float = 0.5                   # PAPER.md:402, 768 ("lambda = 1/2")

    @property
    def m(self):
        return self.cost.shape[0]

    @property
    def n(self):
        return self.cost.shape[1]


def _discrete_gauss(t, mu, sigma):
    w = np.exp(-0.5 * ((t - mu) / sigma) ** 2)
    return w / w.sum()


def transport_ds1(n: int) -> Transport:
    """Data set 1: m = n; u a discretised Gaussian, v a
    discretised mixture of two Gaussians, cost = u u^T (the discretised
    isotropic two-dimensional Gaussian).  The paper gives no means or
    widths; reading R31: grid t_i = i / (n - 1), u = N(0.5, 0.15),
    v = 1/2 N(0.3, 0.08) + 1/2 N(0.7, 0.08), each normalised to sum 1.
    Deterministic (no seed)."""
    t = np.linspace(0.0, 1.0, n)
    u = _discrete_gauss(t, 0.5, 0.15)
    v = 0.5 * _discrete_gauss(t, 0.3, 0.08) + 0.5 * _discrete_gauss(t, 0.7, 0.08)
    v = v / v.sum()
    cost = np.asfortranarray(np.outer(u, u))
    return Transport(f"jp_ds1_{n}", cost, u, v)


def transport_ds2(n: int, seed: int) -> Transport:
    """Data set 2 (after Frogner & Poggio): m = 2n; u, v ~ U(0,1)
    scaled to sum 1; cost entries ~ U(0,1); lam = 1/2."""
    rng = np.random.default_rng([seed, 0xD52])
    m = 2 * n
    u = rng.uniform(size=m); u = u / u.sum()
    v = rng.uniform(size=n); v = v / v.sum()
    cost = np.asfortranarray(rng.uniform(size=(m, n)))
    return Transport(f"jp_ds2_{m}x{n}", cost, u, v)


# Named configurations of BASELINE.json "configs"
CONFIGS = {
    "C1": lambda seed=1: nnls_gaussian(200, 100, seed, "C1_nnls_200x100"),
    "C2": lambda seed=2: nnls_gaussian(20000, 10000, seed, "C2_nnls_20000x10000"),
    "C3": lambda seed=3: lasso_split(10000, 50000, seed, alpha=1.0),
    "C3en": lambda seed=3: lasso_split(10000, 50000, seed, alpha=0.5),
    "C4": lambda seed=4: svm_dual_linear(100000, 1000, seed),
}
