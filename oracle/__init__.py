"""CPU oracle for the modified L-BFGS-B of arXiv 2203.16340 (ctypes wrapper).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product package ``paper_2203_16340_b200`` never imports it and
the two share no code: this module wraps ``oracle/oracle.c`` (plain C, fp64,
sequential loops, ``-ffp-contract=off``) and nothing else.

Every function cites the paper passage it follows (``PAPER.md:N``); the
readings of the paper it takes are listed in DESIGN.md section 3 (R1..R28).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

CONVERGED, MAX_ITERS, LINESEARCH_FAILURE, AL_MAX_OUTER, AL_INNER_FAILURE = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (no GPU needed)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
               _SRC, "-o", _LIB + ".tmp", "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


_lib = None


class using_library:
    """Context manager: route every call of this module through another build
    of oracle.c (the mutation tests compile deliberately broken copies and
    check that the pins reject them)."""

    def __init__(self, path):
        self.path = path

    def __enter__(self):
        global _lib
        self._saved = _lib
        lib = C.CDLL(self.path)
        _setup(lib)
        _lib = lib
        return self

    def __exit__(self, *exc):
        global _lib
        _lib = self._saved
        return False


def build_variant(out_path, replacements):
    """Compile a copy of oracle.c with each (old, new) text replacement applied
    (each ``old`` must occur exactly once).  Test infrastructure for the
    mutation pins only."""
    src = open(_SRC).read()
    for old, new in replacements:
        assert src.count(old) == 1, ("mutation anchor not unique", old)
        src = src.replace(old, new)
    cpath = out_path + ".c"
    with open(cpath, "w") as f:
        f.write(src)
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
                           cpath, "-o", out_path, "-lm"])
    return out_path


def _L():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _setup(_lib)
    return _lib


_dp = C.POINTER(C.c_double)
_u8p = C.POINTER(C.c_uint8)


class _Lsq(C.Structure):
    _fields_ = [("m", C.c_int64), ("ncols", C.c_int64), ("lda", C.c_int64),
                ("M", _dp), ("colscale", _dp), ("split", C.c_int32),
                ("b", _dp), ("c", _dp), ("delta", C.c_double),
                ("n_eq", C.c_int32), ("E", _dp), ("e", _dp), ("lam", _dp),
                ("n_in", C.c_int32), ("G", _dp), ("hv", _dp), ("mu", _dp),
                ("rho", C.c_double), ("qp", C.c_int32), ("ent", C.c_double),
                ("tm", C.c_int64)]


class _Opts(C.Structure):
    _fields_ = [("eps", C.c_double), ("c1", C.c_double), ("shrink", C.c_double),
                ("tol", C.c_double), ("max_backtracks", C.c_int32),
                ("screen_full_norm", C.c_int32), ("no_projection", C.c_int32),
                ("armijo_diff", C.c_int32), ("refresh_every", C.c_int32), ("max_iters", C.c_int64)]


class _Res(C.Structure):
    _fields_ = [("f", C.c_double), ("pg_inf", C.c_double), ("gfree_inf", C.c_double),
                ("iters", C.c_int64), ("n_fg", C.c_int64), ("n_backtracks", C.c_int64),
                ("n_free", C.c_int64), ("status", C.c_int32), ("last_branch", C.c_int32),
                ("n_fallbacks", C.c_int64)]


class _AlOpts(C.Structure):
    _fields_ = [("feas_tol", C.c_double), ("rho0", C.c_double), ("rho_factor", C.c_double),
                ("rho_cap", C.c_double), ("max_outer", C.c_int32)]


class _AlRes(C.Structure):
    _fields_ = [("violation_inf", C.c_double), ("rho", C.c_double), ("f", C.c_double),
                ("outer_iters", C.c_int64), ("inner_iters_total", C.c_int64),
                ("status", C.c_int32)]


def _setup(L):
    i64, i32, d = C.c_int64, C.c_int32, C.c_double
    L.orc_clip.argtypes = [i64, _dp, _dp, _dp, _dp]
    L.orc_working_set.argtypes = [i64, _dp, _dp, _dp, _dp, d, _u8p]
    L.orc_masked_dot.argtypes = [i64, _dp, _dp, _u8p]
    L.orc_masked_dot.restype = d
    L.orc_matvec.argtypes = [i64, i64, _dp, i64, _dp, _dp]
    L.orc_matvec_t.argtypes = [i64, i64, _dp, i64, _dp, _dp]
    L.orc_set_threads.argtypes = [i32]
    L.orc_get_threads.restype = i32
    L.orc_two_loop.argtypes = [i64, _dp, _u8p, i32, _dp, _dp, d, i32, _dp]
    L.orc_project_direction.argtypes = [i64, _dp, _dp, _dp, _dp, _dp, d, _dp]
    L.orc_project_direction.restype = i32
    L.orc_max_step.argtypes = [i64, _dp, _dp, _dp, _dp]
    L.orc_max_step.restype = d
    L.orc_minimize_lsq.argtypes = [C.POINTER(_Lsq), _dp, _dp, i32, C.POINTER(_Opts), _dp,
                                   C.POINTER(_Res)]
    L.orc_al_solve.argtypes = [C.POINTER(_Lsq), _dp, _dp, _dp, _dp, i32, C.POINTER(_Opts),
                               C.POINTER(_AlOpts), _dp, C.POINTER(_AlRes)]
    L.orc_al_solve_ex.argtypes = [C.POINTER(_Lsq), _dp, _dp, _dp, _dp, i32, C.POINTER(_Opts),
                                  C.POINTER(_AlOpts), _dp, i32, _dp, C.POINTER(_AlRes)]
    L.orc_al_violation.argtypes = [i32, _dp, i32, _dp, _dp, d]
    L.orc_al_violation.restype = d
    L.orc_al_update_multipliers.argtypes = [i32, _dp, _dp, i32, _dp, _dp, d]
    L.orc_al_update_rho.argtypes = [d, d, d, d, d]
    L.orc_al_update_rho.restype = d
    L.orc_armijo_lsq.argtypes = [C.POINTER(_Lsq), C.POINTER(_Opts), i64, _dp, _dp, _dp, _dp, _dp,
                                 _dp, d, d, d, _dp, _dp, _dp, _dp, C.POINTER(i64)]
    L.orc_armijo_lsq.restype = i32
    L.orc_check_convergence.argtypes = [i64, _dp, _u8p, d]
    L.orc_check_convergence.restype = i32
    L.orc_lsq_value.argtypes = [C.POINTER(_Lsq), _dp]
    L.orc_lsq_value.restype = d
    L.orc_lsq_grad.argtypes = [C.POINTER(_Lsq), _dp, _dp]
    L.orc_armijo_delta.argtypes = [C.POINTER(_Lsq), i64, _dp, _dp, _dp, _dp, _dp, _dp, d]
    L.orc_armijo_delta.restype = d
    L.orc_compact_m.argtypes = [i64, i32, _dp, _dp, d, _dp]
    L.orc_compact_m.restype = i32
    L.orc_cauchy_point.argtypes = [i64, _dp, _dp, _dp, _dp, i32, _dp, _dp, d, _dp, _dp]
    L.orc_cauchy_point.restype = i64
    L.orc_lbfgsb_original.argtypes = [C.POINTER(_Lsq), _dp, _dp, i32, C.POINTER(_Opts), _dp,
                                      C.POINTER(_Res), C.POINTER(d)]
    L.orc_armijo_scalar_quadratic.argtypes = [d, d, d, d, d, i32]
    L.orc_armijo_scalar_quadratic.restype = d


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


def _u8(a):
    return np.ascontiguousarray(a, dtype=np.uint8)


# --------------------------------------------------------------------------
# Elementwise pieces
# --------------------------------------------------------------------------
def clip(x, l=None, u=None):
    """min(max(x, l), u) -- Alg. 2 line 1."""
    x = _f64(x); l = None if l is None else _f64(l); u = None if u is None else _f64(u)
    out = np.empty_like(x)
    _L().orc_clip(x.size, _ptr(x), _ptr(l), _ptr(u), _ptr(out))
    return out


def working_set(x, g, l, u, eps):
    """Eq. (1).  Returns a bool mask of FREE variables."""
    x, g = _f64(x), _f64(g)
    l = None if l is None else _f64(l); u = None if u is None else _f64(u)
    fr = np.empty(x.size, dtype=np.uint8)
    _L().orc_working_set(x.size, _ptr(x), _ptr(g), _ptr(l), _ptr(u), eps,
                         fr.ctypes.data_as(_u8p))
    return fr.astype(bool)


def masked_dot(u, v, free=None):
    """<u[S], v[S]> (Alg. 3 line 3)."""
    u, v = _f64(u), _f64(v)
    fr = None if free is None else _u8(free)
    return _L().orc_masked_dot(u.size, _ptr(u), _ptr(v),
                               None if fr is None else fr.ctypes.data_as(_u8p))


def set_threads(t: int):
    """Threads of the oracle's matvecs (OpenMP over output elements only: the
    results are bit-identical to 1 thread).  Default 1."""
    _L().orc_set_threads(int(t))


def get_threads() -> int:
    return int(_L().orc_get_threads())


def matvec(A, x):
    """A x with A column-major (Fortran-ordered numpy array)."""
    A = np.asfortranarray(A, dtype=np.float64); x = _f64(x)
    m, n = A.shape
    out = np.empty(m)
    _L().orc_matvec(m, n, _ptr(A), m, _ptr(x), _ptr(out))
    return out


def matvec_t(A, r):
    """A^T r with A column-major."""
    A = np.asfortranarray(A, dtype=np.float64); r = _f64(r)
    m, n = A.shape
    out = np.empty(n)
    _L().orc_matvec_t(m, n, _ptr(A), m, _ptr(r), _ptr(out))
    return out


def two_loop(g, free, S=(), Y=(), eps=1e-9, screen_full_norm=False):
    """Alg. 3 literal; pairs oldest first.  Returns d = -q (R5)."""
    g = _f64(g); n = g.size
    fr = _u8(free)
    nh = len(S)
    Sm = _f64(np.reshape(S, (nh, n))) if nh else np.zeros((1, n))
    Ym = _f64(np.reshape(Y, (nh, n))) if nh else np.zeros((1, n))
    d = np.empty(n)
    _L().orc_two_loop(n, _ptr(g), fr.ctypes.data_as(_u8p), nh, _ptr(Sm), _ptr(Ym), eps,
                      int(bool(screen_full_norm)), _ptr(d))
    return d


def project_direction(x, g, d, l, u, eps):
    """Alg. 2.  Returns (p, projected: bool)."""
    x, g, d = _f64(x), _f64(g), _f64(d)
    l = None if l is None else _f64(l); u = None if u is None else _f64(u)
    p = np.empty_like(x)
    br = _L().orc_project_direction(x.size, _ptr(x), _ptr(g), _ptr(d), _ptr(l), _ptr(u),
                                    eps, _ptr(p))
    return p, bool(br)


def max_step(x, p, l, u):
    """Minimum blocking ratio (R10)."""
    x, p = _f64(x), _f64(p)
    l = None if l is None else _f64(l); u = None if u is None else _f64(u)
    return _L().orc_max_step(x.size, _ptr(x), _ptr(p), _ptr(l), _ptr(u))


def check_convergence(g, free, tol):
    g = _f64(g); fr = _u8(free)
    return bool(_L().orc_check_convergence(g.size, _ptr(g), fr.ctypes.data_as(_u8p), tol))


def compact_m(S, Y, theta):
    """M of the compact L-BFGS form B = theta I - W M W^T, W = [Y, theta S]
    (Byrd-Lu-Nocedal-Zhu 1995).  S, Y: (h, n) pairs, oldest first."""
    S = np.ascontiguousarray(S, dtype=np.float64); Y = np.ascontiguousarray(Y, dtype=np.float64)
    h, n = S.shape
    M = np.zeros((2 * h, 2 * h))
    rc = _L().orc_compact_m(n, h, _ptr(S), _ptr(Y), float(theta), _ptr(M))
    if rc:
        raise np.linalg.LinAlgError("singular middle matrix")
    return M


def cauchy_point(x, g, l, u, S=None, Y=None, theta=1.0):
    """Generalized Cauchy point of the original L-BFGS-B (Algorithm CP of
    Byrd et al. 1995; the step PAPER.md:19-23, 436-440 removes).  Returns
    (xcp, c = W^T (xcp - x), number of breakpoints passed)."""
    x = _f64(x); g = _f64(g); n = len(x)
    l = None if l is None else _f64(np.broadcast_to(l, (n,)))
    u = None if u is None else _f64(np.broadcast_to(u, (n,)))
    if S is None or len(S) == 0:
        h = 0; Sp = np.zeros((1, n)); Yp = np.zeros((1, n))
    else:
        Sp = np.ascontiguousarray(S, dtype=np.float64); Yp = np.ascontiguousarray(Y, dtype=np.float64)
        h = Sp.shape[0]
    xcp = np.empty(n); c = np.zeros(max(2 * h, 1))
    passed = _L().orc_cauchy_point(n, _ptr(x), _ptr(g), _ptr(l), _ptr(u), h, _ptr(Sp), _ptr(Yp),
                                   float(theta), _ptr(xcp), _ptr(c))
    if passed < 0:
        raise np.linalg.LinAlgError("singular middle matrix")
    return xcp, c[:2 * h], int(passed)


def armijo_scalar_quadratic(x, p, amax=1.0, c1=1e-4, shrink=0.5, max_bt=50):
    return _L().orc_armijo_scalar_quadratic(x, p, amax, c1, shrink, max_bt)


# --------------------------------------------------------------------------
# LSQ objective family + Alg. 1 / Alg. 4
# --------------------------------------------------------------------------
@dataclass
class Options:
    eps: float = 1e-9          # R1
    c1: float = 1e-4           # R11
    shrink: float = 0.5        # R11
    tol: float = 1e-6          # R15
    max_backtracks: int = 50   # R11
    screen_full_norm: bool = False  # R3
    max_iters: int = 10000
    no_projection: bool = False     # PAPER.md:201 variant
    armijo_diff: bool = False       # R29: Armijo on the expanded difference (N4)
    refresh_every: int = 0          # R13: exact r, f, g every R iterations (0: only the final refresh)


@dataclass
class ALOptions:
    feas_tol: float = 1e-6
    rho0: float = 1.0
    rho_factor: float = 2.0
    rho_cap: float = 1e12
    max_outer: int = 100


class LSQ:
    """f(x) = 1/2||M~x - b||^2 + c^T x + delta/2||x||^2 (+ AL terms of Eq. (3)).

    M is m x ncols (numpy, any order; stored column-major); M~ = M diag(colscale),
    or [M, -M] when ``split``.  Linear constraints: E^T x = e (E nvars x n_eq),
    G^T x <= hv (G nvars x n_in).
    """

    def __init__(self, M, b=None, c=None, delta=0.0, colscale=None, split=False,
                 E=None, e=None, G=None, hv=None, qp=False, ent=0.0, tm=0):
        self.M = np.asfortranarray(M, dtype=np.float64)
        self.m, self.ncols = self.M.shape
        self.qp = bool(qp)           # 1/2 x^T D M D x (+ c, delta, AL); M square symmetric
        if self.qp:
            assert self.m == self.ncols and not split and b is None
        self.split = bool(split)
        self.nvars = 2 * self.ncols if split else self.ncols
        self.b = None if b is None else _f64(b)
        self.c = None if c is None else _f64(c)
        self.delta = float(delta)
        self.colscale = None if colscale is None else _f64(colscale)
        self.E = None if E is None else np.asfortranarray(np.reshape(E, (self.nvars, -1)), dtype=np.float64)
        self.e = None if e is None else _f64(np.atleast_1d(e))
        self.G = None if G is None else np.asfortranarray(np.reshape(G, (self.nvars, -1)), dtype=np.float64)
        self.hv = None if hv is None else _f64(np.atleast_1d(hv))
        self.ent = float(ent)         # + ent * sum x log x (SURVEY N2 entropy regulariser)
        self.tm = int(tm)             # > 0: equality constraints = marginals of P (tm x nvars/tm)
        if self.tm > 0:
            assert self.E is None and self.nvars % self.tm == 0 and self.e is not None
            self.n_eq = self.tm + self.nvars // self.tm
            assert len(self.e) == self.n_eq
        else:
            self.n_eq = 0 if self.E is None else self.E.shape[1]
        self.n_in = 0 if self.G is None else self.G.shape[1]
        self.lam = np.zeros(max(self.n_eq, 1))
        self.mu = np.zeros(max(self.n_in, 1))
        self.rho = 1.0

    @classmethod
    def transport(cls, cost, u, v, reg="entropy", lam=0.5):
        """Joint probability / regularised OT:
        min <cost, P> + lam r(P)  s.t. P 1 = u, P^T 1 = v, P >= 0, with
        r = sum P log P (reg="entropy") or 1/2 ||P||_F^2 (reg="gaussian").
        Variables x = vec(P) column-major (m*n); no quadratic data term."""
        cost = np.asarray(cost, dtype=np.float64)
        m, n = cost.shape
        c = cost.reshape(-1, order="F")
        e = np.concatenate([_f64(u), _f64(v)])
        if reg == "entropy":
            return cls(np.zeros((0, m * n)), c=c, ent=lam, tm=m, e=e)
        if reg == "gaussian":
            return cls(np.zeros((0, m * n)), c=c, delta=lam, tm=m, e=e)
        raise ValueError(reg)

    def _struct(self):
        s = _Lsq()
        s.m, s.ncols, s.lda = self.m, self.ncols, self.m
        s.M = _ptr(self.M)
        s.colscale = _ptr(self.colscale)
        s.split = int(self.split)
        s.b = _ptr(self.b); s.c = _ptr(self.c); s.delta = self.delta
        s.n_eq = self.n_eq; s.E = _ptr(self.E); s.e = _ptr(self.e); s.lam = _ptr(self.lam)
        s.n_in = self.n_in; s.G = _ptr(self.G); s.hv = _ptr(self.hv); s.mu = _ptr(self.mu)
        s.rho = self.rho
        s.qp = int(self.qp)
        s.ent = self.ent
        s.tm = self.tm
        return s

    def value(self, x):
        x = _f64(x); s = self._struct()
        return _L().orc_lsq_value(C.byref(s), _ptr(x))

    def grad(self, x):
        x = _f64(x); s = self._struct(); g = np.empty(self.nvars)
        _L().orc_lsq_grad(C.byref(s), _ptr(x), _ptr(g))
        return g

    def apply(self, v):
        """M~ v (QP: Q~ v = D M D v), plain numpy."""
        v = _f64(v)
        if self.split:
            v = v[:self.ncols] - v[self.ncols:]
        if self.colscale is not None:
            v = self.colscale * v
        out = self.M @ v
        if self.qp and self.colscale is not None:
            out = self.colscale * out
        return out

    def armijo_delta(self, x, p, alpha, l=None, u=None):
        """f(x + alpha p) - f(x) by the expanded form of reading R29
        (orc_armijo_delta), with the carried r (LSQ: M~x - b, QP: w = Q~x) and
        q = M~p formed here."""
        x = _f64(x); p = _f64(p)
        r = self.apply(x)
        if not self.qp and self.b is not None:
            r = r - self.b
        q = self.apply(p)
        s = self._struct()
        lb = None if l is None else _f64(np.broadcast_to(l, (self.nvars,)))
        ub = None if u is None else _f64(np.broadcast_to(u, (self.nvars,)))
        return _L().orc_armijo_delta(C.byref(s), self.nvars, _ptr(x), _ptr(_f64(r)), _ptr(_f64(q)),
                                     _ptr(p), _ptr(lb), _ptr(ub), float(alpha))


@dataclass
class Result:
    x: np.ndarray
    f: float
    pg_inf: float
    gfree_inf: float
    iters: int
    n_fg: int
    n_backtracks: int
    n_free: int
    status: int
    last_branch: int
    n_fallbacks: int


def minimize_lsq(P: LSQ, l=None, u=None, x0=None, m_hist=5, opts: Options | None = None):
    """Alg. 1 on the LSQ objective, with Alg. 2/3 and Armijo."""
    o = opts or Options()
    x = np.zeros(P.nvars) if x0 is None else _f64(x0).copy()
    l = None if l is None else _f64(np.broadcast_to(l, (P.nvars,)))
    u = None if u is None else _f64(np.broadcast_to(u, (P.nvars,)))
    so = _Opts(o.eps, o.c1, o.shrink, o.tol, o.max_backtracks, int(o.screen_full_norm),
               int(o.no_projection), int(o.armijo_diff), int(o.refresh_every), o.max_iters)
    res = _Res()
    s = P._struct()
    _L().orc_minimize_lsq(C.byref(s), _ptr(l), _ptr(u), m_hist, C.byref(so), _ptr(x),
                          C.byref(res))
    return Result(x, res.f, res.pg_inf, res.gfree_inf, res.iters, res.n_fg, res.n_backtracks,
                  res.n_free, res.status, res.last_branch, res.n_fallbacks)


def minimize_lsq_original(P: LSQ, l=None, u=None, x0=None, m_hist=5, opts: Options | None = None):
    """The ORIGINAL L-BFGS-B (Byrd et al. 1995: Cauchy point + direct primal
    subspace minimisation + backtracking; SURVEY N3 baseline).
    Returns (Result, seconds spent in the Cauchy point)."""
    o = opts or Options()
    assert o.m_hist_ok(m_hist) if hasattr(o, "m_hist_ok") else m_hist <= 16
    x = np.zeros(P.nvars) if x0 is None else _f64(x0).copy()
    l = None if l is None else _f64(np.broadcast_to(l, (P.nvars,)))
    u = None if u is None else _f64(np.broadcast_to(u, (P.nvars,)))
    so = _Opts(o.eps, o.c1, o.shrink, o.tol, o.max_backtracks, int(o.screen_full_norm),
               int(o.no_projection), int(o.armijo_diff), int(o.refresh_every), o.max_iters)
    res = _Res()
    tcp = C.c_double(0.0)
    s = P._struct()
    _L().orc_lbfgsb_original(C.byref(s), _ptr(l), _ptr(u), m_hist, C.byref(so), _ptr(x), C.byref(res),
                             C.byref(tcp))
    return (Result(x, res.f, res.pg_inf, res.gfree_inf, res.iters, res.n_fg, res.n_backtracks,
                   res.n_free, res.status, res.last_branch, res.n_fallbacks), tcp.value)


@dataclass
class ALResult:
    x: np.ndarray
    lam: np.ndarray
    mu: np.ndarray
    f: float
    violation_inf: float
    rho: float
    outer_iters: int
    inner_iters_total: int
    status: int


def al_solve(P: LSQ, l=None, u=None, m_hist=5, opts: Options | None = None,
             al_opts: ALOptions | None = None, x0=None, lam0=None, mu0=None, trace=False):
    """Alg. 4 for linear constraints.

    Cold start (default): x^0 = clip(0), lam = mu = 0 (R19).  Passing any of
    x0 / lam0 / mu0 re-enters the method from that state (missing parts are
    zero).  trace=True also returns, per outer iteration, a dict with the rho
    the inner solve used, the violation v after the multiplier update, the rho
    after the penalty rule, lam, mu and x."""
    o = opts or Options(); ao = al_opts or ALOptions()
    warm = x0 is not None or lam0 is not None or mu0 is not None
    x = np.zeros(P.nvars) if x0 is None else _f64(x0).copy()
    l = None if l is None else _f64(np.broadcast_to(l, (P.nvars,)))
    u = None if u is None else _f64(np.broadcast_to(u, (P.nvars,)))
    lam = np.zeros(max(P.n_eq, 1)); mu = np.zeros(max(P.n_in, 1))
    if lam0 is not None:
        lam[:P.n_eq] = lam0
    if mu0 is not None:
        mu[:P.n_in] = mu0
    so = _Opts(o.eps, o.c1, o.shrink, o.tol, o.max_backtracks, int(o.screen_full_norm),
               int(o.no_projection), int(o.armijo_diff), int(o.refresh_every), o.max_iters)
    sa = _AlOpts(ao.feas_tol, ao.rho0, ao.rho_factor, ao.rho_cap, ao.max_outer)
    s = P._struct()
    res = _AlRes()
    rec = 3 + P.n_eq + P.n_in + P.nvars
    tb = np.zeros(ao.max_outer * rec) if trace else None
    _L().orc_al_solve_ex(C.byref(s), _ptr(lam), _ptr(mu), _ptr(l), _ptr(u), m_hist, C.byref(so),
                         C.byref(sa), _ptr(x), int(warm), _ptr(tb), C.byref(res))
    out = ALResult(x, lam[:P.n_eq].copy(), mu[:P.n_in].copy(), res.f, res.violation_inf,
                   res.rho, res.outer_iters, res.inner_iters_total, res.status)
    if trace:
        recs = []
        for it in range(res.outer_iters):
            t = tb[it * rec:(it + 1) * rec]
            recs.append({"rho_used": t[0], "v": t[1], "rho_next": t[2],
                         "lam": t[3:3 + P.n_eq].copy(), "mu": t[3 + P.n_eq:3 + P.n_eq + P.n_in].copy(),
                         "x": t[3 + P.n_eq + P.n_in:].copy()})
        return out, recs
    return out


def al_violation(h=(), g=(), mu=None, rho=1.0):
    """Violation measure of Alg. 4's penalty rule / stop test (R21)."""
    h = _f64(np.atleast_1d(h)) if len(h) else np.zeros(1)
    gg = _f64(np.atleast_1d(g)) if len(g) else np.zeros(1)
    mu = np.zeros_like(gg) if mu is None else _f64(np.atleast_1d(mu))
    return _L().orc_al_violation(len(np.atleast_1d(h)) if len(h) else 0, _ptr(h),
                                 len(g), _ptr(gg), _ptr(mu), float(rho))


def al_update_multipliers(lam, h, mu, g, rho):
    """Alg. 4 lines 6-7.  Returns (lam', mu')."""
    lam = _f64(np.atleast_1d(lam)).copy() if len(lam) else np.zeros(1)
    mu = _f64(np.atleast_1d(mu)).copy() if len(mu) else np.zeros(1)
    hh = _f64(np.atleast_1d(h)) if len(h) else np.zeros(1)
    gg = _f64(np.atleast_1d(g)) if len(g) else np.zeros(1)
    _L().orc_al_update_multipliers(len(h), _ptr(lam), _ptr(hh), len(g), _ptr(mu), _ptr(gg), float(rho))
    return lam[:len(h)], mu[:len(g)]


def al_update_rho(rho, vprev, v, factor=2.0, cap=1e12):
    """Penalty rule of Alg. 4 (R20)."""
    return _L().orc_al_update_rho(float(rho), float(vprev), float(v), float(factor), float(cap))


def armijo_lsq(P: LSQ, x, p, amax, l=None, u=None, opts: Options | None = None):
    """The oracle's Armijo backtracking on the carried residual (R10, R11, R13)
    from the state (x, r = M~x - b, f, g) along p with upper bound amax.
    Returns (accepted, alpha, f_t, number of rejected trials, x_t)."""
    o = opts or Options()
    x = _f64(x); p = _f64(p)
    l = None if l is None else _f64(np.broadcast_to(l, (P.nvars,)))
    u = None if u is None else _f64(np.broadcast_to(u, (P.nvars,)))
    r = P.apply(x)
    if not P.qp and P.b is not None:
        r = _f64(r - P.b)
    q = _f64(P.apply(p))
    f = P.value(x)
    g = P.grad(x)
    gp = float(np.dot(g, p))
    so = _Opts(o.eps, o.c1, o.shrink, o.tol, o.max_backtracks, int(o.screen_full_norm),
               int(o.no_projection), int(o.armijo_diff), int(o.refresh_every), o.max_iters)
    xt = np.empty(P.nvars); rt = np.empty(max(P.m, 1))
    fo = C.c_double(0.0); ao = C.c_double(0.0); nbt = C.c_int64(0)
    s = P._struct()
    ok = _L().orc_armijo_lsq(C.byref(s), C.byref(so), P.nvars, _ptr(x), _ptr(l), _ptr(u), _ptr(_f64(r)),
                             _ptr(q), _ptr(p), f, gp, float(amax), _ptr(xt), _ptr(rt), C.byref(fo),
                             C.byref(ao), C.byref(nbt))
    return bool(ok), ao.value, fo.value, int(nbt.value), xt


# --------------------------------------------------------------------------
# Generic objective (callback) + general Alg. 4 (linear and nonlinear constraints)
# --------------------------------------------------------------------------
_FG = C.CFUNCTYPE(C.c_int32, C.c_void_p, _dp, _dp, _dp)
_HG = C.CFUNCTYPE(C.c_int32, C.c_void_p, _dp, _dp, _dp)
_JTV = C.CFUNCTYPE(C.c_int32, C.c_void_p, _dp, _dp, _dp, _dp)


class _GCons(C.Structure):
    _fields_ = [("nv", C.c_int64), ("P", C.c_void_p), ("fg", _FG), ("fg_ctx", C.c_void_p),
                ("m_eq", C.c_int32), ("p_in", C.c_int32), ("E", _dp), ("e", _dp), ("G", _dp), ("hv", _dp),
                ("m_nl", C.c_int32), ("p_nl", C.c_int32), ("hg", _HG), ("jtv", _JTV), ("nl_ctx", C.c_void_p)]


def _arr(ptr, n):
    return np.ctypeslib.as_array(ptr, shape=(max(n, 1),))[:n]


def _fg_cb(fun, n):
    """ctypes trampoline for fun(x) -> (f, g) (numpy)."""
    def cb(_ctx, xp, gp, fp):
        try:
            f, g = fun(_arr(xp, n).copy())
            _arr(gp, n)[:] = g
            fp[0] = float(f)
            return 0
        except Exception:          # noqa: BLE001 -- reported as a callback failure
            return 1
    return _FG(cb)


def _setup_general(L):
    L.orc_minimize_fg.argtypes = [C.c_int64, _FG, C.c_void_p, _dp, _dp, C.c_int32, C.POINTER(_Opts), _dp,
                                  C.POINTER(_Res)]
    L.orc_minimize_fg.restype = C.c_int32
    L.orc_al_general.argtypes = [C.POINTER(_GCons), _dp, _dp, _dp, _dp, C.c_int32, C.POINTER(_Opts),
                                 C.POINTER(_AlOpts), _dp, C.c_int32, C.POINTER(_AlRes)]
    L.orc_al_general.restype = C.c_int32


def _opts_c(o):
    return _Opts(o.eps, o.c1, o.shrink, o.tol, o.max_backtracks, int(o.screen_full_norm),
                 int(o.no_projection), int(o.armijo_diff), int(o.refresh_every), o.max_iters)


def minimize_fg(fun, n, l=None, u=None, x0=None, m_hist=5, opts: Options | None = None):
    """Alg. 1 on a generic objective fun(x) -> (f, grad) with every
    trial value evaluated (orc_minimize_fg)."""
    L = _L(); _setup_general(L)
    o = opts or Options()
    x = np.zeros(n) if x0 is None else _f64(x0).copy()
    l = None if l is None else _f64(np.broadcast_to(l, (n,)))
    u = None if u is None else _f64(np.broadcast_to(u, (n,)))
    cb = _fg_cb(fun, n)
    res = _Res()
    so = _opts_c(o)
    rc = L.orc_minimize_fg(n, cb, None, _ptr(l), _ptr(u), m_hist, C.byref(so), _ptr(x), C.byref(res))
    if rc:
        raise RuntimeError(f"objective callback failed ({rc})")
    return Result(x, res.f, res.pg_inf, res.gfree_inf, res.iters, res.n_fg, res.n_backtracks,
                  res.n_free, res.status, res.last_branch, res.n_fallbacks)


def al_general(n, base=None, fun=None, E=None, e=None, G=None, hv=None, m_nl=0, p_nl=0, hg=None, jtv=None,
               l=None, u=None, m_hist=5, opts: Options | None = None, al_opts: ALOptions | None = None,
               x0=None, lam0=None, mu0=None):
    """Alg. 4 on min f(x) s.t. h(x) = 0, g(x) <= 0, l <= x <= u
    with h = [E^T x - e; h_nl(x)], g = [G^T x - hv; g_nl(x)] (orc_al_general).
    base: an LSQ (no constraints of its own) or None with fun(x) -> (f, grad);
    hg(x) -> (h_nl (m_nl), g_nl (p_nl)); jtv(x, v_eq, v_in) -> J_h^T v_eq + J_g^T v_in.
    Cold start unless x0 / lam0 / mu0 is given (warm re-entry)."""
    L = _L(); _setup_general(L)
    o = opts or Options(); ao = al_opts or ALOptions()
    E = None if E is None else np.asfortranarray(np.reshape(E, (n, -1)), dtype=np.float64)
    G = None if G is None else np.asfortranarray(np.reshape(G, (n, -1)), dtype=np.float64)
    m_eq = 0 if E is None else E.shape[1]
    p_in = 0 if G is None else G.shape[1]
    e = None if e is None else _f64(np.atleast_1d(e))
    hv = None if hv is None else _f64(np.atleast_1d(hv))
    neq, nin = m_eq + m_nl, p_in + p_nl
    keep = []
    s = _GCons()
    s.nv = n
    if base is not None:
        assert base.n_eq == 0 and base.n_in == 0
        bs = base._struct(); keep.append(bs)
        s.P = C.cast(C.pointer(bs), C.c_void_p)
        s.fg = _FG(0)
    else:
        s.P = None
        s.fg = _fg_cb(fun, n)
    keep.append(s.fg)
    s.m_eq, s.p_in, s.E, s.e, s.G, s.hv = m_eq, p_in, _ptr(E), _ptr(e), _ptr(G), _ptr(hv)
    s.m_nl, s.p_nl = m_nl, p_nl
    if m_nl + p_nl:
        def hg_c(_ctx, xp, hp, gp):
            try:
                h_, g_ = hg(_arr(xp, n).copy())
                if m_nl:
                    _arr(hp, m_nl)[:] = h_
                if p_nl:
                    _arr(gp, p_nl)[:] = g_
                return 0
            except Exception:      # noqa: BLE001
                return 1

        def jtv_c(_ctx, xp, ve, vi, op):
            try:
                _arr(op, n)[:] = jtv(_arr(xp, n).copy(), _arr(ve, m_nl).copy(), _arr(vi, p_nl).copy())
                return 0
            except Exception:      # noqa: BLE001
                return 1
        s.hg, s.jtv = _HG(hg_c), _JTV(jtv_c)
    else:
        s.hg, s.jtv = _HG(0), _JTV(0)
    keep += [s.hg, s.jtv]
    warm = x0 is not None or lam0 is not None or mu0 is not None
    x = np.zeros(n) if x0 is None else _f64(x0).copy()
    lam = np.zeros(max(neq, 1)); mu = np.zeros(max(nin, 1))
    if lam0 is not None:
        lam[:neq] = lam0
    if mu0 is not None:
        mu[:nin] = mu0
    l = None if l is None else _f64(np.broadcast_to(l, (n,)))
    u = None if u is None else _f64(np.broadcast_to(u, (n,)))
    so = _opts_c(o)
    sa = _AlOpts(ao.feas_tol, ao.rho0, ao.rho_factor, ao.rho_cap, ao.max_outer)
    res = _AlRes()
    rc = L.orc_al_general(C.byref(s), _ptr(lam), _ptr(mu), _ptr(l), _ptr(u), m_hist, C.byref(so), C.byref(sa),
                          _ptr(x), int(warm), C.byref(res))
    if rc:
        raise RuntimeError(f"callback failed ({rc})")
    return ALResult(x, lam[:neq].copy(), mu[:nin].copy(), res.f, res.violation_inf, res.rho,
                    res.outer_iters, res.inner_iters_total, res.status)
