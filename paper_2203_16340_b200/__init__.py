"""paper_2203_16340_b200 -- B200-native (sm_100a, fp64) hot path of the
GPU-efficient, Cauchy-point-free L-BFGS-B of arXiv 2203.16340 (Alg. 1-3) and
its augmented-Lagrangian wrapper (Alg. 4).

This module is a THIN ctypes binding over the C ABI of ``include/lbfgsb.h``
and ``include/lbfgsb_ops.h`` (``liblbfgsb.so``, built in-tree by
``_build.py``): argument marshalling only, every step of the method runs in
the library's CUDA kernels.  PyTorch is used for device memory and streams.
There is no CPU fallback: if the extension is missing or no GPU is usable,
calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

from . import _build

__all__ = ["Options", "ALOptions", "Result", "ALResult", "Solver", "LSQObjective",
           "CallbackObjective", "op_gemv", "op_gemvt", "load", "LbfgsbError", "colmajor",
           "solve_loopback", "nccl_unique_id", "QPObjective", "op_gaussian_kernel",
           "TransportObjective", "solve_batched_lsq", "colmajor_batch", "p2p_connect_local",
           "p2p_open_group", "solve_group"]

_c_d, _c_i32, _c_i64, _c_vp = C.c_double, C.c_int32, C.c_int64, C.c_void_p

CONVERGED, MAX_ITERS, LINESEARCH_FAILURE, AL_MAX_OUTER, AL_INNER_FAILURE = 0, 1, 2, 3, 4
STATUS_NAMES = {0: "converged", 1: "max_iters", 2: "linesearch_failure", 3: "al_max_outer",
                4: "al_inner_failure"}


class _Opts(C.Structure):
    _fields_ = [("eps", _c_d), ("c1", _c_d), ("shrink", _c_d), ("tol", _c_d),
                ("max_backtracks", _c_i32), ("screen_full_norm", _c_i32),
                ("check_every", _c_i32), ("use_graph", _c_i32), ("profile", _c_i32),
                ("no_projection", _c_i32), ("armijo_diff", _c_i32), ("refresh_every", _c_i32),
                ("trials_per_pass", _c_i32), ("max_iters", _c_i64)]


class _Res(C.Structure):
    _fields_ = [("f", _c_d), ("pg_inf", _c_d), ("gfree_inf", _c_d), ("seconds", _c_d),
                ("iters", _c_i64), ("n_fg", _c_i64), ("n_backtracks", _c_i64),
                ("n_free", _c_i64), ("n_fallbacks", _c_i64), ("status", _c_i32),
                ("last_branch", _c_i32)]


class _AlOpts(C.Structure):
    _fields_ = [("feas_tol", _c_d), ("rho0", _c_d), ("rho_factor", _c_d), ("rho_cap", _c_d),
                ("max_outer", _c_i32), ("warm_start", _c_i32)]


HG_CB = C.CFUNCTYPE(_c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp)
JTV_CB = C.CFUNCTYPE(_c_i32, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp)


class _AlCons(C.Structure):
    _fields_ = [("m_eq", _c_i64), ("p_in", _c_i64), ("E", _c_vp), ("e", C.POINTER(_c_d)),
                ("G", _c_vp), ("hv", C.POINTER(_c_d)), ("m_nl", _c_i64), ("p_nl", _c_i64),
                ("hg", HG_CB), ("jtv", JTV_CB), ("user", _c_vp)]


class _AlRes(C.Structure):
    _fields_ = [("violation_inf", _c_d), ("f", _c_d), ("rho", _c_d), ("pg_inf", _c_d),
                ("outer_iters", _c_i64), ("inner_iters_total", _c_i64), ("status", _c_i32),
                ("pad_", _c_i32)]


FG_CB = C.CFUNCTYPE(_c_i32, _c_vp, _c_vp, _c_vp, C.POINTER(_c_d), _c_vp)

_lib = None


class LbfgsbError(RuntimeError):
    pass


def load(build_if_needed: bool = True):
    """Load liblbfgsb.so (building it with nvcc if sources changed)."""
    global _lib
    if _lib is not None:
        return _lib
    if build_if_needed and _build.needs_build():
        _build.build()
    if not os.path.exists(_build.LIB):
        raise LbfgsbError(f"CUDA extension missing: {_build.LIB} (run _build.py); no CPU fallback")
    L = C.CDLL(_build.LIB)
    ip, vp = C.POINTER(_c_i32), _c_vp
    L.lbfgsb_last_error.restype = C.c_char_p
    L.lbfgsb_opts_default.argtypes = [C.POINTER(_Opts)]
    L.al_opts_default.argtypes = [C.POINTER(_AlOpts)]
    L.lbfgsb_create.argtypes = [_c_i64, _c_i32, vp, vp, C.POINTER(_Opts), vp, C.POINTER(vp)]
    L.lbfgsb_create_sharded.argtypes = [_c_i64, _c_i64, _c_i32, vp, vp, C.POINTER(_Opts), vp, vp,
                                        _c_i32, _c_i32, C.POINTER(vp)]
    L.lbfgsb_destroy.argtypes = [vp]
    L.lbfgsb_objective_lsq.argtypes = [vp, _c_i64, _c_i64, _c_i64, vp, _c_i32, vp, vp, _c_d,
                                       C.POINTER(vp)]
    L.lbfgsb_objective_callback.argtypes = [FG_CB, vp, C.POINTER(vp)]
    L.lbfgsb_objective_free.argtypes = [vp]
    L.lbfgsb_solve.argtypes = [vp, vp, vp, _c_d, C.POINTER(_Res)]
    L.lbfgsb_solve_lsq_host.argtypes = [vp, vp, _c_i64, _c_i64, vp, vp, _c_d, C.POINTER(_Res)]
    L.al_solve.argtypes = [vp, vp, C.POINTER(_AlCons), C.POINTER(_AlOpts), vp, vp, vp,
                           C.POINTER(_AlRes)]
    L.lbfgsb_op_gemv.argtypes = [vp, vp, vp, vp]
    L.lbfgsb_op_gemvt.argtypes = [vp, vp, vp, vp]
    L.lbfgsb_op_direction.argtypes = [vp, vp, vp, _c_i32, vp, vp, vp, vp, vp, ip,
                                      C.POINTER(_c_d), C.POINTER(_c_d)]
    L.lbfgsb_op_trials.argtypes = [vp, vp, vp, vp, vp, vp, _c_d, _c_i32, C.POINTER(_c_d)]
    L.lbfgsb_profile_get.argtypes = [vp, _c_i32, C.POINTER(C.c_char_p), C.POINTER(_c_d),
                                     C.POINTER(_c_i64), ip, _c_i32]
    L.lbfgsb_solve_loopback.argtypes = [C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), _c_i32, _c_d,
                                        C.POINTER(_Res)]
    L.lbfgsb_nccl_unique_id.argtypes = [vp]
    L.lbfgsb_create_sharded_p2p.argtypes = [_c_i64, _c_i64, _c_i32, vp, vp, C.POINTER(_Opts), vp, _c_i32,
                                            _c_i32, _c_i64, C.POINTER(vp)]
    L.lbfgsb_p2p_ipc_handle.argtypes = [vp, vp]
    L.lbfgsb_p2p_open.argtypes = [vp, vp]
    L.lbfgsb_p2p_connect_local.argtypes = [C.POINTER(vp), _c_i32, _c_i64]
    L.lbfgsb_p2p_open_group.argtypes = [C.POINTER(vp), _c_i32, vp]
    L.lbfgsb_solve_group.argtypes = [C.POINTER(vp), C.POINTER(vp), C.POINTER(vp), _c_i32, _c_d,
                                     C.POINTER(_Res)]
    L.lbfgsb_solve_lsq_host_batch.argtypes = [vp, _c_i32, C.POINTER(vp), _c_i64, _c_i64, C.POINTER(vp),
                                              C.POINTER(vp), _c_d, C.POINTER(_Res)]
    L.lbfgsb_objective_qp.argtypes = [vp, _c_i64, _c_i64, vp, vp, _c_d, C.POINTER(vp)]
    L.lbfgsb_op_gaussian_kernel.argtypes = [vp, _c_i64, _c_i64, _c_d, vp, _c_i64, vp]
    L.lbfgsb_objective_transport.argtypes = [vp, _c_i64, _c_i64, _c_i32, _c_d, C.POINTER(vp)]
    L.lbfgsb_solve_original.argtypes = [vp, vp, vp, _c_d, C.POINTER(_Res), C.POINTER(_c_d)]
    L.lbfgsb_solve_batched_lsq.argtypes = [_c_i32, _c_i64, _c_i64, vp, vp, vp, vp, vp, _c_i32,
                                           C.POINTER(_Opts), _c_d, vp, C.POINTER(_Res)]
    L.lbfgsb_op_cauchy_point.argtypes = [vp, vp, vp, _c_i32, vp, vp, _c_d, vp, C.POINTER(_c_d),
                                         C.POINTER(_c_i64), C.POINTER(_c_d)]
    L.al_solve_transport.argtypes = [vp, vp, vp, vp, C.POINTER(_AlOpts), vp, vp, C.POINTER(_AlRes)]
    for name in ("lbfgsb_objective_transport", "al_solve_transport", "lbfgsb_op_cauchy_point",
                 "lbfgsb_solve_batched_lsq", "lbfgsb_solve_original",
                 "lbfgsb_create", "lbfgsb_create_sharded", "lbfgsb_objective_lsq",
                 "lbfgsb_objective_callback", "lbfgsb_solve", "lbfgsb_solve_lsq_host", "al_solve",
                 "lbfgsb_op_gemv", "lbfgsb_op_gemvt", "lbfgsb_op_direction", "lbfgsb_op_trials",
                 "lbfgsb_profile_get", "lbfgsb_solve_loopback", "lbfgsb_nccl_unique_id",
                 "lbfgsb_objective_qp", "lbfgsb_op_gaussian_kernel", "lbfgsb_create_sharded_p2p",
                 "lbfgsb_p2p_ipc_handle", "lbfgsb_p2p_open", "lbfgsb_p2p_connect_local",
                 "lbfgsb_p2p_open_group", "lbfgsb_solve_group",
                 "lbfgsb_solve_lsq_host_batch"):
        getattr(L, name).restype = _c_i32
    _lib = L
    return L


def _check(rc):
    if rc != 0:
        msg = _lib.lbfgsb_last_error().decode()
        raise LbfgsbError(f"liblbfgsb error {rc}: {msg}")


def _ptr(t):
    """Device pointer of a CUDA tensor (None -> NULL)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise LbfgsbError("expected a CUDA tensor (the library has no CPU path)")
    if t.dtype.itemsize != 8 and t.dtype.is_floating_point:
        raise LbfgsbError("fp64 tensors required")
    return C.c_void_p(t.data_ptr())


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream) if s.cuda_stream else None


def colmajor(A, device="cuda"):
    """numpy (m, n) array -> torch fp64 CUDA tensor (m, n) with column-major
    strides (1, m), the layout of the C ABI."""
    import numpy as np
    import torch
    At = np.ascontiguousarray(np.asarray(A, dtype=np.float64).T)   # (n, m) row-major
    return torch.from_numpy(At).to(device).T


@dataclass
class Options:
    eps: float = 1e-9
    c1: float = 1e-4
    shrink: float = 0.5
    tol: float = 1e-6
    max_backtracks: int = 50
    screen_full_norm: bool = False
    check_every: int = 8
    use_graph: bool = True
    profile: bool = False
    max_iters: int = 10000
    no_projection: bool = False
    armijo_diff: bool = False       # R29: Armijo on the expanded difference f(x + a p) - f(x)
    refresh_every: int = 0          # R13: exact r, f, g every R iterations (0: final refresh only)
    trials_per_pass: int = 0        # Armijo trials decided per fused pass (1..16; 0 = 16)

    def _c(self):
        return _Opts(self.eps, self.c1, self.shrink, self.tol, self.max_backtracks,
                     int(bool(self.screen_full_norm)), self.check_every, int(bool(self.use_graph)),
                     int(bool(self.profile)), int(bool(self.no_projection)),
                     int(bool(self.armijo_diff)), int(self.refresh_every), int(self.trials_per_pass),
                     self.max_iters)


@dataclass
class ALOptions:
    feas_tol: float = 1e-6
    rho0: float = 1.0
    rho_factor: float = 2.0
    rho_cap: float = 1e12
    max_outer: int = 100


@dataclass
class Result:
    f: float
    pg_inf: float
    gfree_inf: float
    seconds: float
    iters: int
    n_fg: int
    n_backtracks: int
    n_free: int
    n_fallbacks: int
    status: int
    last_branch: int

    @property
    def status_name(self):
        return STATUS_NAMES.get(self.status, str(self.status))

    @classmethod
    def from_c(cls, r):
        return cls(r.f, r.pg_inf, r.gfree_inf, r.seconds, r.iters, r.n_fg, r.n_backtracks, r.n_free,
                   r.n_fallbacks, r.status, r.last_branch)


@dataclass
class ALResult:
    violation_inf: float
    f: float
    rho: float
    pg_inf: float
    outer_iters: int
    inner_iters_total: int
    status: int
    lam: list
    mu: list


class LSQObjective:
    """f(x) = 1/2||M~x - b||^2 + c^T x + delta/2||x||^2, M~ = M diag(colscale)
    or [M, -M] (split).  M: CUDA fp64 tensor (m, ncols) with column-major
    strides (see ``colmajor``); b (m), c (nvars), colscale (ncols): CUDA fp64."""

    def __init__(self, M, b=None, c=None, delta=0.0, colscale=None, split=False):
        L = load()
        if M.dim() != 2 or (M.stride(0) != 1 and M.shape[0] > 1):
            raise LbfgsbError("M must be (m, ncols) column-major: M.stride(0) == 1")
        self.m, self.ncols = M.shape
        self.ld = max(M.stride(1), self.m) if self.ncols > 1 else self.m
        self.split = bool(split)
        self.nvars = 2 * self.ncols if split else self.ncols
        self._keep = (M, b, c, colscale)      # borrowed by the C objective
        h = C.c_void_p()
        _check(L.lbfgsb_objective_lsq(_ptr(M), self.m, self.ncols, self.ld, _ptr(colscale),
                                      int(self.split), _ptr(b), _ptr(c), float(delta),
                                      C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.lbfgsb_objective_free(self._h)
            self._h = None


class QPObjective(LSQObjective):
    """f(x) = 1/2 x^T D Q D x + c^T x + delta/2||x||^2 (lbfgsb_objective_qp): Q CUDA fp64
    (n, n) symmetric column-major, D = diag(colscale) (e.g. the SVM labels)."""

    def __init__(self, Q, c=None, delta=0.0, colscale=None):   # noqa: D107 -- no super().__init__
        L = load()
        if Q.dim() != 2 or Q.shape[0] != Q.shape[1] or (Q.stride(0) != 1 and Q.shape[0] > 1):
            raise LbfgsbError("Q must be square (n, n) column-major")
        self.m = self.ncols = self.nvars = Q.shape[0]
        self.ld = max(Q.stride(1), self.m) if self.ncols > 1 else self.m
        self.split = False
        self._keep = (Q, c, colscale)
        h = C.c_void_p()
        _check(L.lbfgsb_objective_qp(_ptr(Q), self.m, self.ld, _ptr(colscale), _ptr(c), float(delta),
                                     C.byref(h)))
        self._h = h


class TransportObjective(LSQObjective):
    """Joint probability / regularised OT (lbfgsb_objective_transport):
    f(P) = <M, P> + lam r(P), r = sum P log P ("entropy") or 1/2||P||^2
    ("gaussian"); M CUDA fp64 (m, n) column-major; variables vec(P) (m*n)."""

    def __init__(self, M, reg="entropy", lam=0.5):   # noqa: D107 -- no super().__init__
        L = load()
        if M.dim() != 2 or (M.stride(0) != 1 and M.shape[0] > 1) or \
                (M.shape[1] > 1 and M.stride(1) != M.shape[0]):
            raise LbfgsbError("M must be (m, n) column-major with ld = m")
        if reg not in ("entropy", "gaussian"):
            raise LbfgsbError("reg must be 'entropy' or 'gaussian'")
        self.m, self.n = M.shape
        self.nvars = self.m * self.n
        self.reg = reg
        self._keep = (M,)
        h = C.c_void_p()
        _check(L.lbfgsb_objective_transport(_ptr(M), self.m, self.n, 0 if reg == "entropy" else 1,
                                            float(lam), C.byref(h)))
        self._h = h


class CallbackObjective:
    """User objective: ``fg(x, g) -> f`` with x, g CUDA fp64 tensors (g written
    in place).  Runs on the current torch stream."""

    def __init__(self, fg, n):
        import torch
        L = load()
        self.n = n
        self.nvars = n
        self._err = None

        def _cb(user, xp, gp, fhost, stream):
            try:
                x = _wrap(xp, n)
                g = _wrap(gp, n)
                f = fg(x, g)
                fhost[0] = float(f)
                torch.cuda.current_stream().synchronize()
                return 0
            except Exception as e:  # noqa: BLE001 -- surfaced after the call
                self._err = e
                return 1

        self._cb = FG_CB(_cb)
        h = C.c_void_p()
        _check(L.lbfgsb_objective_callback(self._cb, None, C.byref(h)))
        self._h = h

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.lbfgsb_objective_free(self._h)
            self._h = None


def _wrap(ptr, n):
    """Non-owning torch view of a library device buffer (valid during the callback)."""
    import torch

    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_CAI(), device="cuda")


class Solver:
    """lbfgsb_create handle: n variables, box [lower, upper] (CUDA fp64 tensors
    or None for -inf / +inf), m_hist curvature pairs.  With ``nccl_id`` (the
    128-byte ncclUniqueId), ``rank`` and ``nranks`` it is an
    lbfgsb_create_sharded handle owning n of ``n_global`` variables.  With
    ``p2p_m_max`` instead (and rank / nranks) it is an
    lbfgsb_create_sharded_p2p handle: the exchange runs over peer memory
    (connect with ipc_handle() on every rank, then p2p_open(all handles))."""

    def __init__(self, n, m_hist=5, lower=None, upper=None, opts: Options | None = None,
                 stream=None, nccl_id: bytes | None = None, rank=0, nranks=1, n_global=None,
                 p2p_m_max: int | None = None):
        L = load()
        self.n = int(n)
        self.m_hist = int(m_hist)
        self.opts = opts or Options()
        o = self.opts._c()
        h = C.c_void_p()
        if p2p_m_max is not None:
            _check(L.lbfgsb_create_sharded_p2p(self.n, int(n_global if n_global is not None else n),
                                               self.m_hist, _ptr(lower), _ptr(upper), C.byref(o),
                                               _stream_ptr(stream), int(rank), int(nranks),
                                               int(p2p_m_max), C.byref(h)))
        elif nccl_id is None:
            _check(L.lbfgsb_create(self.n, self.m_hist, _ptr(lower), _ptr(upper), C.byref(o),
                                   _stream_ptr(stream), C.byref(h)))
        else:
            idb = C.create_string_buffer(bytes(nccl_id), 128)
            _check(L.lbfgsb_create_sharded(self.n, int(n_global if n_global is not None else n),
                                           self.m_hist, _ptr(lower), _ptr(upper), C.byref(o),
                                           _stream_ptr(stream), C.cast(idb, C.c_void_p), int(rank),
                                           int(nranks), C.byref(h)))
        self._h = h

    def ipc_handle(self) -> bytes:
        """lbfgsb_p2p_ipc_handle: the 64-byte CUDA IPC handle of this rank's mailbox."""
        buf = C.create_string_buffer(64)
        _check(_lib.lbfgsb_p2p_ipc_handle(self._h, C.cast(buf, C.c_void_p)))
        return buf.raw

    def p2p_open(self, handles):
        """lbfgsb_p2p_open: map the mailboxes of all ranks (list of 64-byte handles, rank order)."""
        blob = C.create_string_buffer(b"".join(bytes(h) for h in handles), 64 * len(handles))
        _check(_lib.lbfgsb_p2p_open(self._h, C.cast(blob, C.c_void_p)))

    def close(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.lbfgsb_destroy(self._h)
            self._h = None

    __del__ = close

    def solve(self, obj, x, tol=0.0) -> Result:
        """Alg. 1 from x (CUDA fp64 tensor, updated in place with x*)."""
        r = _Res()
        rc = _lib.lbfgsb_solve(self._h, obj._h, _ptr(x), float(tol), C.byref(r))
        if isinstance(obj, CallbackObjective) and obj._err is not None:
            e, obj._err = obj._err, None
            raise LbfgsbError(f"callback raised: {e!r}") from e
        _check(rc)
        return Result(r.f, r.pg_inf, r.gfree_inf, r.seconds, r.iters, r.n_fg, r.n_backtracks,
                      r.n_free, r.n_fallbacks, r.status, r.last_branch)

    def solve_lsq_host(self, M_host, b_host, x_host, tol=0.0) -> Result:
        """lbfgsb_solve_lsq_host: numpy (pinned or pageable) buffers in/out.
        M_host: (m, n) Fortran-ordered float64; b_host (m); x_host (n, in/out)."""
        import numpy as np
        assert M_host.flags.f_contiguous and M_host.dtype == np.float64
        assert x_host.flags.c_contiguous and x_host.dtype == np.float64
        m, n = M_host.shape
        r = _Res()
        _check(_lib.lbfgsb_solve_lsq_host(self._h, C.c_void_p(M_host.ctypes.data), m, n,
                                          C.c_void_p(b_host.ctypes.data) if b_host is not None else None,
                                          C.c_void_p(x_host.ctypes.data), float(tol), C.byref(r)))
        return Result(r.f, r.pg_inf, r.gfree_inf, r.seconds, r.iters, r.n_fg, r.n_backtracks,
                      r.n_free, r.n_fallbacks, r.status, r.last_branch)

    def solve_lsq_host_batch(self, Ms, bs, xs, tol=0.0):
        """lbfgsb_solve_lsq_host_batch: len(Ms) problems from host numpy buffers
        (M: (m, n) Fortran-ordered float64, b: (m) or None, x: (n) in/out),
        the next problem's H2D overlapping the current solve."""
        import numpy as np
        k = len(Ms)
        if not (len(xs) == k and (bs is None or len(bs) == k)):
            raise LbfgsbError("Ms, bs, xs lengths differ")
        if k == 0:
            return []
        m, n = Ms[0].shape
        for M_, x_ in zip(Ms, xs):
            assert M_.flags.f_contiguous and M_.dtype == np.float64 and M_.shape == (m, n)
            assert x_.flags.c_contiguous and x_.dtype == np.float64 and x_.shape == (n,)
        Mp = (_c_vp * k)(*[M_.ctypes.data for M_ in Ms])
        bp = (_c_vp * k)(*[(b_.ctypes.data if b_ is not None else None) for b_ in bs]) if bs is not None else None
        xp = (_c_vp * k)(*[x_.ctypes.data for x_ in xs])
        res = (_Res * k)()
        _check(_lib.lbfgsb_solve_lsq_host_batch(self._h, k, Mp, m, n, bp, xp, float(tol), res))
        return [Result(r.f, r.pg_inf, r.gfree_inf, r.seconds, r.iters, r.n_fg, r.n_backtracks,
                       r.n_free, r.n_fallbacks, r.status, r.last_branch) for r in res]

    def al_solve(self, obj, x, E=None, e=None, G=None, hv=None,
                 al_opts: ALOptions | None = None, hg=None, jtv=None, m_nl=0, p_nl=0,
                 lam0=None, mu0=None, warm_start=False) -> ALResult:
        """Alg. 4 (al_solve): linear constraints E^T x = e, G^T x <= hv (E (n, m_eq),
        G (n, p_in) CUDA fp64; any number of them) and nonlinear ones through
        hg(x, h_out, g_out) (h_out (m_nl), g_out (p_nl) CUDA views written in place)
        and jtv(x, v_eq, v_in, out) (out (n) = J_h^T v_eq + J_g^T v_in).  obj: an
        LSQObjective or a CallbackObjective.  warm_start: re-enter from x and
        lam0 / mu0 (host sequences of m_eq + m_nl / p_in + p_nl) instead of
        x = clip(0), lambda = mu = 0."""
        import torch
        ao = al_opts or ALOptions()
        c_ao = _AlOpts(ao.feas_tol, ao.rho0, ao.rho_factor, ao.rho_cap, ao.max_outer, int(bool(warm_start)))
        m_eq = 0 if E is None else (E.shape[1] if E.dim() == 2 else 1)
        p_in = 0 if G is None else (G.shape[1] if G.dim() == 2 else 1)
        Ec = None if E is None else E.reshape(self.n, m_eq).T.contiguous()   # (m_eq, n) rows = columns
        Gc = None if G is None else G.reshape(self.n, p_in).T.contiguous()
        e_arr = (_c_d * max(m_eq, 1))(*([float(v) for v in torch.as_tensor(e).flatten()] if m_eq else [0.0]))
        h_arr = (_c_d * max(p_in, 1))(*([float(v) for v in torch.as_tensor(hv).flatten()] if p_in else [0.0]))
        n = self.n
        errs = []

        def _hg(user, xp, hp, gp, stream):
            try:
                hg(_wrap(xp, n), _wrap(hp, m_nl) if m_nl else None, _wrap(gp, p_nl) if p_nl else None)
                torch.cuda.current_stream().synchronize()
                return 0
            except Exception as ex:          # noqa: BLE001 -- surfaced after the call
                errs.append(ex)
                return 1

        def _jtv(user, xp, vep, vip, op, stream):
            try:
                jtv(_wrap(xp, n), _wrap(vep, m_nl) if m_nl else None, _wrap(vip, p_nl) if p_nl else None,
                    _wrap(op, n))
                torch.cuda.current_stream().synchronize()
                return 0
            except Exception as ex:          # noqa: BLE001
                errs.append(ex)
                return 1
        nl = (m_nl + p_nl) > 0
        hg_c = HG_CB(_hg) if nl else HG_CB(0)
        jtv_c = JTV_CB(_jtv) if nl else JTV_CB(0)
        cons = _AlCons(m_eq, p_in, _ptr(Ec), e_arr, _ptr(Gc), h_arr, int(m_nl), int(p_nl), hg_c, jtv_c, None)
        neq, nin = m_eq + m_nl, p_in + p_nl
        lam = (_c_d * max(neq, 1))(*(list(map(float, lam0)) if lam0 is not None else []))
        mu = (_c_d * max(nin, 1))(*(list(map(float, mu0)) if mu0 is not None else []))
        r = _AlRes()
        rc = _lib.al_solve(self._h, obj._h, C.byref(cons), C.byref(c_ao), _ptr(x), lam, mu, C.byref(r))
        if isinstance(obj, CallbackObjective) and obj._err is not None:
            e_, obj._err = obj._err, None
            raise LbfgsbError(f"objective callback raised: {e_!r}") from e_
        if errs:
            raise LbfgsbError(f"constraint callback raised: {errs[0]!r}") from errs[0]
        _check(rc)
        return ALResult(r.violation_inf, r.f, r.rho, r.pg_inf, r.outer_iters, r.inner_iters_total,
                        r.status, list(lam)[:neq], list(mu)[:nin])

    def al_solve_transport(self, obj, x, u, v, lam_out=None,
                           al_opts: ALOptions | None = None) -> ALResult:
        """Alg. 4 with the marginal equalities P 1 = u, P^T 1 = v (u, v CUDA fp64);
        x (m*n) out = vec(P*) column-major; lam_out (m+n, CUDA) receives the multipliers."""
        ao = al_opts or ALOptions()
        c_ao = _AlOpts(ao.feas_tol, ao.rho0, ao.rho_factor, ao.rho_cap, ao.max_outer, 0)
        r = _AlRes()
        _check(_lib.al_solve_transport(self._h, obj._h, _ptr(u), _ptr(v), C.byref(c_ao), _ptr(x),
                                       _ptr(lam_out), C.byref(r)))
        return ALResult(r.violation_inf, r.f, r.rho, r.pg_inf, r.outer_iters, r.inner_iters_total,
                        r.status, [], [])

    # ---- op-level entry points (lbfgsb_ops.h) ----
    def solve_original(self, obj, x, tol: float = 0.0):
        """The original L-BFGS-B (SURVEY N3 baseline): returns (Result, Cauchy-point ms)."""
        r = _Res()
        ms = _c_d()
        _check(_lib.lbfgsb_solve_original(self._h, obj._h, _ptr(x), float(tol), C.byref(r), C.byref(ms)))
        return Result.from_c(r), ms.value

    def op_cauchy_point(self, x, g, S=None, Y=None, theta=1.0):
        """Generalized Cauchy point of the original L-BFGS-B (baseline):
        returns dict(xcp, c, passed, scan_ms)."""
        import torch
        nh = 0 if S is None else S.shape[0]
        xcp = torch.empty_like(x)
        c = (_c_d * max(2 * nh, 1))()
        passed = _c_i64()
        ms = _c_d()
        Sc = None if S is None else S.contiguous()
        Yc = None if Y is None else Y.contiguous()
        _check(_lib.lbfgsb_op_cauchy_point(self._h, _ptr(x), _ptr(g), nh, _ptr(Sc), _ptr(Yc), float(theta),
                                           _ptr(xcp), c, C.byref(passed), C.byref(ms)))
        return dict(xcp=xcp, c=list(c)[:2 * nh], passed=passed.value, scan_ms=ms.value)

    def op_direction(self, x, g, S=None, Y=None):
        """Working set + vector-free Alg. 3 + Alg. 2 on (x, g, pairs oldest first)."""
        import torch
        nh = 0 if S is None else S.shape[0]
        fr = torch.empty(self.n, dtype=torch.uint8, device=x.device)
        d = torch.empty_like(x)
        p = torch.empty_like(x)
        br = _c_i32()
        gp, am = _c_d(), _c_d()
        Sc = None if S is None else S.contiguous()
        Yc = None if Y is None else Y.contiguous()
        _check(_lib.lbfgsb_op_direction(self._h, _ptr(x), _ptr(g), nh, _ptr(Sc), _ptr(Yc),
                                        _ptr(fr), _ptr(d), _ptr(p), C.byref(br), C.byref(gp),
                                        C.byref(am)))
        return dict(free=fr.bool(), d=d, p=p, projected=bool(br.value), gp=gp.value, amax=am.value)

    def op_trials(self, obj, r, q, x, p, alpha0, ntrials=16):
        f = (_c_d * ntrials)()
        _check(_lib.lbfgsb_op_trials(self._h, obj._h, _ptr(r), _ptr(q), _ptr(x), _ptr(p),
                                     float(alpha0), ntrials, f))
        return list(f)

    def profile(self, reset=False):
        names = (C.c_char_p * 8)()
        ms = (_c_d * 8)()
        cnt = (_c_i64 * 8)()
        k = _c_i32()
        _check(_lib.lbfgsb_profile_get(self._h, 8, names, ms, cnt, C.byref(k), int(bool(reset))))
        return {names[i].decode(): (ms[i], cnt[i]) for i in range(k.value)}


def nccl_unique_id() -> bytes:
    """lbfgsb_nccl_unique_id: 128 bytes to broadcast from rank 0."""
    buf = C.create_string_buffer(128)
    _check(load().lbfgsb_nccl_unique_id(C.cast(buf, C.c_void_p)))
    return buf.raw


def p2p_connect_local(solvers, m_max):
    """lbfgsb_p2p_connect_local: give len(solvers) single-GPU handles wired
    mailboxes so that solve_loopback runs the P2P exchange protocol."""
    R = len(solvers)
    hs = (_c_vp * R)(*[s._h.value for s in solvers])
    _check(load().lbfgsb_p2p_connect_local(hs, R, int(m_max)))


def p2p_open_group(solvers, handles):
    """lbfgsb_p2p_open_group: wire the logical ranks this process hosts
    (P2P-sharded Solvers) to all C mailboxes (``handles``: the 64-byte IPC
    handles of every logical rank, in logical-rank order)."""
    R = len(solvers)
    hs = (_c_vp * R)(*[s._h.value for s in solvers])
    blob = b"".join(handles)
    _check(load().lbfgsb_p2p_open_group(hs, R, C.cast(C.create_string_buffer(blob, len(blob)), C.c_void_p)))


def solve_group(solvers, objs, xs, tol=0.0) -> Result:
    """lbfgsb_solve_group: one P2P-sharded solve over the logical ranks this
    process hosts (bitwise independent of the process / GPU count)."""
    R = len(solvers)
    hs = (_c_vp * R)(*[s._h.value for s in solvers])
    os_ = (_c_vp * R)(*[o._h.value for o in objs])
    xp = (_c_vp * R)(*[x.data_ptr() for x in xs])
    r = _Res()
    _check(load().lbfgsb_solve_group(hs, os_, xp, R, float(tol), C.byref(r)))
    return Result.from_c(r)


def solve_loopback(solvers, objs, xs, tol=0.0) -> Result:
    """lbfgsb_solve_loopback: the column-sharded path with len(solvers) logical
    ranks on one GPU (verification of the NCCL path's exchange and decisions)."""
    R = len(solvers)
    hs = (_c_vp * R)(*[s._h.value for s in solvers])
    os_ = (_c_vp * R)(*[o._h.value for o in objs])
    xp = (_c_vp * R)(*[x.data_ptr() for x in xs])
    r = _Res()
    _check(load().lbfgsb_solve_loopback(hs, os_, xp, R, float(tol), C.byref(r)))
    return Result(r.f, r.pg_inf, r.gfree_inf, r.seconds, r.iters, r.n_fg, r.n_backtracks,
                  r.n_free, r.n_fallbacks, r.status, r.last_branch)


def op_gaussian_kernel(X, gamma, stream=None):
    """K = exp(-gamma ||x_i - x_j||^2) for X (N, d) row-major CUDA fp64; returns K (N, N)
    column-major (lbfgsb_op_gaussian_kernel)."""
    import torch
    N, d = X.shape
    Xc = X.contiguous()
    Kt = torch.empty((N, N), dtype=torch.float64, device=X.device)   # column-major K = Kt^T
    _check(load().lbfgsb_op_gaussian_kernel(_ptr(Xc), N, d, float(gamma), _ptr(Kt), N,
                                            _stream_ptr(stream)))
    return Kt.T


def solve_batched_lsq(M, b, x, lower=None, upper=None, m_hist=5, opts: Options | None = None, tol=0.0):
    """N4 replicas (lbfgsb_solve_batched_lsq): M (batch, n, m) CUDA fp64 whose
    [k] is A_k stored column-major (i.e. A_k^T contiguous, see ``colmajor_batch``),
    b (batch, m), x (batch, n) in/out, lower/upper (batch, n) or None.  One CTA
    per problem.  Returns a list of Result."""
    import torch
    L = load()
    B, n, m = M.shape
    o = (opts or Options())._c()
    res = (_Res * max(B, 1))()
    for t in (M, b, x):
        if not t.is_contiguous():
            raise LbfgsbError("M, b, x must be contiguous")
    lo = None if lower is None else lower.contiguous()
    up = None if upper is None else upper.contiguous()
    stream = torch.cuda.current_stream().cuda_stream
    _check(L.lbfgsb_solve_batched_lsq(B, m, n, _ptr(M), _ptr(b), _ptr(lo), _ptr(up), _ptr(x), m_hist,
                                      C.byref(o), float(tol), C.c_void_p(stream), res))
    return [Result.from_c(res[i]) for i in range(B)]


def colmajor_batch(A):
    """(batch, m, n) host/CUDA array -> CUDA fp64 (batch, n, m) contiguous (each A_k column-major)."""
    import torch
    t = torch.as_tensor(A, dtype=torch.float64)
    return t.transpose(1, 2).contiguous().cuda()


def op_gemv(obj: LSQObjective, p, q, stream=None):
    """q = M~ p (the a1 forward GEMV kernel over all columns)."""
    _check(load().lbfgsb_op_gemv(obj._h, _ptr(p), _ptr(q), _stream_ptr(stream)))
    return q


def op_gemvt(obj: LSQObjective, r, g, stream=None):
    """g = M~^T r (the a3 backward GEMV kernel, no epilogue)."""
    _check(load().lbfgsb_op_gemvt(obj._h, _ptr(r), _ptr(g), _stream_ptr(stream)))
    return g
