/*
 * lbfgsb.h -- C ABI of the B200-native (sm_100a, fp64) hot path of the
 * GPU-efficient, Cauchy-point-free L-BFGS-B method of arXiv 2203.16340 and
 * its augmented-Lagrangian wrapper.
 *
 * Citations are lines of the paper's LaTeX source (PAPER.md:N, section /
 * algorithm / equation); "R<k>" names a reading of the paper recorded in
 * DESIGN.md section 3.
 *
 *   problem (section 3):  min f(x)  s.t.  l <= x <= u,
 *                                      l, u in R^n u {-inf, +inf}
 *   Alg. 1   main loop      -> lbfgsb_solve
 *   Alg. 2  projectDirection
 *   Eq. (1) working set S^k
 *   Alg. 3 modified two-loop recursion (computed in its
 *                              vector-free, Gram-matrix form on the device)
 *   Alg. 4 augmented Lagrangian, Eq. (3)
 *                              -> al_solve
 *
 * Conventions (all entry points):
 *  - fp64 throughout.  Pointers are DEVICE pointers unless marked (host).
 *  - Matrices are column-major: element (i, j) at M[i + j*ld], ld >= m.
 *  - Ownership: the caller owns every buffer it passes (M, b, c, bounds,
 *    x, constraint data, lambda, mu); they must stay valid for the duration
 *    of the call that uses them (objectives BORROW M/b/c/colscale until
 *    lbfgsb_objective_free).  The library owns the workspace it allocates in
 *    lbfgsb_create and frees it in lbfgsb_destroy; bounds are copied at
 *    create time.
 *  - Streams: all device work of a handle runs on the cuda stream given to
 *    lbfgsb_create; NULL makes the handle create a private blocking stream
 *    (implicitly ordered with the legacy default stream), because CUDA
 *    graphs cannot be captured on the legacy stream.  Solve calls return
 *    host-synchronously.  A handle is not thread-safe (one solve at a time).
 *  - Errors are return codes (never exceptions across the ABI); details via
 *    lbfgsb_last_error().  The solve OUTCOME (converged, max iterations,
 *    line-search failure) is a status in the result struct, not an error.
 *  - The library never falls back to a CPU path: if no CUDA device is
 *    usable every entry point that touches the device returns
 *    LBFGSB_ERR_CUDA.
 */
#ifndef LBFGSB_H_
#define LBFGSB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LBFGSB_ABI_VERSION 1
#define LBFGSB_MAX_HIST 16      /* m_hist <= 16                                  */
#define LBFGSB_MAX_CONS 4       /* linear AL constraints fused on device (m_eq+p_in) */

typedef struct lbfgsb_t lbfgsb_t;                 /* opaque solver handle            */
typedef struct lbfgsb_objective lbfgsb_objective; /* opaque objective descriptor     */

typedef enum {
    LBFGSB_OK = 0,
    LBFGSB_ERR_ARG = 1,         /* NULL where required, bad option value          */
    LBFGSB_ERR_DIM = 2,         /* dimension mismatch / out of range               */
    LBFGSB_ERR_BOUNDS = 3,      /* l_i > u_i or NaN bound            */
    LBFGSB_ERR_NONFINITE = 4,   /* f or gradient not finite at the start point     */
    LBFGSB_ERR_CALLBACK = 5,    /* user callback returned nonzero                  */
    LBFGSB_ERR_CUDA = 6,        /* CUDA runtime error / no device                  */
    LBFGSB_ERR_NCCL = 7,        /* NCCL error in a sharded handle                  */
    LBFGSB_ERR_OOM = 8,         /* device allocation failed                        */
    LBFGSB_ERR_UNSUPPORTED = 9  /* feature not available in this build / handle    */
} lbfgsb_err;

typedef enum {
    LBFGSB_CONVERGED = 0,          /* ||grad f[S^k]||_inf <= tol or S^k empty (R15) */
    LBFGSB_MAX_ITERS = 1,
    LBFGSB_LINESEARCH_FAILURE = 2, /* Armijo failed after the steepest-descent fallback (R14) */
    AL_MAX_OUTER = 3,
    AL_INNER_FAILURE = 4
} lbfgsb_status;

/* Solver options (the paper fixes none of these values; R1, R3, R11, R15). */
typedef struct {
    double eps;                 /* epsilon of Eq. (1), Alg. 2 line 3, Alg. 3 line 4 (R1,R2); default 1e-9 */
    double c1;                  /* Armijo constant (R11); default 1e-4                  */
    double shrink;              /* backtracking factor beta (R11); default 0.5          */
    double tol;                 /* stop when ||g[S]||_inf <= tol (R15); default 1e-6     */
    int32_t max_backtracks;     /* trials t = 0..max_backtracks per search (R11); 50     */
    int32_t screen_full_norm;   /* 0: screen with ||y[S]||^2 (R3), 1: ||y||^2; default 0 */
    int32_t check_every;        /* iterations launched between host checks; default 8   */
    int32_t use_graph;          /* 1: replay a CUDA graph of check_every iterations; 1  */
    int32_t profile;            /* 1: CUDA events around the two GEMV launches (ops.h)  */
    int32_t no_projection;      /* 1: skip Alg. 2's projected branch, always truncate
                                   (the proof-only variant of PAPER.md:201); default 0 */
    int32_t armijo_diff;        /* 1: Armijo test on the exact expansion of f(x+a p) - f(x)
                                   (LSQ / QP objectives; reading R29, avoids the
                                   cancellation floor of f_t <= f + c1 a g^T p); default 0 */
    int32_t refresh_every;      /* R > 0: the carried residual is replaced by r = M~x - b (and f, g
                                   recomputed exactly) at the top of every iteration k with
                                   k % R == 0, k > 0 (R13's optional refresh, for long runs);
                                   0: only the final refresh.  LSQ / QP objectives; default 0 */
    int32_t trials_per_pass;    /* Armijo trials alpha_0 beta^t decided per fused pass (1..16;
                                   0 = 16): beyond them the host continues with the next batch.
                                   The accepted trial does not depend on it (the trials are
                                   sequential); it only moves the batch boundaries. default 0 */
    int64_t max_iters;          /* default 10000                                        */
} lbfgsb_opts;

/* Outcome of one box-constrained solve (host struct). */
typedef struct {
    double f;                   /* objective at x* after the final residual refresh     */
    double pg_inf;              /* ||clip(x - g) - x||_inf  (KKT measure, R15)           */
    double gfree_inf;           /* ||g[S]||_inf at x*                                    */
    double seconds;             /* wall time of the solve (host clock, sync to sync)     */
    int64_t iters;              /* Alg. 1 iterations                                     */
    int64_t n_fg;               /* objective evaluations (setup + line-search trials)    */
    int64_t n_backtracks;       /* rejected Armijo trials                                */
    int64_t n_free;             /* |S| at x*                                             */
    int64_t n_fallbacks;        /* steepest-descent fallbacks taken (R14)                */
    int32_t status;             /* lbfgsb_status                                         */
    int32_t last_branch;        /* 1 = projected, 0 = truncated (Alg. 2) in the last iteration */
} lbfgsb_result;

void lbfgsb_opts_default(lbfgsb_opts* o);                            /* (host) */

/* Thread-local text describing the last non-OK return (never NULL). */
const char* lbfgsb_last_error(void);

/* Create a solver for n variables with box l <= x <= u and m_hist curvature
 * pairs (1 <= m_hist <= LBFGSB_MAX_HIST; the L-BFGS memory of Alg. 3).
 * lower/upper: DEVICE vectors of length n, or NULL for -inf / +inf
 * everywhere; copied into the handle.  Errors: ARG, DIM, BOUNDS, CUDA, OOM. */
lbfgsb_err lbfgsb_create(int64_t n, int32_t m_hist, const double* lower, const double* upper,
                         const lbfgsb_opts* opts /* NULL = defaults */, void* cuda_stream,
                         lbfgsb_t** out);

/* Column-sharded handle: this rank
 * owns n_local of the n_global variables (a contiguous block of columns of
 * M~; for split objectives the u and v halves of those columns).  M, c,
 * bounds, x and the constraint columns passed later are this rank's block;
 * b is the full (replicated) m-vector.  Each iteration all-gathers, over
 * NCCL (this entry point; lbfgsb_create_sharded_p2p below exchanges over
 * peer memory instead), the m-length partial of q = M~p and small packed reductions (Alg. 2
 * sums, separable trial sums, the Gram of Alg. 3), and every rank reduces
 * them in rank order, so all ranks take bit-identical decisions.  The library
 * creates its own NCCL communicator from the 128-byte ncclUniqueId (host)
 * obtained on rank 0 with lbfgsb_nccl_unique_id and broadcast by the caller
 * (e.g. with torch.distributed); the calling thread's current CUDA device is
 * used.  Returns LBFGSB_ERR_UNSUPPORTED when built without NCCL, NCCL on
 * communicator errors. */
lbfgsb_err lbfgsb_create_sharded(int64_t n_local, int64_t n_global, int32_t m_hist,
                                 const double* lower_local, const double* upper_local,
                                 const lbfgsb_opts* opts, void* cuda_stream,
                                 const void* nccl_unique_id /* (host) 128 bytes */,
                                 int32_t rank, int32_t nranks, lbfgsb_t** out);

/* Fill out (host, 128 bytes) with a fresh ncclUniqueId (call on rank 0). */
lbfgsb_err lbfgsb_nccl_unique_id(void* out);

/* Column-sharded handle whose per-iteration exchange (SURVEY.md 8(a) a9,
 * 8(e)) runs over PEER MEMORY instead of NCCL: every rank owns a mailbox
 * (device, cudaMalloc, owned by the handle) holding the four gathered pack
 * sections for residual length m <= m_max; the kernels that produce a pack
 * (k_dir, k_fwd row blocks -- the m-length q partial -- k_bwd's Gram tail,
 * k_kkt) store it straight into slot [rank] of every rank's mailbox and bump
 * a counter there, and a one-thread wait kernel gates the rank-order
 * reduction, so the exchanged bytes and their order equal the all-gather's
 * (bit-identical solves).  Same arguments as lbfgsb_create_sharded, no
 * NCCL id; nranks <= 8 (one NVSwitch box).  Connect with
 * lbfgsb_p2p_ipc_handle on every rank, an all-gather of the 64-byte handles
 * by the caller (e.g. torch.distributed), then lbfgsb_p2p_open; all ranks
 * must be connected before any rank solves.  Errors: ARG (rank / nranks),
 * DIM (m_max < 1, n_global < n_local), OOM, CUDA.  A peer that stops
 * signalling makes lbfgsb_solve return LBFGSB_ERR_NCCL after 60 s. */
lbfgsb_err lbfgsb_create_sharded_p2p(int64_t n_local, int64_t n_global, int32_t m_hist,
                                     const double* lower_local, const double* upper_local,
                                     const lbfgsb_opts* opts, void* cuda_stream, int32_t rank,
                                     int32_t nranks, int64_t m_max, lbfgsb_t** out);

/* out (host, 64 bytes): the cudaIpcMemHandle_t of this rank's mailbox. */
lbfgsb_err lbfgsb_p2p_ipc_handle(lbfgsb_t* h, void* out);

/* handles (host, nranks x 64 bytes, rank order, as gathered from
 * lbfgsb_p2p_ipc_handle): map every peer's mailbox into this process
 * (cudaIpcOpenMemHandle, peer access over NVLink enabled lazily; closed by
 * lbfgsb_destroy).  The own slot is ignored.  Errors: ARG, CUDA. */
lbfgsb_err lbfgsb_p2p_open(lbfgsb_t* h, const void* handles);

/* Loopback form of the P2P exchange: nranks plain single-GPU handles of one
 * process get mailboxes (m <= m_max) wired to each other directly, so that
 * lbfgsb_solve_loopback (lbfgsb_ops.h) runs the P2P protocol -- pushes
 * from the producing kernels, counter waits -- among logical ranks on one
 * device.  Errors: ARG, DIM, OOM. */
lbfgsb_err lbfgsb_p2p_connect_local(lbfgsb_t* const* hs, int32_t nranks, int64_t m_max);

/* SURVEY 8(e) bitwise P-invariance ("fixed C chunks, independent of P"):
 * the n global variables are cut into C = nranks fixed column chunks, each a
 * LOGICAL rank (an lbfgsb_create_sharded_p2p handle with rank = chunk index,
 * nranks = C), and a process hosts any subset of them (C/P on each of P
 * GPUs).  lbfgsb_p2p_open_group wires the n_local handles a process hosts
 * to all C mailboxes: the local ones directly, the others through CUDA IPC
 * (handles: host, C x 64 bytes in logical-rank order, e.g. all-gathered
 * from lbfgsb_p2p_ipc_handle; each remote mailbox is mapped once per
 * process and the mapping is owned by hs[0] -- destroy the group's handles
 * together).  Errors: ARG (not P2P handles of one group, a logical rank
 * hosted twice), CUDA. */
lbfgsb_err lbfgsb_p2p_open_group(lbfgsb_t* const* hs, int32_t n_local, const void* handles);

/* Solve one P2P-sharded problem over the n_local logical ranks this process
 * hosts (Alg. 1; objs[p] = the LSQ objective of hs[p]'s
 * chunk with the replicated b, xs[p] its DEVICE variable block, in x0 /
 * out x*).  Each logical rank runs with the kernel geometry of its own
 * chunk, and every decision reduces the C packs in logical-rank order, so x,
 * f and the iteration count are BITWISE independent of how the C chunks are
 * spread over processes and GPUs (P = 1, 2, 4, 8 for C = 8).  All launches
 * go to hs[0]'s stream (one CUDA graph per check interval).  res (host)
 * receives the global result.  Errors: ARG (handles not of one connected P2P
 * group), DIM, CUDA, NCCL (a peer stopped signalling for 60 s). */
lbfgsb_err lbfgsb_solve_group(lbfgsb_t* const* hs, const lbfgsb_objective* const* objs,
                              double* const* xs, int32_t n_local, double tol, lbfgsb_result* res);

void lbfgsb_destroy(lbfgsb_t* h);

/* ---- objectives --------------------------------------------------------- */

/* Built-in least-squares family (the paper's NNLS workload PAPER.md:368-374,
 * the linear-kernel dual SVM of PAPER.md:349-352, split-variable lasso):
 *    f(x) = 1/2 ||M~ x - b||^2 + c^T x + delta/2 ||x||^2            (R16)
 * with M~ = M diag(colscale) (colscale NULL = identity), or, when split = 1,
 * M~ = [M, -M] over n = 2*ncols variables (x = (u, v), u - v the lasso
 * coefficients).  M: m x ncols column-major with leading dimension ld >= m
 * (DEVICE, borrowed); b: m (NULL = 0); c: n (NULL = 0).  The objective's
 * hot path is the fused GEMV / GEMV^T pair of DESIGN.md section 5.
 * For a sharded handle, M holds this rank's ncols_local columns and b is
 * the full (replicated) m-vector.  Errors: ARG, DIM. */
lbfgsb_err lbfgsb_objective_lsq(const double* M, int64_t m, int64_t ncols, int64_t ld,
                                const double* colscale, int32_t split, const double* b,
                                const double* c, double delta, lbfgsb_objective** out);

/* Built-in dense QP (the Gaussian-kernel dual SVM of
 * PAPER.md:349-355):  f(x) = 1/2 x^T D Q D x + c^T x + delta/2 ||x||^2, with Q
 * n x n symmetric column-major (ld >= n, DEVICE, borrowed) and D =
 * diag(colscale) (NULL = identity; the SVM labels y).  The gradient is
 * carried as w = D Q D x (w' = w + alpha D Q D p, reading R13 for QPs), so an
 * iteration needs ONE pass over the active columns of Q; trial values are
 * 1/2 x^T w + alpha p^T w + 1/2 alpha^2 p^T (DQDp) + c^T x_t + ....
 * Single-GPU handles only (sharded: UNSUPPORTED).  Errors: ARG, DIM. */
lbfgsb_err lbfgsb_objective_qp(const double* Q, int64_t n, int64_t ld, const double* colscale,
                               const double* c, double delta, lbfgsb_objective** out);

/* Joint probability / regularised optimal transport (SURVEY.md 8(f) N2,
 * PAPER.md:393-402): variables x = vec(P), P m x n column-major (n_vars = m n),
 *   f(P) = <M, P> + lam r(P),   r = sum_ij P_ij log P_ij   (reg = 0, entropy)
 *                               r = 1/2 ||P||_F^2          (reg = 1, Gaussian),
 * M: m x n column-major cost (ld = m, DEVICE, borrowed); lam > 0 (the paper
 * uses 1/2).  The marginal equalities P 1 = u, P^T 1 = v are
 * attached by al_solve_transport (lbfgsb_solve returns UNSUPPORTED).  The
 * entropy needs a positive lower bound on the handle (reading R30: 1e-300).
 * Single-GPU handles only.  Errors: ARG, DIM. */
lbfgsb_err lbfgsb_objective_transport(const double* M, int64_t m, int64_t n, int32_t reg, double lam,
                                      lbfgsb_objective** out);

/* User objective: fg(user, x, g, f_host, stream) must write grad f(x) into
 * the DEVICE vector g (length n), *f_host = f(x) (host), enqueue its device
 * work on `stream` (or synchronise it), and return 0 (nonzero -> the solve
 * returns LBFGSB_ERR_CALLBACK).  x and g are library-owned device buffers
 * valid only during the call. */
typedef int32_t (*lbfgsb_fg_cb)(void* user, const double* x, double* g, double* f_host,
                                void* cuda_stream);
lbfgsb_err lbfgsb_objective_callback(lbfgsb_fg_cb fg, void* user, lbfgsb_objective** out);

void lbfgsb_objective_free(lbfgsb_objective* obj);

/* ---- Alg. 1 -------------------------------------------------------------- */

/* Minimise obj over the handle's box with Alg. 1.  x (DEVICE, length n):
 * in = x^0 (clipped into the box first), out = x*.
 * tol overrides opts.tol when > 0.  res (host) receives the outcome.
 * Errors: ARG, DIM, NONFINITE (f or g(x^0) not finite), CALLBACK, CUDA. */
lbfgsb_err lbfgsb_solve(lbfgsb_t* h, const lbfgsb_objective* obj, double* x, double tol,
                        lbfgsb_result* res);

/* Same as lbfgsb_solve for the LSQ family, but every input and the output
 * are HOST buffers: M_host (m x ncols, column-major, ld = m), b_host (m),
 * x_host (in x^0 / out x*).  The handle keeps a device copy buffer between
 * calls of the same shape; the host->device copies of M and b and the
 * device->host copy of x are part of the call (the bench's e2e number). */
lbfgsb_err lbfgsb_solve_lsq_host(lbfgsb_t* h, const double* M_host, int64_t m, int64_t ncols,
                                 const double* b_host, double* x_host, double tol,
                                 lbfgsb_result* res);

/* `count` independent LSQ problems of one shape, all from HOST buffers
 * (M_hosts[k]: m x ncols column-major, ld = m; b_hosts NULL or b_hosts[k]
 * NULL = 0; x_hosts[k] in x^0 / out x*; res[k] (host) its outcome), solved
 * one after the other on this handle.  The handle double-buffers the device
 * copies: the host->device copy of problem k+1 runs on a copy stream while
 * problem k is solved, so PCIe overlaps the solves; every problem's
 * host->device and device->host copies happen inside the call (the bench's
 * e2e number, pinned host memory recommended).  The handle keeps two device
 * copies of the operator between calls and two captured graphs.  Errors:
 * ARG, DIM, UNSUPPORTED (sharded handle), NONFINITE, CUDA, OOM. */
lbfgsb_err lbfgsb_solve_lsq_host_batch(lbfgsb_t* h, int32_t count, const double* const* M_hosts, int64_t m,
                                       int64_t ncols, const double* const* b_hosts, double* const* x_hosts,
                                       double tol, lbfgsb_result* res);

/* SURVEY 8(f) N4 "replicas": `batch` independent LSQ problems of one shape,
 *   min 1/2 ||A_k x - b_k||^2  s.t.  l_k <= x <= u_k,   k = 0..batch-1,
 * each solved by Alg. 1 in ONE CTA (A_k resident in shared
 * memory when m*n*8 plus the vectors fit in 200 KB, e.g. the C1 size 200 x
 * 100; larger problems up to the shared-memory limit read A_k from global
 * memory).  All DEVICE pointers: M batch x (m x n column-major, problem k at
 * M + k*m*n); b batch x m; lower / upper batch x n each (NULL = -inf / +inf);
 * x batch x n, in x^0 (clipped) / out x*.  res (host) receives `batch`
 * results (seconds = the whole call).  opts as lbfgsb_create (NULL =
 * defaults; check_every / use_graph / profile / armijo_diff unused); tol
 * overrides opts.tol when > 0.  Synchronous on cuda_stream (NULL = legacy).
 * Errors: ARG (NULL pointer, option values outside the ranges lbfgsb_create
 * accepts, tol < 0 or NaN), DIM (batch < 0, shape too large for one CTA),
 * BOUNDS (some l_i > u_i or a NaN bound), CUDA. */
lbfgsb_err lbfgsb_solve_batched_lsq(int32_t batch, int64_t m, int64_t n, const double* M, const double* b,
                                    const double* lower, const double* upper, double* x, int32_t m_hist,
                                    const lbfgsb_opts* opts, double tol, void* cuda_stream,
                                    lbfgsb_result* res);

/* ---- Alg. 4 -------------------------------------------------------------- */

typedef struct {
    double feas_tol;            /* stop when violation <= feas_tol (R22); default 1e-6  */
    double rho0;                /* initial penalty; default 1            */
    double rho_factor;          /* rho *= rho_factor if violation not halved; 2 */
    double rho_cap;             /* default 1e12                                          */
    int32_t max_outer;          /* default 100                                           */
    int32_t warm_start;         /* 0: x^0 = clip(0), lambda = mu = 0 (Alg. 4 line 3, R19);
                                   1: re-enter from the given x, lambda, mu (x clipped)  */
} al_opts;

void al_opts_default(al_opts* o);                                    /* (host) */

/* Nonlinear constraint callbacks (h: R^n -> R^m, g: R^n -> R^p
 * differentiable).  All pointers DEVICE, work enqueued on `stream` (or
 * synchronous); return 0 on success, nonzero = failure (al_solve then returns
 * LBFGSB_ERR_CALLBACK).
 *   hg:  h_out (m_nl) = h_nl(x), g_out (p_nl) = g_nl(x);
 *   jtv: out (n) = J_h(x)^T v_eq + J_g(x)^T v_in  (v_eq: m_nl, v_in: p_nl). */
typedef int32_t (*al_hg_cb)(void* user, const double* x, double* h_out, double* g_out, void* stream);
typedef int32_t (*al_jtv_cb)(void* user, const double* x, const double* v_eq, const double* v_in,
                             double* out, void* stream);

/* Constraints of Alg. 4: h(x) = [E^T x - e; h_nl(x)] = 0 and
 * g(x) = [G^T x - hv; g_nl(x)] <= 0.
 * Linear blocks: E n x m_eq, G n x p_in column-major (DEVICE, column k = the
 * coefficients of constraint k, contiguous); e (m_eq), hv (p_in) HOST.
 * Nonlinear blocks: m_nl equalities and p_nl inequalities through hg / jtv
 * (NULL when m_nl = p_nl = 0).  Multipliers are stacked the same way:
 * lambda = [linear m_eq; nonlinear m_nl], mu = [linear p_in; nonlinear p_nl]. */
typedef struct {
    int64_t m_eq, p_in;
    const double* E;
    const double* e;
    const double* G;
    const double* hv;
    int64_t m_nl, p_nl;
    al_hg_cb hg;
    al_jtv_cb jtv;
    void* user;
} al_constraints;

typedef struct {
    double violation_inf;       /* max(||h||_inf, ||min(-g, mu/rho)||_inf) (R21)      */
    double f;                   /* original objective f(x*) (no AL terms)              */
    double rho;                 /* final penalty                                       */
    double pg_inf;              /* KKT measure of the last inner solve                  */
    int64_t outer_iters, inner_iters_total;
    int32_t status;             /* LBFGSB_CONVERGED, AL_MAX_OUTER, AL_INNER_FAILURE     */
    int32_t pad_;
} al_result;

/* Alg. 4: x^0 = clip(0) (R19), lambda^0 = 0, mu^0 = 0,
 * rho = rho0 (or the given x, lambda, mu when opts->warm_start); each outer
 * iteration minimises the augmented Lagrangian Eq. (3)
 * over the box with Alg. 1 (warm x, empty history, inner tol
 * max(tol, 0.1 v), R22), then lambda += rho h(x), mu = (mu + rho g(x))_+
 * and rho *= rho_factor if the violation was not halved
 * (R20).
 * Two paths, the same method:
 *  - fused: an LSQ objective with m_eq + p_in <= LBFGSB_MAX_CONS linear
 *    constraints and no nonlinear ones -- the AL terms ride inside the
 *    iteration kernels (carried constraint values, the trial sums of k_sep);
 *  - general: any other case -- an LSQ or callback objective, any number of
 *    linear constraints (E^T x and E w on the GEMV kernels, one pass over E
 *    each), nonlinear constraints through hg / jtv.  The inner solve is the
 *    callback-objective Alg. 1: every trial value is evaluated.
 * x (DEVICE, n) in (warm start) / out; lambda (host, m_eq + m_nl) and mu
 * (host, p_in + p_nl) in (warm start) / out.  Errors: ARG, DIM, UNSUPPORTED
 * (QP or transport objective with constraints other than the fused path's),
 * CALLBACK, NONFINITE, CUDA. */
lbfgsb_err al_solve(lbfgsb_t* h, const lbfgsb_objective* obj, const al_constraints* cons,
                    const al_opts* opts, double* x, double* lambda, double* mu,
                    al_result* res);

/* Alg. 4 for a transport objective with its m + n marginal equalities
 * h(P) = [P 1 - u; P^T 1 - v]: x^0 = clip(0) (R19), lambda^0 =
 * 0, rho = rho0; each outer iteration minimises Eq. (3) over the box with
 * Alg. 1 (inner tol max(tol, 0.1 v), R22), then lambda += rho h(x)
 * and rho *= rho_factor if v = ||h||_inf was not halved
 * (R20).  The Armijo test is always the difference form of
 * reading R29.  u (m), v (n): DEVICE; x (DEVICE, m n) out = vec(P*);
 * lambda (DEVICE, m + n, may be NULL) out; res (host).  res->f is <M, P> +
 * lam r(P) at P*.  Errors: ARG, DIM, UNSUPPORTED (sharded handle), CUDA. */
lbfgsb_err al_solve_transport(lbfgsb_t* h, const lbfgsb_objective* obj, const double* u,
                              const double* v, const al_opts* opts, double* x, double* lambda,
                              al_result* res);

#ifdef __cplusplus
}
#endif
#endif /* LBFGSB_H_ */
