/*
 * lbfgsb_ops.h -- op-level C ABI: the individual hot-path kernels of
 * lbfgsb_solve exposed one by one, so that each can be checked against the
 * CPU oracle on identical inputs (tests/test_gpu_parity.py) and timed alone
 * (bench.py roofline).  Same conventions as lbfgsb.h: fp64, DEVICE pointers
 * unless marked (host), column-major matrices, caller-owned buffers,
 * errors as return codes, all work on the given stream, host-synchronous
 * return.
 */
#ifndef LBFGSB_OPS_H_
#define LBFGSB_OPS_H_

#include <stdint.h>
#include "lbfgsb.h"

#ifdef __cplusplus
extern "C" {
#endif

/* a1 forward GEMV (PAPER.md:371 objective):
 * q = M~ p over ALL columns, M~ the LSQ objective's operator (colscale /
 * split applied).  p: n (= nvars) DEVICE, q: m DEVICE.  Errors: ARG, CUDA. */
lbfgsb_err lbfgsb_op_gemv(const lbfgsb_objective* obj, const double* p, double* q,
                          void* cuda_stream);

/* a3 backward GEMV (row a3, without the iteration epilogue):
 * g = M~^T r.  r: m DEVICE, g: n DEVICE.  Errors: ARG, CUDA. */
lbfgsb_err lbfgsb_op_gemvt(const lbfgsb_objective* obj, const double* r, double* g,
                           void* cuda_stream);

/* Gaussian kernel matrix of SURVEY.md 8(f) N1 ("standard
 * Gaussian kernel with bandwidth parameter gamma"): K(i, j) =
 * exp(-gamma ||x_i - x_j||^2) by direct differences.  X: N x d row-major
 * (sample i at X + i*d, DEVICE); K: N x N column-major, ld ldk >= N (DEVICE,
 * caller-allocated, N*ldk*8 bytes).  Errors: ARG, CUDA. */
lbfgsb_err lbfgsb_op_gaussian_kernel(const double* X, int64_t N, int64_t d, double gamma, double* K,
                                     int64_t ldk, void* cuda_stream);

/* Direction pipeline of one iteration (rows a4, a5, a6): working set Eq. (1)
 * (PAPER.md:104-110), masked Gram + vector-free Alg. 3,
 * d[S-bar] = 0, Alg. 2.
 * Inputs: x, g (n, DEVICE) and nh <= m_hist curvature pairs S, Y
 * (DEVICE, nh*n each, pair i at S + i*n, OLDEST first); bounds, eps and the
 * screen norm come from the handle.  Outputs: free_out (n bytes, 1 = in
 * S^k), d_out (n), p_out (n, the direction Alg. 2 returns), and (host)
 * *projected (1 projected branch / 0 truncated), *gp = <g, p>,
 * *amax (1 for projected, blocking ratio for truncated, +inf if none).
 * Any output pointer may be NULL.  Errors: ARG, DIM, CUDA. */
lbfgsb_err lbfgsb_op_direction(lbfgsb_t* h, const double* x, const double* g, int32_t nh,
                               const double* S, const double* Y, uint8_t* free_out,
                               double* d_out, double* p_out, int32_t* projected, double* gp,
                               double* amax);

/* One Armijo batch of the line search (row a2): for t = 0..ntrials-1,
 * alpha_t = alpha0 * shrink^t (repeated multiplication), and
 *   f_t = 1/2 || fma(alpha_t, q, r) ||^2 + phi(clip(fma(alpha_t, p, x)))
 * (phi = c^T x + delta/2 ||x||^2 of the LSQ objective; reading R13).
 * r, q: m DEVICE; x, p: n DEVICE; f_out (host) ntrials values.
 * ntrials <= 16.  Errors: ARG, CUDA. */
lbfgsb_err lbfgsb_op_trials(lbfgsb_t* h, const lbfgsb_objective* obj, const double* r,
                            const double* q, const double* x, const double* p, double alpha0,
                            int32_t ntrials, double* f_out);

/* the generalized Cauchy point of the ORIGINAL L-BFGS-B
 * (Byrd, Lu, Nocedal, Zhu 1995, Algorithm CP), the sequential step the paper
 * removes, on the GPU as the baseline: the
 * breakpoints, reductions and final update in parallel kernels, the
 * breakpoint loop (a (t_i, i)-keyed binary heap, O(h^2) per breakpoint) on
 * ONE thread.  x, g: n DEVICE (n = the handle's); the box is the handle's;
 * nh <= 8 pairs S, Y (DEVICE, nh*n each, pair i at S + i*n, OLDEST first;
 * the compact form B = theta I - W M W^T, W = [Y, theta S]).  Outputs:
 * xcp (n, DEVICE); (host, may be NULL) c (2*nh) = W^T (xcp - x), *passed =
 * breakpoints passed by the loop, *scan_ms = device time of the
 * single-thread loop (CUDA events).  Errors: ARG, UNSUPPORTED, CUDA. */
lbfgsb_err lbfgsb_op_cauchy_point(lbfgsb_t* h, const double* x, const double* g, int32_t nh,
                                  const double* S, const double* Y, double theta, double* xcp,
                                  double* c, int64_t* passed, double* scan_ms);

/* the ORIGINAL L-BFGS-B (Byrd, Lu, Nocedal, Zhu 1995) on the
 * GPU, the paper's "L-BFGS-B GPU" baseline: per iteration
 * the projected-gradient test, the generalized Cauchy point (breakpoint loop
 * on one thread, as lbfgsb_op_cauchy_point), the direct primal subspace
 * minimisation with backtracking, Armijo (c1, shrink of the options) along
 * xbar - x, the pair kept iff s^T y > eps y^T y.  Host-driven, one sync per
 * step.  obj: an LSQ objective without c / delta (plain least squares); the
 * handle's box; m_hist <= 8.  x (DEVICE) in x^0 / out x*.  res->f is
 * 1/2 ||M~x - b||^2 at x*; (host, may be NULL) *cp_ms = device time of the
 * single-thread Cauchy-point loops.  Errors: ARG, UNSUPPORTED, CUDA. */
lbfgsb_err lbfgsb_solve_original(lbfgsb_t* h, const lbfgsb_objective* obj, double* x, double tol,
                                 lbfgsb_result* res, double* cp_ms);

/* Loopback verification of the column-sharded path on ONE device: the nranks
 * handles hs[p] (created with lbfgsb_create, n = that shard's variables, all
 * on the same device) act as logical ranks p = 0..nranks-1 of a sharded
 * solve of the concatenated problem, objs[p] / xs[p] their column blocks.
 * The cross-rank exchange is the same rank-ordered all-gather of packs that
 * lbfgsb_create_sharded performs over NCCL, done with device copies, and all
 * work runs on hs[0]'s stream.  res (host) is rank 0's outcome (all ranks
 * decide identically).  Errors: ARG, DIM, CUDA. */
lbfgsb_err lbfgsb_solve_loopback(lbfgsb_t* const* hs, const lbfgsb_objective* const* objs,
                                 double* const* xs, int32_t nranks, double tol, lbfgsb_result* res);

/* Device time of the hot-path GEMV launches of the solves run on this
 * handle since the last reset (host): names[i] / ms[i] (summed event time)
 * / launches[i], i < *count (<= cap).  Recorded only when opts.profile = 1
 * (CUDA events on the handle's stream around each gemv / gemvT launch,
 * inside the replayed graph as well).  reset != 0 clears the counters after
 * reading.  Errors: ARG. */
lbfgsb_err lbfgsb_profile_get(lbfgsb_t* h, int32_t cap, const char** names, double* ms,
                              int64_t* launches, int32_t* count, int32_t reset);

#ifdef __cplusplus
}
#endif
#endif /* LBFGSB_OPS_H_ */
