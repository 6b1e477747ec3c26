// impl.cuh -- internal types shared by the kernels (kernels.cu) and the
// host control code (solver.cu) of liblbfgsb.  Not part of the ABI.
//
// Design: one Alg. 1 iteration of the LSQ objective is
// a fixed sequence of device kernels driven entirely by a device-resident
// control block (Ctrl), so that a chunk of iterations can be captured once
// into a CUDA graph and replayed without host round trips:
//
//   k_gram      working set Eq. (1) + masked Gram of {s_i, y_i, g} on S^k
//   k_recur     1 CTA: reduce Gram, convergence test, vector-free Alg. 3
//   k_dir       d = -sum_b c_b B_b on S^k, Alg. 2 candidates + reductions
//   k_branch    1 CTA: Alg. 2 line 3 decision, alpha_max
//   k_fwd       a1: q = M~ p (active columns only), split-K partials
//   k_ls        a2: reduce q partials, Armijo trial batch (16 trials)
//   k_ls_decide 1 CTA: first accepted trial, ring bookkeeping
//   k_rupd      r <- fma(alpha, q, r)
//   k_bwd       a3: g' = M~^T r' + fused epilogue (x', s, y ring write)
//
// Every kernel returns immediately when ctrl->done or ctrl->stall is set;
// the rare events (line-search continuation beyond 16 trials, the
// steepest-descent fallback of reading R14) "stall" the device loop and
// are handled by the host.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/lbfgsb.h"

namespace lb {

constexpr int MAXH = LBFGSB_MAX_HIST;
constexpr int MAXB = 2 * MAXH + 1;                 // Gram basis {s_i, y_i, g}
constexpr int MAXE = MAXB * (MAXB + 1) / 2;        // upper-triangle entries
constexpr int GRAM_STRIDE = MAXE + MAXH + 4;       // + full ||y||^2 + (gfree, nfree)
constexpr int MAXC = LBFGSB_MAX_CONS;
constexpr int KT = 16;                             // Armijo trials per batch
constexpr int NSEP = 2 + MAXC;                     // separable sums per trial
constexpr int NT = 256;                            // threads per CTA of the vector kernels
constexpr int TILE = 256;                          // coordinates per Gram tile
constexpr int FWD_ROWS = 2 * NT;                   // rows per k_fwd CTA (double2 per thread)
constexpr int FWD_SUB = 1024;                      // columns per compaction sub-tile
constexpr int BWD_NB = 8;                          // columns per k_bwd CTA

enum Stall : int { ST_NONE = 0, ST_FALLBACK = 1, ST_LS_CONT = 2 };
enum Status : int { S_CONVERGED = 0, S_MAX_ITERS = 1, S_LS_FAIL = 2 };

// Device-resident control block.  Written only by single-thread "decide"
// kernels (k_recur, k_branch, k_ls_decide, setup/kkt decides) and by the host
// while the stream is idle.
struct Ctrl {
    long long k;            // completed iterations
    long long n_fg, n_bt, n_fallbacks, nfree;
    int done, status, stall, nh, head, branch, fallback, ls_batch;
    int slot;               // ring slot the current iteration writes
    int nonfinite;
    double f;               // f(x^k)
    double f_new;
    double f_base;          // setup/refresh: f without the AL terms
    double gp, amax, alpha0, alpha, gfree, pg;
    double tol;
    double coef[MAXB];      // d = sum_b coef[b] B_b on S (basis order s_0..s_{nh-1}, y_0.., g)
    double ccoef[MAXC];     // AL gradient coefficients at the point whose gradient k_bwd forms
    double hval[MAXC];      // constraint values h_k / g_k at that point
    // AL parameters (set by the host between inner solves)
    double rho;
    double lam[MAXC];       // lambda (eq) then mu (ineq), by constraint index
    double rhs[MAXC];       // e (eq) then hv (ineq)
};

// Kernel arguments: constant for a given (handle, objective, x buffer); the
// per-iteration state lives in Ctrl.
struct Prob {
    // problem
    int64_t n;              // variables on this rank
    int64_t m, ncols, ld;
    const double* M;
    const double* colscale;
    int split;
    const double* b;
    const double* c;
    double delta;
    const double* l;
    const double* u;
    int n_eq, n_in;
    const double* Ecol[MAXC];  // constraint columns (n each): E_1..E_neq then G_1..G_nin
    // options
    double eps, c1, shrink;
    int max_bt, screen_full, mh;
    long long max_iters;
    // workspace
    double* x; double* g; double* d; double* pp; double* pt;
    double* S; double* Y;   // mh x n each
    double* r; double* q; double* qpart;
    uint8_t* mask;
    double* gram_part; double* dir_part; double* ls_part; double* sep_part; double* kkt_part;
    Ctrl* ctrl;
    // launch geometry
    int G1;                 // CTAs of the n-vector kernels (k_gram, k_dir, kkt)
    int fwd_rb, fwd_cc;     // k_fwd: row blocks x column chunks
    int64_t fwd_chunk;      // columns per chunk
    int GL, GS;             // k_ls: row CTAs, separable CTAs
    int bwd_blocks;
};

// ---- launchers (kernels.cu) ----
enum FwdMode : int { FWD_ITER = 0, FWD_X = 1, FWD_P = 2 };
enum BwdMode : int { BWD_ITER = 0, BWD_SETUP = 1, BWD_PLAIN = 2 };
enum LsMode : int { LS_ITER0 = 0, LS_ITER_NEXT = 1, LS_SETUP = 2, LS_OP = 3 };

void launch_clip(const Prob& P, cudaStream_t st);
void launch_gram(const Prob& P, cudaStream_t st, int op_mode);
void launch_recur(const Prob& P, cudaStream_t st, int op_mode);
void launch_dir(const Prob& P, cudaStream_t st, int op_mode);
void launch_branch(const Prob& P, cudaStream_t st, int op_mode);
void launch_fwd(const Prob& P, cudaStream_t st, int mode, const double* pvec);
void launch_resid(const Prob& P, cudaStream_t st, int subtract_b, double* out);
void launch_ls(const Prob& P, cudaStream_t st, int mode, const double* pvec);
void launch_ls_decide(const Prob& P, cudaStream_t st, int mode, double* f_out_dev, int ntr);
void launch_rupd(const Prob& P, cudaStream_t st);
void launch_bwd(const Prob& P, cudaStream_t st, int mode, const double* rvec, double* gout);
void launch_kkt(const Prob& P, cudaStream_t st);
void launch_cons(const Prob& P, cudaStream_t st);
void launch_ring_load(const Prob& P, cudaStream_t st, int nh, const double* S, const double* Y);
void launch_cb_trial(const Prob& P, cudaStream_t st, double alpha, double* xt);
void launch_cb_commit(const Prob& P, cudaStream_t st, const double* xt, const double* gt, int slot);

int sm_count();
void init_kernels();

}  // namespace lb
