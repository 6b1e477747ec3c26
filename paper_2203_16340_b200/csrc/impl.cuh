// impl.cuh -- internal types shared by the kernels (kernels.cu) and the
// host control code (solver.cu) of liblbfgsb.  Not part of the ABI.
//
// Design.  One Alg. 1 iteration of the LSQ objective
// is THREE kernels, each ending in a deterministic "last-CTA" tail that
// takes the iteration's scalar decision on the device, so that a chunk of
// iterations replays as one CUDA graph with no host round trip:
//
//   k_dir   a6: d = sum_b coef_b B_b on S^k, Alg. 2 candidates and sums;
//           tail: Alg. 2 line 3 decision, alpha_max
//  [k_sep]  a2 separable part of the Armijo trials (only if c, delta or AL terms)
//   k_fwd   a1: q = M~ p over the ACTIVE columns, split-K partials; per-row-
//           block tail: q, 16 Armijo trial sums; global tail: accept alpha,
//           store-pair bookkeeping
//   k_bwd   a3: g' = M~^T r', r' = fma(alpha, q, r) on the fly, persistent
//           balanced column ranges; fused epilogue x', s, y, g', Eq. (1) mask
//           and the masked Gram of the NEXT basis; 2-level tail: Gram
//           reduce, convergence test, vector-free Alg. 3 -> coef
//
// Every kernel returns at entry when ctrl->done or ctrl->stall is set; the
// rare events (line search beyond 16 trials, the steepest-descent fallback
// of reading R14) "stall" the device loop and the host finishes them.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "../../include/lbfgsb.h"

namespace lb {

constexpr int MAXH = LBFGSB_MAX_HIST;
constexpr int P2P_MAXR = 8;                        // ranks of a P2P-exchange group (one NVSwitch box)
constexpr int MAXB = 2 * MAXH + 1;                 // Gram basis {s_i, y_i, g}
constexpr int MAXE = MAXB * (MAXB + 1) / 2;        // upper-triangle entries
constexpr int GRAM_STRIDE = MAXE + MAXH + 4;       // + full ||y||^2 + (gfree, nfree)
constexpr int MAXC = LBFGSB_MAX_CONS;
constexpr int KT = 16;                             // Armijo trials per batch
constexpr int NSEP = 2 + MAXC;                     // separable sums per trial
constexpr int NT = 256;                            // threads per CTA
constexpr int TILE = 256;                          // coordinates per Gram tile (k_gram)
constexpr int FWD_ROWS = 2 * NT;                   // rows per k_fwd CTA (double2 per thread)
constexpr int FWD_GRPC = 16;                      // k_fwd split-K partials reduced per chunk group
constexpr int FWD_MAXCG = 64;                      // chunk groups per row block (CC <= 1024)
constexpr int FWD_SUB = 1024;                      // columns per compaction sub-tile
constexpr int BWD_NB = 8;                          // columns per register group in k_bwd
constexpr int GRP = 32;                            // k_bwd CTAs per level-1 Gram group
constexpr int NTICKETS = 8192;
constexpr int TICKETS_EXTRA = 8192 + 4096;          // tickets[] holds NTICKETS + TICKETS_EXTRA counters
constexpr int SEP_MAXG = 64;                       // max k_sep CTAs

enum Stall : int { ST_NONE = 0, ST_FALLBACK = 1, ST_LS_CONT = 2 };
enum Status : int { S_CONVERGED = 0, S_MAX_ITERS = 1, S_LS_FAIL = 2 };

// Device-resident control block.  Written only by single-thread decisions in
// kernel tails and by the host while the stream is idle.
struct Ctrl {
    long long k;            // completed iterations
    long long n_fg, n_bt, n_fallbacks, nfree;
    long long nact;         // sum over iterations of active columns read by k_fwd
    int done, status, stall, nh, head, branch, fallback, ls_batch;
    int ls_tried, cont;     // trials evaluated this search; 1: device-side continuation pending (N2)
    int slot;               // ring slot the current iteration writes
    int nonfinite;
    int rsel;               // which residual buffer holds r(x^k)
    int pad_;
    double f;               // f(x^k)
    double f_new;
    double f_base;          // setup/refresh: f without the AL terms
    double gp, amax, alpha0, alpha, gfree, pg;
    double qp_xw, qp_pw, qp_pq;   // QP objective: x^T w, p^T w, p^T q of the current step
    double tol;
    double coef[MAXB];      // d = sum_b coef[b] B_b on S (basis s_0..s_{nh-1}, y_0.., g)
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
    int tpp;                // Armijo trials decided per fused pass (opts.trials_per_pass, 1..KT)
    int no_projection;      // Alg. 2 without the projected branch
    int diff;               // Armijo on the expanded difference (R29): trial sums -> r^T q, q^T q, c^T p ...
    int qp;                 // 1: f = 1/2 x^T D M D x + ... (M n x n symmetric); rbuf holds w = Q~ x
    long long max_iters;
    // workspace
    double* x; double* g; double* d; double* pp; double* pt;
    double* S; double* Y;   // mh x n each
    double* rbuf[2];        // residual double buffer (ctrl->rsel selects r(x^k))
    double* q; double* qpart;
    uint8_t* mask;
    double* gram_part;      // [max(GB, G1)][GRAM_STRIDE]
    double* gram_grp;       // [ceil(GB/GRP)][GRAM_STRIDE]
    double* dir_part;       // [G1][4]
    double* lsp;            // [max(RB, GLS)][KT]
    double* sep_part;       // [GS][KT][NSEP]
    double* kkt_part;       // [G1][3]
    unsigned* tickets;      // NTICKETS zeroed counters (reset by the tails)
    Ctrl* ctrl;
    // launch geometry
    int G1;                 // CTAs of the n-vector kernels (k_dir, k_gram, k_kkt)
    int RB, CC;             // k_fwd: row blocks x column chunks
    int64_t chunk;          // columns per k_fwd chunk
    int GB;                 // k_bwd persistent CTAs
    int GS;                 // k_sep CTAs (0: no separable part)
    int GLS;                // k_ls CTAs (host-driven trial batches)
    // column sharding: nranks > 1 makes every tail write
    // a LOCAL pack; the host all-gathers the packs and a *_decide kernel
    // reduces them in rank order, so all ranks take identical decisions.
    int nranks;
    int sharded;            // 1: sharded protocol (nranks > 1, or a 1-rank NCCL handle)
    double* pk_loc;         // [QS: m + KT*NSEP][DIR: 4][GRAM: GRAM_STRIDE][KKT: 4]
    double* qs_all;         // [nranks][m + KT*NSEP]   (q partial | separable trial sums)
    double* dir_all;        // [nranks][4]
    double* gram_all;       // [nranks][GRAM_STRIDE]
    double* kkt_all;        // [nranks][4]
    // P2P exchange (p2p.cu): instead of an NCCL all-gather,
    // the producing kernel's tail stores this rank's pack straight into slot
    // [rank_id] of every peer's mailbox (NVLink / CUDA IPC mapped) and bumps
    // the peer's section counter; the consuming kernel spins on the local counter.
    int p2p;
    int rank_id;
    double* peer_mb[P2P_MAXR];          // mailbox base of every rank (own one included)
    unsigned long long* mb_hdr;         // own mailbox header: [4] section counters, [4] timeout flag
    unsigned long long* p2p_tgt;        // [8] counts consumed so far per header slot (own device memory)
    // joint-probability / regularised OT objective (transport.cu):
    // x = vec(P), P tm x tn column-major; c = cost; delta (Gaussian) or ent
    // (entropy) weight; rbuf[rsel] holds the carried marginal residual
    // h = [P1 - u; P^T 1 - v] (tm + tn), tap = [p 1; p^T 1] of the direction
    int tp;
    int64_t tm, tn;
    double ent;
    double* tlam;           // [tm + tn] AL multipliers (device)
    const double* te;       // [tm + tn] right-hand sides (u; v)
    double* tap;            // [tm + tn]
    double* trow;           // [TCB][tm] row partials
    double* tcol;           // [TRB][tn] column partials
    double* tsp;            // [TRB * TCB][TNS] per-CTA sums
    double* tspr;           // [TRB][2] row-block finisher sums
    double* tspc;           // [TCB][2] column-chunk finisher sums
    unsigned* tticket;      // [TRB + TCB + 1]
    int TRB, TCB;           // k_tsum grid: row blocks of NT rows x chunks of TCOLS columns
};

__host__ __device__ inline int64_t qs_len(const Prob& P) { return P.m + (int64_t)KT * NSEP; }
__host__ __device__ inline int64_t off_dir(const Prob& P) { return qs_len(P); }
__host__ __device__ inline int64_t off_gram(const Prob& P) { return qs_len(P) + 4; }
__host__ __device__ inline int64_t off_kkt(const Prob& P) { return qs_len(P) + 4 + GRAM_STRIDE; }
__host__ __device__ inline int64_t pk_len(const Prob& P) { return qs_len(P) + 4 + GRAM_STRIDE + 4; }
// mailbox layout (doubles): header (8 x u64), then [R][qs_len] | [R][4] | [R][GRAM_STRIDE] | [R][4],
// i.e. the four gathered sections in pack order; section sec starts at mb_off(P, sec)
enum XSec : int { XS_QS = 0, XS_DIR = 1, XS_GRAM = 2, XS_KKT = 3 };
constexpr int MB_HDR = 8;
constexpr int MB_BARRIER = 5;              // header slot of the stall-path barrier counter (k_p2p_ack)
__host__ __device__ inline int64_t mb_off(const Prob& P, int sec)
{
    const int64_t R = P.nranks;
    const int64_t o[4] = {0, qs_len(P), qs_len(P) + 4, qs_len(P) + 4 + GRAM_STRIDE};
    return MB_HDR + R * o[sec];
}
__host__ __device__ inline int64_t mb_len(const Prob& P) { return MB_HDR + (int64_t)P.nranks * pk_len(P); }

// ---- launch modes
enum FwdMode : int { FWD_ITER = 0, FWD_SETUP = 1, FWD_P = 2 };
enum BwdMode : int { BWD_ITER = 0, BWD_SETUP = 1, BWD_PLAIN = 2, BWD_REFRESH = 3 };
enum SepMode : int { SEP_ITER = 0, SEP_NEXT = 1, SEP_SETUP = 2, SEP_OP = 3 };
enum LsMode : int { LS_NEXT = 0, LS_OP = 1, LS_SH_ITER = 2, LS_SH_SETUP = 3 };
enum TsMode : int { TS_ITER = 0, TS_NEXT = 1, TS_SETUP = 2, TS_CONT = 3 };
constexpr int TCOLS = 16;                  // k_tsum columns per CTA
constexpr int TT = 4;                      // entropy Armijo trials per batch
constexpr int TNS = 3 + TT;                // k_tsum per-CTA sums

// ---- launchers (kernels.cu)
void init_kernels();
int sm_count();
int bwd_ctas_per_sm();
int fwd_ctas_per_sm(int64_t m);
void launch_clip(const Prob& P, cudaStream_t st);
void launch_dir(const Prob& P, cudaStream_t st, int op_mode);
void launch_sep(const Prob& P, cudaStream_t st, int mode, const double* pvec);
void launch_fwd(const Prob& P, cudaStream_t st, int mode, const double* pvec, double* qout);
void launch_ls(const Prob& P, cudaStream_t st, int mode, const double* r, const double* q,
               double* f_out_dev, int ntr);
void launch_bwd(const Prob& P, cudaStream_t st, int mode, const double* rvec, double* gout);
void launch_gram_recur(const Prob& P, cudaStream_t st, int op_mode);
void launch_kkt(const Prob& P, cudaStream_t st);
// sharded decisions (after the host's all-gather of the local packs)
void launch_dir_decide(const Prob& P, cudaStream_t st);
void launch_gram_decide(const Prob& P, cudaStream_t st, int bwd_mode);
void launch_kkt_decide(const Prob& P, cudaStream_t st);
// p2p.cu: exchange over peer memory (the producers push from their tails)
void launch_p2p_put(const Prob& P, cudaStream_t st, int sec, int64_t off, int64_t cnt);
void launch_p2p_barrier(const Prob* Ps, int n, cudaStream_t st);
// al.cu: the stacked-constraint pieces of the general Alg. 4
void launch_al_terms(int64_t neq, const double* h, const double* lam, int64_t nin, const double* g,
                     const double* mu, double rho, double* weq, double* win, double* out, cudaStream_t st);
void launch_al_update(int64_t neq, const double* h, double* lam, int64_t nin, const double* g, double* mu,
                      double rho, double* vout, cudaStream_t st);
void launch_al_violation(int64_t neq, const double* h, int64_t nin, const double* g, const double* mu, double rho,
                         double* vout, cudaStream_t st);
void launch_lsq_value(int64_t m, const double* r, int64_t n, const double* x, const double* c, double delta,
                      double* g, double* out, cudaStream_t st);
void launch_sub(int64_t n, double* r, const double* b, cudaStream_t st);
void launch_axpy(int64_t n, const double* x, double* y, cudaStream_t st);
void launch_gauss(const double* X, int64_t N, int64_t d, double gamma, double* K, int64_t ldk,
                  cudaStream_t st);
void launch_ring_load(const Prob& P, cudaStream_t st, int nh, const double* S, const double* Y);
void launch_cb_trial(const Prob& P, cudaStream_t st, double alpha, double* xt);
void launch_cb_commit(const Prob& P, cudaStream_t st, const double* xt, const double* gt, int slot);
// batch.cu: one CTA per small LSQ problem
int launch_batch(int32_t batch, int64_t m, int64_t n, const double* M, const double* b, const double* lo,
                 const double* up, double* x, int mh, const lbfgsb_opts& o, double tol, lbfgsb_result* res,
                 cudaStream_t st);
// cauchy.cu: generalized Cauchy point of the original L-BFGS-B
int launch_cauchy(int64_t n, const double* x, const double* g, const double* l, const double* u, int h,
                  const double* S, const double* Y, double theta, double* d, double* tk, double* xcp,
                  double* part, double* red, unsigned* ticket, double* heap_g, double* scal,
                  cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1, double* Mout = nullptr);
int cauchy_nr();
// original.cu: the rest of the original L-BFGS-B iteration
struct OrigArgs {
    int64_t n, m;
    const double* x; const double* g; const double* l; const double* u;
    const double* xc;                        // Cauchy point
    int h;                                   // pairs (compact, oldest first)
    const double* S; const double* Y;
    double theta;
    const double* Mm;                        // M (2h x 2h) then M c (2h) from the Cauchy scan
    double* rc;                              // n: reduced gradient on F (0 elsewhere)
    double* du;                              // n: subspace step on F
    double* d;                               // n: search direction xbar - x
    double* part; double* red; unsigned* ticket;
    double* z;                               // 2h: N^{-1} M W^T Z r^c
    double* out;                             // scalars: [0] alpha*, [1] g^T d, [2] pg, [3] s^T y, [4] y^T y, [5] sum r^2
};
void launch_orig_pg(const OrigArgs& A, cudaStream_t st);
void launch_orig_subspace(const OrigArgs& A, cudaStream_t st);
void launch_orig_step(const OrigArgs& A, double* x, const double* dvec, double* r, const double* q, double alpha,
                      double* s_out, cudaStream_t st);
void launch_orig_pair(const OrigArgs& A, const double* gnew, const double* gold, const double* s, double* y_out,
                      cudaStream_t st);
void launch_orig_residual(const OrigArgs& A, double* r, const double* b, cudaStream_t st);
int orig_nr();
// transport.cu
void launch_tsum(const Prob& P, cudaStream_t st, int mode);
void launch_tviol(const Prob& P, cudaStream_t st, double rho, int update, double* out_dev);

}  // namespace lb
