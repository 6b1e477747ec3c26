/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the modified
 * (Cauchy-point-free) L-BFGS-B method of arXiv 2203.16340 and its augmented
 * Lagrangian wrapper.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg may load this file's
 * shared library.  The product path (paper_2203_16340_b200/) never links,
 * imports or executes anything under oracle/; the two share no code,
 * headers, helpers or constants.
 *
 * Everything is fp64 with sequential loops, compiled with -O2
 * -ffp-contract=off so that every fused multiply-add below is an explicit
 * fma() call (reading R12) and nothing else is contracted.
 * Matrices are column-major (element (i,j) at A[i + j*lda]).
 *
 * Citations: PAPER.md:N is a line of the paper's LaTeX source;
 * "R<k>" is a reading of the paper recorded in DESIGN.md section 3.
 *
 * Parity pins: every function below is pinned by a -m "not gpu" test in
 * tests/test_oracle_*.py against something other than itself (worked
 * examples, closed forms, brute force, scipy).  No function is
 * "parity unpinned" except the iteration COUNT of orc_minimize (the paper
 * prints no trajectory; PAPER.md:438 gives only "30-40 iterations").
 */
#define _POSIX_C_SOURCE 199309L   /* clock_gettime for the N3 Cauchy-point timer */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ------------------------------------------------------------------ */
/* Elementwise pieces                                                  */
/* ------------------------------------------------------------------ */

/* clip(x) = min(max(x, l), u); Alg. 2 line 1 "project z^k onto feasible
 * region".  l/u may be NULL meaning -inf/+inf. */
static double clip1(double v, const double* l, const double* u, int64_t i)
{
    if (l && v < l[i]) v = l[i];
    if (u && v > u[i]) v = u[i];
    return v;
}

void orc_clip(int64_t n, const double* x, const double* l, const double* u, double* out)
{
    for (int64_t i = 0; i < n; ++i) out[i] = clip1(x[i], l, u, i);
}

static double lo_of(const double* l, int64_t i) { return l ? l[i] : -INFINITY; }
static double up_of(const double* u, int64_t i) { return u ? u[i] : INFINITY; }

/* Eq. (1): i is FIXED iff
 *   (x_i <= l_i + eps and g_i >= 0) or (x_i >= u_i - eps and g_i <= 0).
 * free[i] = 1 for i in S^k.  Ties (g_i == 0 at a bound) are fixed (R17). */
void orc_working_set(int64_t n, const double* x, const double* g, const double* l,
                     const double* u, double eps, uint8_t* free_)
{
    for (int64_t i = 0; i < n; ++i) {
        int fixed_lo = (x[i] <= lo_of(l, i) + eps) && (g[i] >= 0.0);
        int fixed_up = (x[i] >= up_of(u, i) - eps) && (g[i] <= 0.0);
        free_[i] = (uint8_t)!(fixed_lo || fixed_up);
    }
}

/* <u[S], v[S]> (Alg. 3 line 3), sequential order. */
double orc_masked_dot(int64_t n, const double* u, const double* v, const uint8_t* free_)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i)
        if (!free_ || free_[i]) s += u[i] * v[i];
    return s;
}

/* Thread count of the matvecs ("an OpenMP variant parallelizes
 * over output elements only, with the same per-output summation order, so it
 * is bit-identical to the 1-thread oracle").  Default 1: the oracle as it
 * stands; bench.py's cpu_baseline also reports the all-cores figure. */
static int g_threads = 1;
void orc_set_threads(int32_t t) { g_threads = t > 0 ? t : 1; }
int32_t orc_get_threads(void) { return g_threads; }

/* out = A x   (A m x n column-major): out_i = sum_j A_ij x_j in increasing j
 * (loop order: for j, for i).  With threads > 1 each thread owns a block of
 * rows and runs the same j-then-i loops on it: every out_i sees the same
 * additions in the same order. */
void orc_matvec(int64_t m, int64_t n, const double* A, int64_t lda, const double* x, double* out)
{
    const int64_t T = g_threads;
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
    for (int64_t t = 0; t < T; ++t) {
        const int64_t i0 = t * m / T, i1 = (t + 1) * m / T;
        for (int64_t i = i0; i < i1; ++i) out[i] = 0.0;
        for (int64_t j = 0; j < n; ++j) {
            const double xj = x[j];
            const double* a = A + j * lda;
            for (int64_t i = i0; i < i1; ++i) out[i] += a[i] * xj;
        }
    }
}

/* out = A^T r, out_j = sum_i A_ij r_i in increasing i (threads: over j). */
void orc_matvec_t(int64_t m, int64_t n, const double* A, int64_t lda, const double* r, double* out)
{
#pragma omp parallel for num_threads(g_threads) schedule(static) if (g_threads > 1)
    for (int64_t j = 0; j < n; ++j) {
        const double* a = A + j * lda;
        double s = 0.0;
        for (int64_t i = 0; i < m; ++i) s += a[i] * r[i];
        out[j] = s;
    }
}

/* ------------------------------------------------------------------ */
/* Alg. 3: modified two-loop recursion, literal.     */
/* S, Y: nh pairs, pair i at S + i*n, OLDEST first (i = 0), newest     */
/* last (i = nh-1) -- "i = k-1, ..., k-m" of PAPER.md:488 is newest     */
/* first.  Returns d = -q on S, 0 off S (R5; Alg. 1 line 5 PAPER.md:73) */
/* screen_full_norm = 0: ||y_i[S]||^2 (R3); 1: ||y_i||^2 literal.        */
/* ------------------------------------------------------------------ */
void orc_two_loop(int64_t n, const double* g, const uint8_t* free_, int32_t nh,
                  const double* S, const double* Y, double eps, int32_t screen_full_norm,
                  double* d_out)
{
    double* q = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    double* a = (double*)malloc(sizeof(double) * (size_t)(nh > 0 ? nh : 1));
    double* rho = (double*)malloc(sizeof(double) * (size_t)(nh > 0 ? nh : 1));
    double* nu = (double*)malloc(sizeof(double) * (size_t)(nh > 0 ? nh : 1));
    int* ok = (int*)malloc(sizeof(int) * (size_t)(nh > 0 ? nh : 1));

    /* line 1: q = grad f(x^k)[S^k] */
    for (int64_t j = 0; j < n; ++j) q[j] = free_[j] ? g[j] : 0.0;

    /* lines 2-8: for i = k-1 ... k-m (newest to oldest) */
    for (int32_t i = nh - 1; i >= 0; --i) {
        const double* si = S + (int64_t)i * n;
        const double* yi = Y + (int64_t)i * n;
        rho[i] = orc_masked_dot(n, si, yi, free_);                       /* line 3 */
        nu[i] = screen_full_norm ? orc_masked_dot(n, yi, yi, NULL)
                                 : orc_masked_dot(n, yi, yi, free_);
        ok[i] = rho[i] > eps * nu[i];                                    /* line 4 */
        a[i] = 0.0;
        if (ok[i]) {
            a[i] = orc_masked_dot(n, si, q, free_) / rho[i];             /* line 5 */
            for (int64_t j = 0; j < n; ++j)                              /* line 6 */
                if (free_[j]) q[j] = q[j] - a[i] * yi[j];
        }
    }
    /* lines 9-11: initial scaling from pair k-1 only (R4) */
    if (nh > 0 && ok[nh - 1]) {
        const double gam = rho[nh - 1] / nu[nh - 1];
        for (int64_t j = 0; j < n; ++j)
            if (free_[j]) q[j] = gam * q[j];
    }
    /* lines 12-17: for i = k-m ... k-1 (oldest to newest) */
    for (int32_t i = 0; i < nh; ++i) {
        if (!ok[i]) continue;
        const double* si = S + (int64_t)i * n;
        const double* yi = Y + (int64_t)i * n;
        const double beta = orc_masked_dot(n, yi, q, free_) / rho[i];    /* line 14 */
        const double coef = a[i] - beta;
        for (int64_t j = 0; j < n; ++j)                                  /* line 15 */
            if (free_[j]) q[j] = q[j] + coef * si[j];
    }
    for (int64_t j = 0; j < n; ++j) d_out[j] = free_[j] ? -q[j] : 0.0;
    free(q); free(a); free(rho); free(nu); free(ok);
}

/* Alg. 2, projectDirection.  Returns 1 for the
 * projected branch (line 3 test passed), 0 for the truncated branch.
 * p_out receives the chosen direction.  Inequalities as printed (R9). */
int32_t orc_project_direction(int64_t n, const double* x, const double* g, const double* d,
                              const double* l, const double* u, double eps, double* p_out)
{
    double pg = 0.0, pp = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        const double z = clip1(x[j] + d[j], l, u, j);   /* line 1 */
        p_out[j] = z - x[j];                           /* line 2 */
        pg += p_out[j] * g[j];
        pp += p_out[j] * p_out[j];
    }
    if (pg <= -eps * pp && pp >= eps) return 1;        /* line 3 */
    for (int64_t j = 0; j < n; ++j) {                  /* lines 6-8 */
        double pj = d[j];
        if (d[j] < 0.0 && x[j] <= lo_of(l, j) + eps) pj = 0.0;
        if (d[j] > 0.0 && x[j] >= up_of(u, j) - eps) pj = 0.0;
        p_out[j] = pj;
    }
    return 0;
}

/* Alg. 2 lines 6-8 alone: the variant of PAPER.md:201 ("one can skip the
 * projection branch ... and still obtain convergence guarantees").  Returns 0
 * (truncated). */
int32_t orc_truncate_direction(int64_t n, const double* x, const double* d, const double* l,
                               const double* u, double eps, double* p_out)
{
    for (int64_t j = 0; j < n; ++j) {
        double pj = d[j];
        if (d[j] < 0.0 && x[j] <= lo_of(l, j) + eps) pj = 0.0;
        if (d[j] > 0.0 && x[j] >= up_of(u, j) - eps) pj = 0.0;
        p_out[j] = pj;
    }
    return 0;
}

/* Largest alpha >= 0 with l <= x + alpha p <= u, as the minimum blocking
 * ratio; +inf if nothing blocks (Alg. 1 line 7 "appropriate upper bound on
 * alpha^k"; R10). */
double orc_max_step(int64_t n, const double* x, const double* p, const double* l, const double* u)
{
    double amax = INFINITY;
    for (int64_t j = 0; j < n; ++j) {
        double t = INFINITY;
        if (p[j] < 0.0) t = (lo_of(l, j) - x[j]) / p[j];
        else if (p[j] > 0.0) t = (up_of(u, j) - x[j]) / p[j];
        if (t < amax) amax = t;
    }
    if (amax < 0.0) amax = 0.0;
    return amax;
}

/* ------------------------------------------------------------------ */
/* The least-squares objective family (built-in objective) */
/*   f(x) = 1/2 ||M~ x - b||^2 + c^T x + delta/2 ||x||^2               */
/* plus the augmented-Lagrangian terms of Eq. (3)   */
/* for LINEAR constraints h(x) = E^T x - e = 0, g(x) = G^T x - hv <= 0: */
/*   + rho/2 ||h(x) + lam/rho||^2 + rho/2 ||(g(x) + mu/rho)_+||^2       */
/* M~ = M diag(colscale) (colscale may be NULL), or [M, -M] if split.  */
/* NNLS: M = A, b, l = 0, no c/delta/constraints; the    */
/* 1/2 scaling is reading R16.                                          */
/* ------------------------------------------------------------------ */
typedef struct {
    int64_t m, ncols, lda;       /* M is m x ncols column-major */
    const double* M;
    const double* colscale;      /* NULL or ncols */
    int32_t split;               /* 1: variables (u, v), M~ = [M, -M] */
    const double* b;             /* NULL or m */
    const double* c;             /* NULL or nvars */
    double delta;
    int32_t n_eq;                /* E nvars x n_eq column-major, e host n_eq */
    const double* E; const double* e; const double* lam;
    int32_t n_in;                /* G nvars x n_in column-major, hv n_in */
    const double* G; const double* hv; const double* mu;
    double rho;
    int32_t qp;                  /* 1: quadratic objective 1/2 x^T Q~ x, Q~ = D M D (M n x n
                                    symmetric, D = diag(colscale)); "r" holds w = Q~ x */
    double ent;                  /* entropy weight: + ent * sum_j x_j log x_j (0 log 0 = 0;
                                    the joint-probability regulariser) */
    int64_t tm;                  /* > 0: the n_eq equality constraints are the marginals of
                                    x = vec(P), P tm x (nvars/tm) column-major:
                                    h_i = sum_j P_ij - e_i (i < tm), h_{tm+j} = sum_i P_ij -
                                    e_{tm+j}; E unused */
} orc_lsq;

static int64_t lsq_nvars(const orc_lsq* P) { return P->split ? 2 * P->ncols : P->ncols; }

/* q = M~ p  (explicit loops, column order) */
static void lsq_apply(const orc_lsq* P, const double* p, double* q)
{
    const int64_t nc = P->ncols;
    double* pe = (double*)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
    for (int64_t j = 0; j < nc; ++j) {
        double v = P->split ? (p[j] - p[nc + j]) : p[j];
        if (P->colscale) v = P->colscale[j] * v;
        pe[j] = v;
    }
    orc_matvec(P->m, nc, P->M, P->lda, pe, q);
    if (P->qp && P->colscale)                       /* Q~ = D M D: scale the rows too */
        for (int64_t i = 0; i < P->m; ++i) q[i] = P->colscale[i] * q[i];
    free(pe);
}

/* r = M~ x - b   (QP: w = Q~ x) */
static void lsq_residual(const orc_lsq* P, const double* x, double* r)
{
    lsq_apply(P, x, r);
    if (P->b && !P->qp)
        for (int64_t i = 0; i < P->m; ++i) r[i] = r[i] - P->b[i];
}

/* scratch for per-constraint values (n_eq or n_in doubles, at least one) */
static double* cons_buf(int32_t k) { return (double*)calloc((size_t)(k > 0 ? k : 1), sizeof(double)); }

/* x log x with 0 log 0 = 0 */
static double xlogx(double x) { return x > 0.0 ? x * log(x) : 0.0; }

/* constraint values at x */
static void lsq_cons(const orc_lsq* P, const double* x, double* hval, double* gval)
{
    const int64_t nv = lsq_nvars(P);
    if (P->tm > 0 && P->n_eq > 0) {                    /* marginals P 1 = u, P^T 1 = v */
        const int64_t tm = P->tm, tn = nv / tm;
        for (int64_t i = 0; i < tm; ++i) {
            double s = 0.0;
            for (int64_t j = 0; j < tn; ++j) s += x[i + j * tm];
            hval[i] = s - P->e[i];
        }
        for (int64_t j = 0; j < tn; ++j) {
            double s = 0.0;
            for (int64_t i = 0; i < tm; ++i) s += x[i + j * tm];
            hval[tm + j] = s - P->e[tm + j];
        }
    }
    for (int32_t k = 0; k < (P->tm > 0 ? 0 : P->n_eq); ++k) {
        double s = 0.0;
        const double* Ek = P->E + (int64_t)k * nv;
        for (int64_t j = 0; j < nv; ++j) s += Ek[j] * x[j];
        hval[k] = s - P->e[k];
    }
    for (int32_t k = 0; k < P->n_in; ++k) {
        double s = 0.0;
        const double* Gk = P->G + (int64_t)k * nv;
        for (int64_t j = 0; j < nv; ++j) s += Gk[j] * x[j];
        gval[k] = s - P->hv[k];
    }
}

/* Value of the non-residual part phi(x) = c^T x + delta/2 ||x||^2 + AL terms.
 * Also returns the AL gradient coefficients (rho h + lam), (rho g + mu)_+. */
static double lsq_phi(const orc_lsq* P, const double* x, double* coef_eq, double* coef_in)
{
    const int64_t nv = lsq_nvars(P);
    double cx = 0.0, xx = 0.0, xl = 0.0;
    for (int64_t j = 0; j < nv; ++j) {
        if (P->c) cx += P->c[j] * x[j];
        xx += x[j] * x[j];
        if (P->ent != 0.0) xl += xlogx(x[j]);
    }
    double phi = cx + 0.5 * P->delta * xx + P->ent * xl;
    double* hval = cons_buf(P->n_eq);
    double* gval = cons_buf(P->n_in);
    lsq_cons(P, x, hval, gval);
    for (int32_t k = 0; k < P->n_eq; ++k) {
        const double t = hval[k] + P->lam[k] / P->rho;               /* Eq. (3) */
        phi += 0.5 * P->rho * t * t;
        if (coef_eq) coef_eq[k] = P->rho * hval[k] + P->lam[k];
    }
    for (int32_t k = 0; k < P->n_in; ++k) {
        double t = gval[k] + P->mu[k] / P->rho;
        if (t < 0.0) t = 0.0;                                          /* (v)_+ */
        phi += 0.5 * P->rho * t * t;
        if (coef_in) coef_in[k] = P->rho * t;                          /* (rho g + mu)_+ */
    }
    free(hval); free(gval);
    return phi;
}

/* g = M~^T r + c + delta x + E (rho h + lam) + G (rho g + mu)_+
 * (QP: g = w + c + delta x + ..., the gradient of 1/2 x^T Q~ x being w = Q~ x) */
static void lsq_grad(const orc_lsq* P, const double* x, const double* r, double* g)
{
    const int64_t nc = P->ncols, nv = lsq_nvars(P);
    if (P->qp) {
        for (int64_t j = 0; j < nv; ++j) g[j] = r[j];
    } else {
        double* t = (double*)malloc(sizeof(double) * (size_t)(nc > 0 ? nc : 1));
        orc_matvec_t(P->m, nc, P->M, P->lda, r, t);
        for (int64_t j = 0; j < nc; ++j) {
            const double v = P->colscale ? P->colscale[j] * t[j] : t[j];
            g[j] = v;
            if (P->split) g[nc + j] = -v;
        }
        free(t);
    }
    double* ce = cons_buf(P->n_eq);
    double* ci = cons_buf(P->n_in);
    lsq_phi(P, x, ce, ci);
    for (int64_t j = 0; j < nv; ++j) {
        double v = g[j];
        if (P->c) v = v + P->c[j];
        v = v + P->delta * x[j];
        if (P->ent != 0.0) v = v + P->ent * (log(x[j]) + 1.0);       /* d/dx x log x */
        if (P->tm > 0) {                                               /* row i, column jj */
            if (P->n_eq > 0) v = v + ce[j % P->tm] + ce[P->tm + j / P->tm];
        } else {
            for (int32_t k = 0; k < P->n_eq; ++k) v = v + ce[k] * P->E[(int64_t)k * nv + j];
        }
        for (int32_t k = 0; k < P->n_in; ++k) v = v + ci[k] * P->G[(int64_t)k * nv + j];
        g[j] = v;
    }
    free(ce); free(ci);
}

static double half_sq(int64_t m, const double* r)
{
    double s = 0.0;
    for (int64_t i = 0; i < m; ++i) s += r[i] * r[i];
    return 0.5 * s;
}

static double dotv(int64_t n, const double* a, const double* b)
{
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
}

/* quadratic part of f at x with carried r:  LSQ 1/2 ||r||^2,  QP 1/2 x^T w */
static double quad_value(const orc_lsq* P, const double* x, const double* r)
{
    return P->qp ? 0.5 * dotv(P->m, x, r) : half_sq(P->m, r);
}

/* ------------------------------------------------------------------ */
/* Alg. 1 on the LSQ objective.                        */
/* ------------------------------------------------------------------ */
typedef struct {
    double eps, c1, shrink, tol;
    int32_t max_backtracks, screen_full_norm;
    int32_t no_projection;       /* 1: Alg. 2 without the projected branch */
    int32_t armijo_diff;         /* 1: Armijo test on the expanded difference f_t - f (R29) */
    int32_t refresh_every;       /* R > 0: r = M~x - b, f and g recomputed exactly at the top of
                                    every iteration k with k % R == 0, k > 0 (R13's optional refresh) */
    int64_t max_iters;
} orc_opts;

typedef struct {
    double f, pg_inf, gfree_inf;
    int64_t iters, n_fg, n_backtracks, n_free;
    int32_t status, last_branch;
    int64_t n_fallbacks;
} orc_result;

enum { ORC_CONVERGED = 0, ORC_MAX_ITERS = 1, ORC_LINESEARCH_FAILURE = 2,
       ORC_AL_MAX_OUTER = 3, ORC_AL_INNER_FAILURE = 4 };

/* Difference form of the Armijo test (reading R29): for the
 * quadratic-plus-separable objective the change along the segment x + alpha p
 * is, exactly,
 *   f(x + alpha p) - f(x) = alpha (r^T q + c^T p + delta x^T p)
 *                         + alpha^2/2 (q^T q + delta p^T p) + sum_k dphi_k
 * (QP: r^T q -> p^T w, q^T q -> p^T q), with the AL term of constraint k,
 * t0 = h_k(x) + lam_k/rho, a = E_k^T p, t1 = t0 + alpha a,
 *   dphi_k = rho/2 (t1^2 - t0^2) = rho alpha a (t0 + alpha a / 2)
 * (inequalities: rho/2 ((t1)_+^2 - (t0)_+^2), the same product when both
 * are positive).  Evaluated directly, without forming f(x + alpha p). */
double orc_armijo_delta(const orc_lsq* P, int64_t nv, const double* x, const double* r,
                        const double* q, const double* p, const double* l, const double* u,
                        double alpha)
{
    const double rq = P->qp ? dotv(nv, p, r) : dotv(P->m, r, q);
    const double qq = P->qp ? dotv(nv, p, q) : dotv(P->m, q, q);
    const double cp = P->c ? dotv(nv, P->c, p) : 0.0;
    const double xp = dotv(nv, x, p), pp = dotv(nv, p, p);
    double dl = alpha * (rq + cp + P->delta * xp) + 0.5 * alpha * alpha * (qq + P->delta * pp);
    if (P->ent != 0.0) {
        /* entropy at the clipped trial point y = clip(x + alpha p), per element:
         * y log y - x log x = d log x + y log(y / x),  d = y - x, with
         * log(y / x) = log1p(d / x) when |d| < x / 2 (no rounding of y / x near 1) */
        double se = 0.0;
        for (int64_t j = 0; j < nv; ++j) {
            const double y = clip1(fma(alpha, p[j], x[j]), l, u, j), d = y - x[j];
            if (x[j] > 0.0 && y > 0.0) {
                const double lr = fabs(d) < 0.5 * x[j] ? log1p(d / x[j]) : log(y / x[j]);
                se += d * log(x[j]) + y * lr;
            } else {
                se += xlogx(y) - xlogx(x[j]);
            }
        }
        dl += P->ent * se;
    }
    double* hval = cons_buf(P->n_eq);
    double* gval = cons_buf(P->n_in);
    double* ap = cons_buf(P->n_eq + P->n_in);
    lsq_cons(P, x, hval, gval);
    if (P->tm > 0) {                                    /* a = marginals of p */
        double* z = cons_buf(P->n_eq);
        orc_lsq T = *P;
        double* e0 = cons_buf(P->n_eq);
        T.e = e0; T.n_in = 0;
        lsq_cons(&T, p, z, NULL);
        for (int32_t k = 0; k < P->n_eq; ++k) ap[k] = z[k];
        free(z); free(e0);
    }
    for (int32_t k = 0; k < P->n_eq + P->n_in; ++k) {
        const int eq = k < P->n_eq;
        const int32_t kk = eq ? k : k - P->n_eq;
        double a;
        if (eq && P->tm > 0) {
            a = ap[k];
        } else {
            const double* col = eq ? P->E + (int64_t)kk * nv : P->G + (int64_t)kk * nv;
            a = dotv(nv, col, p);
        }
        const double t0 = eq ? hval[kk] + P->lam[kk] / P->rho : gval[kk] + P->mu[kk] / P->rho;
        const double t1 = t0 + alpha * a;
        if (eq || (t0 > 0.0 && t1 > 0.0)) {
            dl += P->rho * alpha * a * (t0 + 0.5 * alpha * a);
        } else {
            const double p0 = t0 > 0.0 ? t0 : 0.0, p1 = t1 > 0.0 ? t1 : 0.0;
            dl += 0.5 * P->rho * (p1 * p1 - p0 * p0);
        }
    }
    free(hval); free(gval); free(ap);
    return dl;
}

/* Armijo backtracking on the incremental residual (R10, R11, R13):
 * alpha_0 = min(1, amax), alpha_t = shrink * alpha_{t-1};
 * trial t: x_t = clip(fma(alpha_t, p, x)),
 *          f_t = 1/2 ||fma(alpha_t, q, r)||^2 + phi(x_t);
 * accept the first t with f_t <= f + c1 alpha_t <g, p>, t <= max_backtracks.
 * Returns 1 on acceptance. */
static int armijo_lsq(const orc_lsq* P, const orc_opts* o, int64_t nv, const double* x,
                      const double* l, const double* u, const double* r, const double* q,
                      const double* p, double f, double gp, double amax,
                      double* x_t, double* r_t, double* f_out, double* alpha_out,
                      int64_t* n_fg, int64_t* n_bt)
{
    double alpha = amax < 1.0 ? amax : 1.0;
    double xw = 0.0, pw = 0.0, pq = 0.0;
    if (P->qp) { xw = dotv(nv, x, r); pw = dotv(nv, p, r); pq = dotv(nv, p, q); }
    for (int32_t t = 0; t <= o->max_backtracks; ++t) {
        if (t > 0) alpha = o->shrink * alpha;
        for (int64_t j = 0; j < nv; ++j) x_t[j] = clip1(fma(alpha, p[j], x[j]), l, u, j);
        for (int64_t i = 0; i < P->m; ++i) r_t[i] = fma(alpha, q[i], r[i]);
        *n_fg += 1;
        if (o->armijo_diff) {                                     /* R29 */
            const double dl = orc_armijo_delta(P, nv, x, r, q, p, l, u, alpha);
            if (dl <= o->c1 * alpha * gp) {
                *f_out = f + dl; *alpha_out = alpha;
                return 1;
            }
            *n_bt += 1;
            continue;
        }
        const double quad = P->qp ? 0.5 * xw + alpha * pw + 0.5 * alpha * alpha * pq
                                  : half_sq(P->m, r_t);
        const double ft = quad + lsq_phi(P, x_t, NULL, NULL);
        if (ft <= f + o->c1 * alpha * gp) {
            *f_out = ft; *alpha_out = alpha;
            return 1;
        }
        *n_bt += 1;
    }
    return 0;
}

/* armijo_lsq exposed for its pins (R10, R11): returns 1 on acceptance and
 * the accepted alpha, f_t, and the number of rejected trials. */
int32_t orc_armijo_lsq(const orc_lsq* P, const orc_opts* o, int64_t nv, const double* x,
                       const double* l, const double* u, const double* r, const double* q,
                       const double* p, double f, double gp, double amax,
                       double* x_t, double* r_t, double* f_out, double* alpha_out, int64_t* n_bt)
{
    int64_t n_fg = 0;
    *n_bt = 0;
    return armijo_lsq(P, o, nv, x, l, u, r, q, p, f, gp, amax, x_t, r_t, f_out, alpha_out,
                      &n_fg, n_bt);
}

/* Solve min f(x) s.t. l <= x <= u with Alg. 1.  x in: x0 (clipped),
 * out: x*.  m_hist pairs, newest last. */
void orc_minimize_lsq(const orc_lsq* P, const double* l, const double* u, int32_t m_hist,
                      const orc_opts* o, double* x, orc_result* res)
{
    const int64_t nv = lsq_nvars(P), m = P->m;
    const size_t nvb = sizeof(double) * (size_t)(nv > 0 ? nv : 1);
    const size_t mb = sizeof(double) * (size_t)(m > 0 ? m : 1);
    double *g = malloc(nvb), *gn = malloc(nvb), *d = malloc(nvb), *p = malloc(nvb);
    double *xt = malloc(nvb), *r = malloc(mb), *rt = malloc(mb), *q = malloc(mb);
    double *Sr = malloc(nvb * (size_t)(m_hist > 0 ? m_hist : 1));
    double *Yr = malloc(nvb * (size_t)(m_hist > 0 ? m_hist : 1));
    uint8_t* fr = malloc((size_t)(nv > 0 ? nv : 1));
    int32_t nh = 0;

    memset(res, 0, sizeof(*res));
    orc_clip(nv, x, l, u, x);                                   /* feasible x^0 */
    lsq_residual(P, x, r);
    double f = quad_value(P, x, r) + lsq_phi(P, x, NULL, NULL);
    lsq_grad(P, x, r, g);
    res->n_fg = 1;

    int64_t k = 0;
    int32_t status = ORC_MAX_ITERS;
    for (;;) {
        if (o->refresh_every > 0 && k > 0 && k % o->refresh_every == 0) {   /* R13 optional refresh */
            lsq_residual(P, x, r);
            f = quad_value(P, x, r) + lsq_phi(P, x, NULL, NULL);
            lsq_grad(P, x, r, g);
        }
        orc_working_set(nv, x, g, l, u, o->eps, fr);             /* Alg. 1 line 3 */
        double gfree = 0.0; int64_t nfree = 0;
        for (int64_t j = 0; j < nv; ++j)
            if (fr[j]) { ++nfree; if (fabs(g[j]) > gfree) gfree = fabs(g[j]); }
        if (nfree == 0 || gfree <= o->tol) { status = ORC_CONVERGED; break; }  /* R15 */
        if (k >= o->max_iters) { status = ORC_MAX_ITERS; break; }

        int accepted = 0;
        double alpha = 0.0, fnew = f;
        for (int attempt = 0; attempt < 2 && !accepted; ++attempt) {
            if (attempt == 1) { nh = 0; res->n_fallbacks += 1; }      /* R14 fallback */
            orc_two_loop(nv, g, fr, nh, Sr, Yr, o->eps, o->screen_full_norm, d);  /* line 4 */
            const int32_t br = o->no_projection ? orc_truncate_direction(nv, x, d, l, u, o->eps, p)
                                                : orc_project_direction(nv, x, g, d, l, u, o->eps, p); /* line 6 */
            res->last_branch = br;
            double gp = 0.0;
            for (int64_t j = 0; j < nv; ++j) gp += g[j] * p[j];
            if (!(gp < 0.0)) continue;                                /* guard, R14 */
            const double amax = br ? 1.0 : orc_max_step(nv, x, p, l, u);
            lsq_apply(P, p, q);
            accepted = armijo_lsq(P, o, nv, x, l, u, r, q, p, f, gp, amax, xt, rt, &fnew,
                                  &alpha, &res->n_fg, &res->n_backtracks);
        }
        if (!accepted) { status = ORC_LINESEARCH_FAILURE; break; }

        /* line 7: x^{k+1}; carried residual r^{k+1} = r + alpha q (R13) */
        lsq_grad(P, xt, rt, gn);
        /* lines 8-9: s = x^{k+1} - x^k, y = grad^{k+1} - grad^k, stored
         * unconditionally (R8), oldest dropped */
        if (m_hist > 0) {
            if (nh == m_hist) {
                memmove(Sr, Sr + nv, nvb * (size_t)(m_hist - 1));
                memmove(Yr, Yr + nv, nvb * (size_t)(m_hist - 1));
                nh = m_hist - 1;
            }
            for (int64_t j = 0; j < nv; ++j) {
                Sr[(int64_t)nh * nv + j] = xt[j] - x[j];
                Yr[(int64_t)nh * nv + j] = gn[j] - g[j];
            }
            nh += 1;
        }
        memcpy(x, xt, nvb); memcpy(g, gn, nvb); memcpy(r, rt, mb);
        f = fnew;
        ++k;
    }

    /* final refresh: r = M~x - b, g, f; pg = ||clip(x - g) - x||_inf */
    lsq_residual(P, x, r);
    f = quad_value(P, x, r) + lsq_phi(P, x, NULL, NULL);
    lsq_grad(P, x, r, g);
    orc_working_set(nv, x, g, l, u, o->eps, fr);
    double pg = 0.0, gfree = 0.0; int64_t nfree = 0;
    for (int64_t j = 0; j < nv; ++j) {
        const double v = fabs(clip1(x[j] - g[j], l, u, j) - x[j]);
        if (v > pg) pg = v;
        if (fr[j]) { ++nfree; if (fabs(g[j]) > gfree) gfree = fabs(g[j]); }
    }
    res->f = f; res->pg_inf = pg; res->gfree_inf = gfree; res->n_free = nfree;
    res->iters = k; res->status = status;
    free(g); free(gn); free(d); free(p); free(xt); free(r); free(rt); free(q);
    free(Sr); free(Yr); free(fr);
}

/* ------------------------------------------------------------------ */
/* Alg. 4, augmented Lagrangian for LINEAR          */
/* constraints E^T x = e, G^T x <= hv.  Readings R18-R22.               */
/* ------------------------------------------------------------------ */
typedef struct {
    double feas_tol, rho0, rho_factor, rho_cap;
    int32_t max_outer;
} orc_al_opts;

typedef struct {
    double violation_inf, rho, f;
    int64_t outer_iters, inner_iters_total;
    int32_t status;
} orc_al_result;

/* Constraint-violation measure of the rho rule and the stopping test
 * ("infinity norm of the constraint violation"; reading R21):
 *   v = max(||h||_inf, ||min(-g, mu/rho)||_inf)
 * -- the complementarity-aware measure of Birgin & Martinez (2014), the
 * reference PAPER.md:531 cites for the convergence of Alg. 4.  For equality
 * constraints it is ||h||_inf; for an inequality it is the violation g_+
 * when g > 0 and otherwise how far mu is from complementary slackness.
 * h: n_eq values, g: n_in values (either may be NULL when its count is 0). */
double orc_al_violation(int32_t n_eq, const double* h, int32_t n_in, const double* g,
                        const double* mu, double rho)
{
    double v = 0.0;
    for (int32_t k = 0; k < n_eq; ++k) if (fabs(h[k]) > v) v = fabs(h[k]);
    for (int32_t k = 0; k < n_in; ++k) {
        double t = -g[k];
        const double mr = mu[k] / rho;
        if (mr < t) t = mr;
        if (fabs(t) > v) v = fabs(t);
    }
    return v;
}

/* Alg. 4 lines 6-7: lam += rho h; mu = (mu + rho g)_+ */
void orc_al_update_multipliers(int32_t n_eq, double* lam, const double* h, int32_t n_in,
                               double* mu, const double* g, double rho)
{
    for (int32_t k = 0; k < n_eq; ++k) lam[k] = lam[k] + rho * h[k];
    for (int32_t k = 0; k < n_in; ++k) {
        const double t = mu[k] + rho * g[k];
        mu[k] = t > 0.0 ? t : 0.0;
    }
}

/* Penalty rule ("If the infinity norm of the constraint violation
 * is not halved in an iteration, then rho is multiplied by a factor of 2";
 * reading R20): rho * factor if v > v_prev / 2, else rho; capped at cap. */
double orc_al_update_rho(double rho, double vprev, double v, double factor, double cap)
{
    if (v > 0.5 * vprev) {
        rho = rho * factor;
        if (rho > cap) rho = cap;
    }
    return rho;
}

static double viol_inf(const orc_lsq* P, const double* x, const double* mu, double rho)
{
    double* hval = cons_buf(P->n_eq);
    double* gval = cons_buf(P->n_in);
    lsq_cons(P, x, hval, gval);
    const double v = orc_al_violation(P->n_eq, hval, P->n_in, gval, mu, rho);
    free(hval); free(gval);
    return v;
}

/* Alg. 4 with an optional warm start and an optional per-outer trace.
 * warm = 0: x^0 = clip(0), lam = 0, mu = 0 (Alg. 4 line 3, R19);
 * warm = 1: x, lam_io, mu_io are taken as given (x clipped) -- re-entering
 *           the method with the multipliers of an earlier run.
 * trace (NULL or max_outer records of 3 + n_eq + n_in + nvars doubles):
 *   [rho used by the inner solve, v after the update, rho after the rule,
 *    lam (n_eq), mu (n_in), x (nvars)].
 * P->lam, P->mu are read AND updated in place (they must point at writable
 * arrays, cast away const by the caller-owned buffers lam_io / mu_io). */
void orc_al_solve_ex(orc_lsq* P, double* lam_io, double* mu_io, const double* l, const double* u,
                     int32_t m_hist, const orc_opts* o, const orc_al_opts* ao, double* x,
                     int32_t warm, double* trace, orc_al_result* res)
{
    const int64_t nv = lsq_nvars(P);
    const int64_t rec = 3 + P->n_eq + P->n_in + nv;
    memset(res, 0, sizeof(*res));
    if (!warm) {
        for (int64_t j = 0; j < nv; ++j) x[j] = 0.0;               /* x^0 = 0 (R19) */
        for (int32_t k = 0; k < P->n_eq; ++k) lam_io[k] = 0.0;
        for (int32_t k = 0; k < P->n_in; ++k) mu_io[k] = 0.0;
    }
    orc_clip(nv, x, l, u, x);
    P->lam = lam_io; P->mu = mu_io;
    double rho = ao->rho0;
    double vprev = viol_inf(P, x, mu_io, rho);
    res->status = ORC_AL_MAX_OUTER;
    for (int32_t it = 0; it < ao->max_outer; ++it) {
        orc_opts oi = *o;
        const double tin = 0.1 * vprev;
        oi.tol = tin > o->tol ? tin : o->tol;                      /* R22 */
        P->rho = rho;
        orc_result ir;
        orc_minimize_lsq(P, l, u, m_hist, &oi, x, &ir);            /* Alg. 4 line 5 */
        res->inner_iters_total += ir.iters;
        res->outer_iters = it + 1;
        if (ir.status == ORC_LINESEARCH_FAILURE) { res->status = ORC_AL_INNER_FAILURE; break; }
        double* hval = cons_buf(P->n_eq);
        double* gval = cons_buf(P->n_in);
        lsq_cons(P, x, hval, gval);
        orc_al_update_multipliers(P->n_eq, lam_io, hval, P->n_in, mu_io, gval, rho);  /* lines 6-7 */
        free(hval); free(gval);
        const double v = viol_inf(P, x, mu_io, rho);
        const double rho_used = rho;
        rho = orc_al_update_rho(rho, vprev, v, ao->rho_factor, ao->rho_cap);          /* line 8, R20 */
        vprev = v;
        if (trace) {
            double* t = trace + (int64_t)it * rec;
            t[0] = rho_used; t[1] = v; t[2] = rho;
            for (int32_t k = 0; k < P->n_eq; ++k) t[3 + k] = lam_io[k];
            for (int32_t k = 0; k < P->n_in; ++k) t[3 + P->n_eq + k] = mu_io[k];
            for (int64_t j = 0; j < nv; ++j) t[3 + P->n_eq + P->n_in + j] = x[j];
        }
        if (ir.status == ORC_CONVERGED && v <= ao->feas_tol && oi.tol == o->tol) {
            res->status = ORC_CONVERGED;
            break;
        }
    }
    /* report the ORIGINAL objective f (no AL terms) at x */
    {
        orc_lsq Q = *P; Q.n_eq = 0; Q.n_in = 0;
        double* r = malloc(sizeof(double) * (size_t)(P->m > 0 ? P->m : 1));
        lsq_residual(&Q, x, r);
        res->f = quad_value(&Q, x, r) + lsq_phi(&Q, x, NULL, NULL);
        free(r);
    }
    res->violation_inf = viol_inf(P, x, mu_io, rho);
    res->rho = rho;
}

void orc_al_solve(orc_lsq* P, double* lam_io, double* mu_io, const double* l, const double* u,
                  int32_t m_hist, const orc_opts* o, const orc_al_opts* ao, double* x,
                  orc_al_result* res)
{
    orc_al_solve_ex(P, lam_io, mu_io, l, u, m_hist, o, ao, x, 0, NULL, res);
}

/* Elementary helpers exposed for the pins (SPEC-style worked examples). */
int32_t orc_check_convergence(int64_t n, const double* g, const uint8_t* free_, double tol)
{
    for (int64_t j = 0; j < n; ++j)
        if (free_[j] && fabs(g[j]) > tol) return 0;
    return 1;
}

double orc_lsq_value(const orc_lsq* P, const double* x)
{
    double* r = malloc(sizeof(double) * (size_t)(P->m > 0 ? P->m : 1));
    lsq_residual(P, x, r);
    const double f = quad_value(P, x, r) + lsq_phi(P, x, NULL, NULL);
    free(r);
    return f;
}

void orc_lsq_grad(const orc_lsq* P, const double* x, double* g)
{
    double* r = malloc(sizeof(double) * (size_t)(P->m > 0 ? P->m : 1));
    lsq_residual(P, x, r);
    lsq_grad(P, x, r, g);
    free(r);
}

/* Armijo on a generic 1-D helper for the SPEC worked example f(x) = x^2:
 * returns the accepted alpha or -1 (pins R11 independently of LSQ). */
double orc_armijo_scalar_quadratic(double x, double p, double amax, double c1, double shrink,
                                   int32_t max_bt)
{
    const double f = x * x, gp = 2.0 * x * p;
    double alpha = amax < 1.0 ? amax : 1.0;
    for (int32_t t = 0; t <= max_bt; ++t) {
        if (t > 0) alpha = shrink * alpha;
        const double xt = fma(alpha, p, x);
        if (xt * xt <= f + c1 * alpha * gp) return alpha;
    }
    return -1.0;
}

/* ------------------------------------------------------------------ */
/* the generalized Cauchy point of the ORIGINAL        */
/* L-BFGS-B (Byrd, Lu, Nocedal, Zhu 1995, Algorithm CP), the step the   */
/* paper removes ("The Cauchy point is         */
/* computed by minimizing a quadratic approximation over the gradient   */
/* projection path").  Compact form B = theta I - W M W^T, W = [Y, theta */
/* S] (n x 2h), M = [[-D, L^T], [L, theta S^T S]]^{-1}, D = diag(s_i^T   */
/* y_i), L_ij = s_i^T y_j (i > j).  Pairs oldest first, column i of S at */
/* S + i n.  Breakpoints are visited in increasing (t_i, i) order.       */
/* ------------------------------------------------------------------ */
static int invert_small(int k, double* A /* k x k row-major, in: A, out: A^{-1} */)
{
    double* T = (double*)calloc((size_t)(k * 2 * k > 0 ? k * 2 * k : 1), sizeof(double));
    for (int i = 0; i < k; ++i) {
        for (int j = 0; j < k; ++j) T[i * 2 * k + j] = A[i * k + j];
        T[i * 2 * k + k + i] = 1.0;
    }
    for (int c = 0; c < k; ++c) {                     /* Gauss-Jordan, partial pivoting */
        int piv = c;
        for (int r = c + 1; r < k; ++r)
            if (fabs(T[r * 2 * k + c]) > fabs(T[piv * 2 * k + c])) piv = r;
        if (T[piv * 2 * k + c] == 0.0) { free(T); return 1; }
        if (piv != c)
            for (int j = 0; j < 2 * k; ++j) {
                const double t = T[c * 2 * k + j]; T[c * 2 * k + j] = T[piv * 2 * k + j]; T[piv * 2 * k + j] = t;
            }
        const double dv = T[c * 2 * k + c];
        for (int j = 0; j < 2 * k; ++j) T[c * 2 * k + j] /= dv;
        for (int r = 0; r < k; ++r) {
            if (r == c) continue;
            const double f = T[r * 2 * k + c];
            if (f == 0.0) continue;
            for (int j = 0; j < 2 * k; ++j) T[r * 2 * k + j] -= f * T[c * 2 * k + j];
        }
    }
    for (int i = 0; i < k; ++i)
        for (int j = 0; j < k; ++j) A[i * k + j] = T[i * 2 * k + k + j];
    free(T);
    return 0;
}

/* M (2h x 2h, row-major) of the compact representation */
int32_t orc_compact_m(int64_t n, int32_t h, const double* S, const double* Y, double theta, double* M)
{
    const int k = 2 * h;
    for (int i = 0; i < h; ++i)
        for (int j = 0; j < h; ++j) {
            const double sy = dotv(n, S + (int64_t)i * n, Y + (int64_t)j * n);
            const double ss = dotv(n, S + (int64_t)i * n, S + (int64_t)j * n);
            M[i * k + j] = (i == j) ? -sy : 0.0;                       /* -D */
            M[(h + i) * k + j] = (i > j) ? sy : 0.0;                   /* L */
            M[j * k + h + i] = (i > j) ? sy : 0.0;                     /* L^T */
            M[(h + i) * k + h + j] = theta * ss;                       /* theta S^T S */
        }
    return invert_small(k, M);
}

/* out = M v (2h) */
static void mat_vec_small(int k, const double* M, const double* v, double* out)
{
    for (int i = 0; i < k; ++i) {
        double s = 0.0;
        for (int j = 0; j < k; ++j) s += M[i * k + j] * v[j];
        out[i] = s;
    }
}

typedef struct { double t; int64_t i; } orc_bp;
static int bp_cmp(const void* a, const void* b)
{
    const orc_bp* x = (const orc_bp*)a; const orc_bp* y = (const orc_bp*)b;
    if (x->t < y->t) return -1;
    if (x->t > y->t) return 1;
    return x->i < y->i ? -1 : (x->i > y->i ? 1 : 0);
}

/* Algorithm CP.  xcp (n) out; c (2h) out = W^T (xcp - x); returns the number
 * of breakpoints passed (the sequential loop's trip count), or -1 if M is
 * singular. */
int64_t orc_cauchy_point(int64_t n, const double* x, const double* g, const double* l, const double* u,
                         int32_t h, const double* S, const double* Y, double theta, double* xcp, double* c)
{
    const int k = 2 * h;
    double* M = (double*)calloc((size_t)(k * k > 0 ? k * k : 1), sizeof(double));
    if (h > 0 && orc_compact_m(n, h, S, Y, theta, M)) { free(M); return -1; }
    double* d = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    orc_bp* F = (orc_bp*)malloc(sizeof(orc_bp) * (size_t)(n > 0 ? n : 1));
    double p[2 * 64], cc[2 * 64], Mv[2 * 64], wb[2 * 64];
    int64_t nf = 0;
    for (int64_t i = 0; i < n; ++i) {                                   /* breakpoints */
        double ti = INFINITY;
        if (g[i] < 0.0 && u) ti = (x[i] - u[i]) / g[i];
        else if (g[i] > 0.0 && l) ti = (x[i] - l[i]) / g[i];
        d[i] = (ti == 0.0) ? 0.0 : -g[i];
        xcp[i] = x[i];
        if (ti > 0.0) { F[nf].t = ti; F[nf].i = i; ++nf; }
    }
    qsort(F, (size_t)nf, sizeof(orc_bp), bp_cmp);
    for (int j = 0; j < k; ++j) { p[j] = 0.0; cc[j] = 0.0; }
    for (int64_t i = 0; i < n; ++i) {                                   /* p = W^T d */
        if (d[i] == 0.0) continue;
        for (int a = 0; a < h; ++a) p[a] += Y[(int64_t)a * n + i] * d[i];
        for (int a = 0; a < h; ++a) p[h + a] += theta * S[(int64_t)a * n + i] * d[i];
    }
    double fp = 0.0;
    for (int64_t i = 0; i < n; ++i) fp -= d[i] * d[i];                 /* f' = -d^T d */
    if (fp == 0.0) {                                                    /* d = 0: x is the Cauchy point */
        for (int j = 0; j < k; ++j) c[j] = 0.0;
        free(M); free(d); free(F);
        return 0;
    }
    mat_vec_small(k, M, p, Mv);
    double pMp = 0.0;
    for (int j = 0; j < k; ++j) pMp += p[j] * Mv[j];
    double fpp = -theta * fp - pMp;
    double dtmin = -fp / fpp;
    double told = 0.0;
    int64_t it = 0, passed = 0;
    double t = nf > 0 ? F[0].t : INFINITY;
    double dt = t - told;
    while (it < nf && dtmin >= dt) {
        const int64_t b = F[it].i;
        ++it; ++passed;
        const double gb = g[b];
        xcp[b] = d[b] > 0.0 ? u[b] : l[b];
        const double zb = xcp[b] - x[b];
        for (int j = 0; j < k; ++j) cc[j] += dt * p[j];
        for (int a = 0; a < h; ++a) { wb[a] = Y[(int64_t)a * n + b]; wb[h + a] = theta * S[(int64_t)a * n + b]; }
        double wMc = 0.0, wMp = 0.0, wMw = 0.0;
        mat_vec_small(k, M, cc, Mv);
        for (int j = 0; j < k; ++j) wMc += wb[j] * Mv[j];
        mat_vec_small(k, M, p, Mv);
        for (int j = 0; j < k; ++j) wMp += wb[j] * Mv[j];
        mat_vec_small(k, M, wb, Mv);
        for (int j = 0; j < k; ++j) wMw += wb[j] * Mv[j];
        fp = fp + dt * fpp + gb * gb + theta * gb * zb - gb * wMc;
        fpp = fpp - theta * gb * gb - 2.0 * gb * wMp - gb * gb * wMw;
        for (int j = 0; j < k; ++j) p[j] += gb * wb[j];
        d[b] = 0.0;
        dtmin = -fp / fpp;
        told = t;
        t = it < nf ? F[it].t : INFINITY;
        dt = t - told;
    }
    if (dtmin < 0.0) dtmin = 0.0;
    told = told + dtmin;
    for (int64_t i = 0; i < n; ++i)
        if (d[i] != 0.0) xcp[i] = x[i] + told * d[i];
    for (int j = 0; j < k; ++j) cc[j] += dtmin * p[j];
    for (int j = 0; j < k; ++j) c[j] = cc[j];
    free(M); free(d); free(F);
    return passed;
}

/* ------------------------------------------------------------------ */
/* the ORIGINAL L-BFGS-B (Byrd, Lu, Nocedal, Zhu 1995) */
/* on the LSQ objective, the baseline of PAPER.md:441-457 ("L-BFGS-B   */
/* CPU"): per iteration                                                */
/*   1. stop when ||P(x - g) - x||_inf <= tol (the projected gradient);  */
/*   2. generalized Cauchy point x^c (Algorithm CP, orc_cauchy_point);   */
/*   3. direct primal subspace minimisation over the free set F of x^c   */
/*      (BLNZ section 5.1): r^c = Z^T (g + theta (x^c - x) - W M c),     */
/*      d^u = -(1/theta) r^c - (1/theta^2) Z^T W N^{-1} M W^T Z r^c,     */
/*      N = I - (1/theta) M W^T Z Z^T W, then the largest a* <= 1 keeping */
/*      x^c + a* d^u in the box (backtrack);                             */
/*   4. Armijo backtracking (same c1 / shrink as the modified method,    */
/*      reading R34) along d = xbar - x from alpha = 1;                   */
/*   5. the pair (s, y) is kept iff s^T y > eps y^T y (BLNZ: skip        */
/*      otherwise), theta = y^T y / s^T y of the newest kept pair, m_hist */
/*      pairs.                                                            */
/* *cp_seconds receives the total time spent in step 2.                 */
/* ------------------------------------------------------------------ */
static double now_s(void)
{
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

void orc_lbfgsb_original(const orc_lsq* P, const double* l, const double* u, int32_t m_hist,
                         const orc_opts* o, double* x, orc_result* res, double* cp_seconds)
{
    const int64_t nv = lsq_nvars(P), m = P->m;
    const size_t nvb = sizeof(double) * (size_t)(nv > 0 ? nv : 1);
    const size_t mb = sizeof(double) * (size_t)(m > 0 ? m : 1);
    double *g = malloc(nvb), *gn = malloc(nvb), *xc = malloc(nvb), *xb = malloc(nvb), *d = malloc(nvb);
    double *xt = malloc(nvb), *r = malloc(mb), *rt = malloc(mb), *q = malloc(mb), *rc = malloc(nvb);
    double *S = malloc(nvb * (size_t)(m_hist > 0 ? m_hist : 1)), *Y = malloc(nvb * (size_t)(m_hist > 0 ? m_hist : 1));
    int32_t h = 0;
    double theta = 1.0, tcp = 0.0;
    memset(res, 0, sizeof(*res));
    orc_clip(nv, x, l, u, x);
    lsq_residual(P, x, r);
    double f = quad_value(P, x, r) + lsq_phi(P, x, NULL, NULL);
    lsq_grad(P, x, r, g);
    res->n_fg = 1;
    int64_t k = 0;
    int32_t status = ORC_MAX_ITERS;
    for (;;) {
        double pg = 0.0;
        for (int64_t j = 0; j < nv; ++j) {
            const double v = fabs(clip1(x[j] - g[j], l, u, j) - x[j]);
            if (v > pg) pg = v;
        }
        if (pg <= o->tol) { status = ORC_CONVERGED; break; }
        if (k >= o->max_iters) { status = ORC_MAX_ITERS; break; }
        /* 2. generalized Cauchy point */
        double c[32];
        const double t0 = now_s();
        if (orc_cauchy_point(nv, x, g, l, u, h, S, Y, theta, xc, c) < 0) { status = ORC_LINESEARCH_FAILURE; break; }
        tcp += now_s() - t0;
        /* 3. subspace minimisation over F = {i : l_i < xc_i < u_i} */
        const int kk = 2 * h;
        double M[32 * 32], v[32], Kf[32 * 32], Nm[32 * 32], tmp[32];   /* 2 m_hist <= 32 */
        if (h > 0) orc_compact_m(nv, h, S, Y, theta, M);
        double Mc[32];
        mat_vec_small(kk, M, c, Mc);
        for (int a = 0; a < kk; ++a) v[a] = 0.0;
        for (int a = 0; a < kk * kk; ++a) Kf[a] = 0.0;
        for (int64_t i = 0; i < nv; ++i) {
            const int fr = (!l || xc[i] > l[i]) && (!u || xc[i] < u[i]);
            if (!fr) { rc[i] = 0.0; continue; }
            double wi[32];
            for (int a = 0; a < h; ++a) { wi[a] = Y[(int64_t)a * nv + i]; wi[h + a] = theta * S[(int64_t)a * nv + i]; }
            double wMc = 0.0;
            for (int a = 0; a < kk; ++a) wMc += wi[a] * Mc[a];
            rc[i] = g[i] + theta * (xc[i] - x[i]) - wMc;                /* reduced gradient */
            for (int a = 0; a < kk; ++a) {
                v[a] += wi[a] * rc[i];                                   /* W^T Z r^c */
                for (int b = 0; b < kk; ++b) Kf[a * kk + b] += wi[a] * wi[b];   /* W^T Z Z^T W */
            }
        }
        if (h > 0) {
            mat_vec_small(kk, M, v, tmp);                                /* M W^T Z r^c */
            for (int a = 0; a < kk; ++a)
                for (int b = 0; b < kk; ++b) {
                    double s = 0.0;
                    for (int e = 0; e < kk; ++e) s += M[a * kk + e] * Kf[e * kk + b];
                    Nm[a * kk + b] = (a == b ? 1.0 : 0.0) - s / theta;
                }
            invert_small(kk, Nm);
            mat_vec_small(kk, Nm, tmp, v);                               /* N^{-1} M W^T Z r^c */
        }
        double astar = 1.0;
        for (int64_t i = 0; i < nv; ++i) {
            const int fr = (!l || xc[i] > l[i]) && (!u || xc[i] < u[i]);
            if (!fr) { d[i] = 0.0; continue; }
            double wv = 0.0;
            for (int a = 0; a < h; ++a) wv += Y[(int64_t)a * nv + i] * v[a] + theta * S[(int64_t)a * nv + i] * v[h + a];
            const double du = -rc[i] / theta - wv / (theta * theta);
            d[i] = du;
            if (du > 0.0 && u) { const double t = (u[i] - xc[i]) / du; if (t < astar) astar = t; }
            if (du < 0.0 && l) { const double t = (l[i] - xc[i]) / du; if (t < astar) astar = t; }
        }
        if (astar < 0.0) astar = 0.0;
        for (int64_t i = 0; i < nv; ++i) xb[i] = xc[i] + astar * d[i];
        for (int64_t i = 0; i < nv; ++i) d[i] = xb[i] - x[i];            /* search direction */
        /* 4. Armijo along d from alpha = 1 */
        double gd = 0.0;
        for (int64_t i = 0; i < nv; ++i) gd += g[i] * d[i];
        if (!(gd < 0.0)) { if (h == 0) { status = ORC_LINESEARCH_FAILURE; break; } h = 0; theta = 1.0; continue; }
        lsq_apply(P, d, q);
        double alpha = 1.0, fnew = f;
        int acc = 0;
        for (int32_t t = 0; t <= o->max_backtracks; ++t) {
            if (t > 0) alpha = o->shrink * alpha;
            for (int64_t j = 0; j < nv; ++j) xt[j] = clip1(fma(alpha, d[j], x[j]), l, u, j);
            for (int64_t i = 0; i < m; ++i) rt[i] = fma(alpha, q[i], r[i]);
            res->n_fg += 1;
            if (o->armijo_diff) {                                       /* R29 */
                const double dl = orc_armijo_delta(P, nv, x, r, q, d, l, u, alpha);
                if (dl <= o->c1 * alpha * gd) { acc = 1; fnew = f + dl; break; }
                res->n_backtracks += 1;
                continue;
            }
            const double ft = quad_value(P, xt, rt) + lsq_phi(P, xt, NULL, NULL);
            if (ft <= f + o->c1 * alpha * gd) { acc = 1; fnew = ft; break; }
            res->n_backtracks += 1;
        }
        if (!acc) { if (h == 0) { status = ORC_LINESEARCH_FAILURE; break; } h = 0; theta = 1.0; continue; }
        lsq_grad(P, xt, rt, gn);
        /* 5. pair update */
        double sy = 0.0, yy = 0.0;
        for (int64_t j = 0; j < nv; ++j) {
            const double sj = xt[j] - x[j], yj = gn[j] - g[j];
            sy += sj * yj; yy += yj * yj;
        }
        if (sy > o->eps * yy && m_hist > 0) {
            if (h == m_hist) {
                memmove(S, S + nv, nvb * (size_t)(m_hist - 1));
                memmove(Y, Y + nv, nvb * (size_t)(m_hist - 1));
                h = m_hist - 1;
            }
            for (int64_t j = 0; j < nv; ++j) { S[(int64_t)h * nv + j] = xt[j] - x[j]; Y[(int64_t)h * nv + j] = gn[j] - g[j]; }
            h += 1;
            theta = yy / sy;
        }
        memcpy(x, xt, nvb); memcpy(g, gn, nvb); memcpy(r, rt, mb);
        f = fnew;
        ++k;
    }
    lsq_residual(P, x, r);
    f = quad_value(P, x, r) + lsq_phi(P, x, NULL, NULL);
    lsq_grad(P, x, r, g);
    double pg = 0.0;
    for (int64_t j = 0; j < nv; ++j) {
        const double v = fabs(clip1(x[j] - g[j], l, u, j) - x[j]);
        if (v > pg) pg = v;
    }
    res->f = f; res->pg_inf = pg; res->iters = k; res->status = status;
    if (cp_seconds) *cp_seconds = tcp;
    free(g); free(gn); free(xc); free(xb); free(d); free(xt); free(r); free(rt); free(q); free(rc);
    free(S); free(Y);
}

/* ------------------------------------------------------------------ */
/* Alg. 1 on a GENERIC objective (f, grad f from a callback) and       */
/* Alg. 4 with general constraints:*/
/* min f(x) s.t. h(x) = 0, g(x) <= 0, l <= x <= u, with h = [E^T x - e; */
/* h_nl(x)], g = [G^T x - hv; g_nl(x)]: linear blocks as E / G columns, */
/* nonlinear blocks through callbacks for the values and for J^T v.     */
/* Every objective value at a trial point is EVALUATED (no carried     */
/* residual): the reading of the callback path (R14's fallback, R10,   */
/* R11 as in orc_minimize_lsq).                                         */
/* ------------------------------------------------------------------ */
typedef int32_t (*orc_fg_fn)(void* ctx, const double* x, double* g, double* f);
typedef int32_t (*orc_hg_fn)(void* ctx, const double* x, double* h, double* gc);
typedef int32_t (*orc_jtv_fn)(void* ctx, const double* x, const double* veq, const double* vin,
                              double* out);

/* Alg. 1 with Alg. 2 / Alg. 3 and Armijo backtracking on
 * f(clip(fma(alpha, p, x))) evaluated by fg.  Returns 0, or the nonzero
 * callback code (res->status untouched then). */
int32_t orc_minimize_fg(int64_t nv, orc_fg_fn fg, void* ctx, const double* l, const double* u,
                        int32_t m_hist, const orc_opts* o, double* x, orc_result* res)
{
    const size_t nvb = sizeof(double) * (size_t)(nv > 0 ? nv : 1);
    double *g = malloc(nvb), *gn = malloc(nvb), *d = malloc(nvb), *p = malloc(nvb), *xt = malloc(nvb);
    double *Sr = malloc(nvb * (size_t)(m_hist > 0 ? m_hist : 1));
    double *Yr = malloc(nvb * (size_t)(m_hist > 0 ? m_hist : 1));
    uint8_t* fr = malloc((size_t)(nv > 0 ? nv : 1));
    int32_t nh = 0, rc = 0;
    memset(res, 0, sizeof(*res));
    orc_clip(nv, x, l, u, x);                                       /* feasible x^0 */
    double f = 0.0;
    rc = fg(ctx, x, g, &f);
    res->n_fg = 1;
    int64_t k = 0;
    int32_t status = ORC_MAX_ITERS;
    while (rc == 0) {
        orc_working_set(nv, x, g, l, u, o->eps, fr);                 /* Alg. 1 line 3 */
        double gfree = 0.0; int64_t nfree = 0;
        for (int64_t j = 0; j < nv; ++j)
            if (fr[j]) { ++nfree; if (fabs(g[j]) > gfree) gfree = fabs(g[j]); }
        if (nfree == 0 || gfree <= o->tol) { status = ORC_CONVERGED; break; }    /* R15 */
        if (k >= o->max_iters) { status = ORC_MAX_ITERS; break; }
        int accepted = 0;
        double alpha = 0.0, ft = f;
        for (int attempt = 0; attempt < 2 && !accepted && rc == 0; ++attempt) {
            if (attempt == 1) { nh = 0; res->n_fallbacks += 1; }      /* R14 fallback */
            orc_two_loop(nv, g, fr, nh, Sr, Yr, o->eps, o->screen_full_norm, d);
            const int32_t br = o->no_projection ? orc_truncate_direction(nv, x, d, l, u, o->eps, p)
                                                : orc_project_direction(nv, x, g, d, l, u, o->eps, p);
            res->last_branch = br;
            double gp = 0.0;
            for (int64_t j = 0; j < nv; ++j) gp += g[j] * p[j];
            if (!(gp < 0.0)) continue;                                 /* guard, R14 */
            const double amax = br ? 1.0 : orc_max_step(nv, x, p, l, u);
            alpha = amax < 1.0 ? amax : 1.0;                           /* R10 */
            for (int32_t t = 0; t <= o->max_backtracks; ++t) {
                if (t > 0) alpha = o->shrink * alpha;                  /* R11 */
                for (int64_t j = 0; j < nv; ++j) xt[j] = clip1(fma(alpha, p[j], x[j]), l, u, j);
                rc = fg(ctx, xt, gn, &ft);
                res->n_fg += 1;
                if (rc) break;
                if (ft <= f + o->c1 * alpha * gp) { accepted = 1; break; }
                res->n_backtracks += 1;
            }
        }
        if (rc) break;
        if (!accepted) { status = ORC_LINESEARCH_FAILURE; break; }
        if (m_hist > 0) {                                              /* PAPER.md:77-80, R8 */
            if (nh == m_hist) {
                memmove(Sr, Sr + nv, nvb * (size_t)(m_hist - 1));
                memmove(Yr, Yr + nv, nvb * (size_t)(m_hist - 1));
                nh = m_hist - 1;
            }
            for (int64_t j = 0; j < nv; ++j) {
                Sr[(int64_t)nh * nv + j] = xt[j] - x[j];
                Yr[(int64_t)nh * nv + j] = gn[j] - g[j];
            }
            nh += 1;
        }
        memcpy(x, xt, nvb); memcpy(g, gn, nvb);
        f = ft;
        ++k;
    }
    if (rc == 0) {
        orc_working_set(nv, x, g, l, u, o->eps, fr);
        double pg = 0.0, gfree = 0.0; int64_t nfree = 0;
        for (int64_t j = 0; j < nv; ++j) {
            const double v = fabs(clip1(x[j] - g[j], l, u, j) - x[j]);
            if (v > pg) pg = v;
            if (fr[j]) { ++nfree; if (fabs(g[j]) > gfree) gfree = fabs(g[j]); }
        }
        res->f = f; res->pg_inf = pg; res->gfree_inf = gfree; res->n_free = nfree;
        res->iters = k; res->status = status;
    }
    free(g); free(gn); free(d); free(p); free(xt); free(Sr); free(Yr); free(fr);
    return rc;
}

/* The constrained problem of the general Alg. 4.  Base objective: the LSQ
 * family P (its own constraint fields must be empty) or, when P is NULL, the
 * callback fg.  Constraint stacking: equalities [linear m_eq; nonlinear
 * m_nl], inequalities [linear p_in; nonlinear p_nl]; multipliers in the same
 * order. */
typedef struct {
    int64_t nv;
    const orc_lsq* P;
    orc_fg_fn fg; void* fg_ctx;
    int32_t m_eq, p_in;           /* linear: E (nv x m_eq col-major), e; G (nv x p_in), hv */
    const double *E, *e, *G, *hv;
    int32_t m_nl, p_nl;           /* nonlinear: values and J^T v through callbacks */
    orc_hg_fn hg; orc_jtv_fn jtv; void* nl_ctx;
} orc_gcons;

typedef struct {
    const orc_gcons* Q;
    const double* lam; const double* mu; double rho;
    double* hv; double* gv;       /* scratch: all equality / inequality values */
    double* weq; double* win;     /* scratch: multiplier-weighted coefficients */
    double* tmp;                  /* scratch nv */
} orc_al_ctx;

/* all constraint values at x: h (m_eq + m_nl), g (p_in + p_nl) */
static int32_t gcons_values(const orc_gcons* Q, const double* x, double* h, double* gc)
{
    for (int32_t k = 0; k < Q->m_eq; ++k) {
        double s = 0.0;
        const double* col = Q->E + (int64_t)k * Q->nv;
        for (int64_t j = 0; j < Q->nv; ++j) s += col[j] * x[j];
        h[k] = s - Q->e[k];
    }
    for (int32_t k = 0; k < Q->p_in; ++k) {
        double s = 0.0;
        const double* col = Q->G + (int64_t)k * Q->nv;
        for (int64_t j = 0; j < Q->nv; ++j) s += col[j] * x[j];
        gc[k] = s - Q->hv[k];
    }
    if (Q->m_nl + Q->p_nl > 0)
        return Q->hg(Q->nl_ctx, x, h + Q->m_eq, gc + Q->p_in);
    return 0;
}

/* Eq. (3): L = f + rho/2 ||h + lam/rho||^2 + rho/2 ||(g + mu/rho)_+||^2,
 * grad L = grad f + J_h^T (rho h + lam) + J_g^T (rho g + mu)_+ */
static int32_t al_fg(void* vctx, const double* x, double* g, double* f)
{
    orc_al_ctx* A = (orc_al_ctx*)vctx;
    const orc_gcons* Q = A->Q;
    const int64_t nv = Q->nv;
    int32_t rc = 0;
    if (Q->P) {
        *f = orc_lsq_value(Q->P, x);
        orc_lsq_grad(Q->P, x, g);
    } else {
        rc = Q->fg(Q->fg_ctx, x, g, f);
        if (rc) return rc;
    }
    rc = gcons_values(Q, x, A->hv, A->gv);
    if (rc) return rc;
    const int32_t neq = Q->m_eq + Q->m_nl, nin = Q->p_in + Q->p_nl;
    double pen = 0.0;
    for (int32_t k = 0; k < neq; ++k) {
        const double t = A->hv[k] + A->lam[k] / A->rho;
        pen += 0.5 * A->rho * t * t;
        A->weq[k] = A->rho * A->hv[k] + A->lam[k];
    }
    for (int32_t k = 0; k < nin; ++k) {
        double t = A->gv[k] + A->mu[k] / A->rho;
        if (t < 0.0) t = 0.0;
        pen += 0.5 * A->rho * t * t;
        A->win[k] = A->rho * t;
    }
    *f = *f + pen;
    for (int64_t j = 0; j < nv; ++j) {
        double v = g[j];
        for (int32_t k = 0; k < Q->m_eq; ++k) v = v + A->weq[k] * Q->E[(int64_t)k * nv + j];
        for (int32_t k = 0; k < Q->p_in; ++k) v = v + A->win[k] * Q->G[(int64_t)k * nv + j];
        g[j] = v;
    }
    if (Q->m_nl + Q->p_nl > 0) {
        rc = Q->jtv(Q->nl_ctx, x, A->weq + Q->m_eq, A->win + Q->p_in, A->tmp);
        if (rc) return rc;
        for (int64_t j = 0; j < nv; ++j) g[j] = g[j] + A->tmp[j];
    }
    return 0;
}

/* Alg. 4 on the general problem, readings R19-R22 as in
 * orc_al_solve_ex (warm = 1 re-enters from x, lam, mu as given).  Returns 0
 * or a nonzero callback code. */
int32_t orc_al_general(const orc_gcons* Q, double* lam, double* mu, const double* l, const double* u,
                       int32_t m_hist, const orc_opts* o, const orc_al_opts* ao, double* x, int32_t warm,
                       orc_al_result* res)
{
    const int64_t nv = Q->nv;
    const int32_t neq = Q->m_eq + Q->m_nl, nin = Q->p_in + Q->p_nl;
    memset(res, 0, sizeof(*res));
    if (!warm) {
        for (int64_t j = 0; j < nv; ++j) x[j] = 0.0;                  /* R19 */
        for (int32_t k = 0; k < neq; ++k) lam[k] = 0.0;
        for (int32_t k = 0; k < nin; ++k) mu[k] = 0.0;
    }
    orc_clip(nv, x, l, u, x);
    orc_al_ctx A;
    A.Q = Q; A.lam = lam; A.mu = mu;
    A.hv = cons_buf(neq); A.gv = cons_buf(nin);
    A.weq = cons_buf(neq); A.win = cons_buf(nin);
    A.tmp = (double*)malloc(sizeof(double) * (size_t)(nv > 0 ? nv : 1));
    double rho = ao->rho0;
    int32_t rc = gcons_values(Q, x, A.hv, A.gv);
    double vprev = rc ? 0.0 : orc_al_violation(neq, A.hv, nin, A.gv, mu, rho);
    res->status = ORC_AL_MAX_OUTER;
    for (int32_t it = 0; it < ao->max_outer && rc == 0; ++it) {
        orc_opts oi = *o;
        const double tin = 0.1 * vprev;
        oi.tol = tin > o->tol ? tin : o->tol;                           /* R22 */
        A.rho = rho;
        orc_result ir;
        rc = orc_minimize_fg(nv, al_fg, &A, l, u, m_hist, &oi, x, &ir); /* Alg. 4 line 5 */
        if (rc) break;
        res->inner_iters_total += ir.iters;
        res->outer_iters = it + 1;
        if (ir.status == ORC_LINESEARCH_FAILURE) { res->status = ORC_AL_INNER_FAILURE; break; }
        rc = gcons_values(Q, x, A.hv, A.gv);
        if (rc) break;
        orc_al_update_multipliers(neq, lam, A.hv, nin, mu, A.gv, rho);  /* lines 6-7 */
        const double v = orc_al_violation(neq, A.hv, nin, A.gv, mu, rho);
        rho = orc_al_update_rho(rho, vprev, v, ao->rho_factor, ao->rho_cap);   /* line 8, R20 */
        vprev = v;
        if (ir.status == ORC_CONVERGED && v <= ao->feas_tol && oi.tol == o->tol) {
            res->status = ORC_CONVERGED;
            break;
        }
    }
    if (rc == 0) {
        double* gtmp = (double*)malloc(sizeof(double) * (size_t)(nv > 0 ? nv : 1));
        if (Q->P) res->f = orc_lsq_value(Q->P, x);
        else rc = Q->fg(Q->fg_ctx, x, gtmp, &res->f);
        free(gtmp);
        if (rc == 0) rc = gcons_values(Q, x, A.hv, A.gv);
        res->violation_inf = orc_al_violation(neq, A.hv, nin, A.gv, mu, rho);
        res->rho = rho;
    }
    free(A.hv); free(A.gv); free(A.weq); free(A.win); free(A.tmp);
    return rc;
}
