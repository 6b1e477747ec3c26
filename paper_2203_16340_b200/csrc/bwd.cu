// bwd.cu -- a3 of SURVEY.md 8(a): the backward GEMV g' = M~^T r' with the
// Alg. 1 iteration epilogue fused in, and the Gram / Alg. 3 tail.  This is
// the dominant kernel of the hot path (one full pass over M per iteration).
//
// Two variants, chosen per problem by launch_bwd:
//  * k_bwd_s  (m <= ~24K rows, 16-byte aligned column-major M): one CTA of
//    512 threads per SM, r' = fma(alpha, q, r) computed ONCE per CTA into
//    shared memory, then the CTA streams its balanced range of columns
//    (8 at a time, 16 x 16-byte loads in flight per thread) against it;
//  * k_bwd    (any shape): persistent CTAs of 256 threads, r' formed on the
//    fly from global r and q for every column group.
// Both write r' rows [c*m/G, (c+1)*m/G) into the other residual buffer (the
// carried residual of reading R13), run the per-variable epilogue
//   x' = clip(fma(alpha, p, x)), g' = dot + c + delta x' + sum_k ccoef_k E_k,
//   s = x' - x, y = g' - g (ring slot), Eq. (1) mask at x',
// accumulate the masked Gram of the NEXT basis {s_i, y_i, g'}, and end in a
// deterministic 2-level last-CTA tail: Gram reduce -> convergence test
// (R15) -> vector-free Alg. 3 -> ctrl->coef.
#include <cstdlib>
#include "common.cuh"

namespace lb {
#ifdef LB_TRACE
void trace_set_bwd(void* b, void* c) { trace_set_tu(b, c); }
#endif

constexpr int NTB = 512;                // threads of k_bwd_s (one CTA per SM)
constexpr int EPI_TILE = 256;           // epilogue tile rows
constexpr int BWD_SMEM_MAX = 210 * 1024;   // dynamic; + ~10 KB static <= 227 KB per CTA

#ifndef BWD_UNR
#define BWD_UNR 4              // row pairs per trip of the generic k_bwd's column stream: 32 x 16-byte
                               // loads in flight per thread; C5 chunk 3070 -> 2845 us per launch
                               // (6.5 -> 7.0 TB/s), bitwise-identical sums (profiles/r02_gemv_ab.txt)
#endif
#ifndef BWD_MINB
#define BWD_MINB 2             // resident CTAs per SM of the generic k_bwd (128-register cap)
#endif
// ---------------------------------------------------------------- column dots
// acc[c] += sum over this thread's rows of M[i, jg + c] * r'_i, rows
// i = 2 tid + 2 blockDim k (row pairs), two row pairs per loop trip.
#ifndef BWDS_UNR
#define BWDS_UNR 3             // row pairs per trip of k_bwd_s's column stream: C2 263.7 -> 261.2 us
                               // (4: 264.9 us); profiles/r02_gemv_ab_c2.txt
#endif
template <int NC, bool TWO = true>
__device__ __forceinline__ void col_dots_smem(const double* __restrict__ M0, int64_t ld, int64_t m,
                                              const double* rs, double* acc)
{
    const int64_t step = 2 * (int64_t)blockDim.x;
    int64_t i = 2 * (int64_t)threadIdx.x;
#if BWDS_UNR > 2
    // BWDS_UNR row pairs per trip (rows ascending per thread: the one-pair summation order)
    for (; TWO && i + (BWDS_UNR - 1) * step + 1 < m; i += BWDS_UNR * step) {
        double2 a[BWDS_UNR][NC];
#pragma unroll
        for (int u = 0; u < BWDS_UNR; ++u)
#pragma unroll
            for (int c = 0; c < NC; ++c)
                a[u][c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i + u * step));
#pragma unroll
        for (int u = 0; u < BWDS_UNR; ++u) {
            const double2 r = *reinterpret_cast<const double2*>(rs + i + u * step);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                acc[c] = fma(a[u][c].x, r.x, acc[c]);
                acc[c] = fma(a[u][c].y, r.y, acc[c]);
            }
        }
    }
#endif
    for (; TWO && i + step + 1 < m; i += 2 * step) {
        double2 a0[NC], a1[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            a0[c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i));
            a1[c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i + step));
        }
        const double2 r0 = *reinterpret_cast<const double2*>(rs + i);
        const double2 r1 = *reinterpret_cast<const double2*>(rs + i + step);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            acc[c] = fma(a0[c].x, r0.x, acc[c]);
            acc[c] = fma(a0[c].y, r0.y, acc[c]);
            acc[c] = fma(a1[c].x, r1.x, acc[c]);
            acc[c] = fma(a1[c].y, r1.y, acc[c]);
        }
    }
    for (; i < m; i += step) {
        if (i + 1 < m) {
            double2 a0[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) a0[c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i));
            const double2 r0 = *reinterpret_cast<const double2*>(rs + i);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                acc[c] = fma(a0[c].x, r0.x, acc[c]);
                acc[c] = fma(a0[c].y, r0.y, acc[c]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = fma(__ldcs(M0 + c * ld + i), rs[i], acc[c]);
        }
    }
}

// global-r' variant: r' = fma(alpha, q, r) (iter) or r, formed per row pair
template <int NC, bool VEC>
__device__ __forceinline__ void col_dots_glob(const double* __restrict__ M0, int64_t ld, int64_t m,
                                              const double* rcur, const double* qv, double alpha,
                                              bool iter, bool wr, double* rnext, int64_t i0, int64_t i1,
                                              double* acc)
{
    int64_t i = 2 * (int64_t)threadIdx.x;
#if BWD_UNR > 1
    // BWD_UNR row pairs per trip (BWD_UNR x NC independent 16-byte loads in flight per
    // thread); the per-column summation order is that of the one-pair loop below (each
    // thread's rows ascending), so the sums are bitwise those of BWD_UNR = 1
    if (VEC) {
        constexpr int U = BWD_UNR;
        const int64_t step = 2 * (int64_t)blockDim.x;
        for (; i + (U - 1) * step + 1 < m; i += U * step) {
            double2 rr[U];
#pragma unroll
            for (int u = 0; u < U; ++u) rr[u] = *reinterpret_cast<const double2*>(rcur + i + u * step);
            if (iter) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const double2 qq = *reinterpret_cast<const double2*>(qv + i + u * step);
                    rr[u].x = fma(alpha, qq.x, rr[u].x);
                    rr[u].y = fma(alpha, qq.y, rr[u].y);
                }
            }
            if (wr) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int64_t k = i + u * step;
                    if (k >= i0 && k < i1) rnext[k] = rr[u].x;
                    if (k + 1 >= i0 && k + 1 < i1) rnext[k + 1] = rr[u].y;
                }
            }
            double2 av[U][NC];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    av[u][c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i + u * step));
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    acc[c] = fma(av[u][c].x, rr[u].x, acc[c]);
                    acc[c] = fma(av[u][c].y, rr[u].y, acc[c]);
                }
        }
    }
#endif
    for (; i < m; i += 2 * (int64_t)blockDim.x) {
        const bool two = i + 1 < m;
        double r0, r1;
        if (VEC && two) {
            const double2 rr = *reinterpret_cast<const double2*>(rcur + i);
            r0 = rr.x; r1 = rr.y;
            if (iter) {
                const double2 qq = *reinterpret_cast<const double2*>(qv + i);
                r0 = fma(alpha, qq.x, r0);
                r1 = fma(alpha, qq.y, r1);
            }
        } else {
            r0 = rcur[i];
            r1 = two ? rcur[i + 1] : 0.0;
            if (iter) {
                r0 = fma(alpha, qv[i], r0);
                if (two) r1 = fma(alpha, qv[i + 1], r1);
            }
        }
        if (wr) {                                               // carried residual r' (R13)
            if (i >= i0 && i < i1) rnext[i] = r0;
            if (two && i + 1 >= i0 && i + 1 < i1) rnext[i + 1] = r1;
        }
        if (VEC && two) {
            double2 av[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) av[c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i));
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                acc[c] = fma(av[c].x, r0, acc[c]);
                acc[c] = fma(av[c].y, r1, acc[c]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                acc[c] = fma(__ldcs(M0 + c * ld + i), r0, acc[c]);
                if (two) acc[c] = fma(__ldcs(M0 + c * ld + i + 1), r1, acc[c]);
            }
        }
    }
}

// 8 block reductions with one barrier pair; dots[c] valid after the call.
__device__ __forceinline__ void reduce8(const double* acc, double* sh /* >= 8 * warps */, double* dots,
                                        int nc)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int c = 0; c < BWD_NB; ++c) {
        const double v = warp_red<0>(acc[c]);
        if (lane == 0) sh[w * BWD_NB + c] = v;
    }
    __syncthreads();
    if ((int)threadIdx.x < nc) {
        double s = sh[threadIdx.x];
        for (int k = 1; k < nw; ++k) s += sh[k * BWD_NB + threadIdx.x];
        dots[threadIdx.x] = s;
    }
    __syncthreads();
}

// ---------------------------------------------------------------- epilogue
struct EpiCtx {
    bool iter, gram;
    double alpha;
    double tol;             // ctrl->tol, ctrl->k, ctrl->rsel at kernel entry (used by the tail)
    long long k;
    int rsel;
    int nh, head, slot, mh, nb, ncons, branch;
    const double* bptr[2 * MAXH];
};

// Per-variable epilogue (Alg. 1 lines 7-9, Eq. (1)): x', g', s, y, mask, and
// the variable's row of the Gram tile.  Every global load comes first -- x, l,
// u, p, c, g, E_k and the ring values of the Gram row (straight into the tile
// row, 8 loads in flight per batch) -- because a load issued after a store
// through a pointer that may alias it cannot be hoisted: with the ring reads
// after the x / g / s / y stores (and each ring value stored to the tile before
// the next was loaded) the epilogue cost 2 nh + 2 dependent L2 round trips per
// variable (C4 shape: 19 us for k_bwd_wd's 2 tiles).
__device__ __forceinline__ void epilogue_var(const Prob& P, const Ctrl* C, const EpiCtx& E, int64_t v,
                                             double dval, double* trow, double* mkv, double& gmax,
                                             double& cnt)
{
    const double xo = P.x[v], lv = P.l[v], uv = P.u[v];
    const double pv = E.iter ? (E.branch ? P.pp[v] : P.pt[v]) : 0.0;
    const double cv = P.c ? P.c[v] : 0.0;
    const double go = E.iter ? P.g[v] : 0.0;
    double ev[MAXC];
#pragma unroll
    for (int k = 0; k < MAXC; ++k) ev[k] = k < E.ncons ? P.Ecol[k][v] : 0.0;
    const int nr = E.gram ? 2 * E.nh : 0;
    for (int b0 = 0; b0 < nr; b0 += 8) {
        double t8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t8[u] = b0 + u < nr ? E.bptr[b0 + u][v] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u)
            if (b0 + u < nr) trow[b0 + u] = t8[u];
    }
    double xn = xo;
    if (E.iter) xn = clipd(fma(E.alpha, pv, xo), lv, uv);      // Alg. 1 line 7
    double gn = dval;
    if (P.c) gn = gn + cv;
    gn = gn + P.delta * xn;
    if (P.ent != 0.0) gn = gn + P.ent * (log(xn) + 1.0);       // d/dx x log x (N2 entropy)
    for (int k = 0; k < E.ncons; ++k) gn = gn + C->ccoef[k] * ev[k];
    double sv = 0.0, yv = 0.0;
    if (E.iter) {
        const int64_t so = (int64_t)E.slot * P.n + v;
        sv = xn - xo;                                           // s^k
        yv = gn - go;                                           // y^k
        P.S[so] = sv;
        P.Y[so] = yv;
    }
    P.x[v] = xn;
    P.g[v] = gn;
    const bool fixed = (xn <= lv + P.eps && gn >= 0.0) || (xn >= uv - P.eps && gn <= 0.0);
    P.mask[v] = fixed ? 0 : 1;                                  // S^{k+1}, Eq. (1)
    if (!fixed) {
        const double ag = fabs(gn);
        gmax = ag > gmax ? ag : gmax;
        cnt += 1.0;
    }
    if (!E.gram) return;
    if (E.iter)                                                 // the new pair's slot holds (s, y) of this step
        for (int b = 0; b < E.nh; ++b)
            if (ring_slot(E.head, E.nh, b, E.mh) == E.slot) {
                trow[b] = sv;
                trow[E.nh + b] = yv;
            }
    trow[2 * E.nh] = gn;
    *mkv = fixed ? 0.0 : 1.0;
}

__device__ __forceinline__ void epi_init(const Prob& P, const Ctrl* C, int mode, EpiCtx& E)
{
    E.iter = mode == BWD_ITER;
    E.gram = mode == BWD_ITER || mode == BWD_SETUP;
    E.alpha = E.iter ? C->alpha : 0.0;
    E.tol = C->tol;
    E.k = C->k;
    E.rsel = C->rsel;
    E.nh = E.gram ? C->nh : 0;
    E.head = C->head;
    E.slot = C->slot;
    E.mh = P.mh;
    E.nb = 2 * E.nh + 1;
    E.ncons = P.n_eq + P.n_in;
    E.branch = C->branch;
    for (int b = 0; b < 2 * E.nh; ++b) {
        const int sl = ring_slot(E.head, E.nh, b < E.nh ? b : b - E.nh, E.mh);
        E.bptr[b] = (b < E.nh ? P.S : P.Y) + (int64_t)sl * P.n;
    }
}

#ifndef RECUR_WARP
#define RECUR_WARP 1           // Alg. 3 of the k_bwd tails on one warp (0: thread 0, serial sums; A/B)
#endif
__device__ void gram_tail_after(const Prob& P, Ctrl* C, const EpiCtx& E, double gmax, double cnt,
                                double* red, double* buf, int bufn, double* stash, double* Gs);

// Per-CTA Gram partial -> 2-level deterministic tail -> Alg. 3 (thread 0).
__device__ void gram_tail(const Prob& P, Ctrl* C, const EpiCtx& E, const GramEnt& ent, const double* gacc,
                          double gmax, double cnt, double* red, double* buf, int bufn, double* stash,
                          double* Gs)
{
    const int nh = E.nh, nb = E.nb, ne = nb * (nb + 1) / 2;
    const int ntot = ne + (P.screen_full ? nh : 0);
    double* out = P.gram_part + (int64_t)blockIdx.x * GRAM_STRIDE;
    ent.finalize(gacc, stash, out, ntot);
    gram_tail_after(P, C, E, gmax, cnt, red, buf, bufn, stash, Gs);
}

// After the CTA's Gram partial is in gram_part[cta]: the norms, then the
// 2-level deterministic tail and Alg. 3 (thread 0 of the last CTA).
__device__ void gram_tail_after(const Prob& P, Ctrl* C, const EpiCtx& E, double gmax, double cnt,
                                double* red, double* buf, int bufn, double* stash, double* Gs)
{
    const int G = gridDim.x, cta = blockIdx.x;
    const int nh = E.nh, nb = E.nb, ne = nb * (nb + 1) / 2;
    const int ntot = ne + (P.screen_full ? nh : 0);
    double* out = P.gram_part + (int64_t)cta * GRAM_STRIDE;
    TR_DECL
    const double bm = block_reduce<1>(gmax, red);
    const double bc = block_reduce<0>(cnt, red);
    if (threadIdx.x == 0) { out[ntot] = bm; out[ntot + 1] = bc; }
    const int nent = ntot + 2;
    auto sel = [ntot](int e) { return e == ntot ? 1 : 0; };
    {
        const int grp = cta / GRP, ngrp = (G + GRP - 1) / GRP;
        const int members = G - grp * GRP < GRP ? G - grp * GRP : GRP;
        if (!last_cta(P.tickets + T_BWD_G1 + grp, members)) return;
        TR_MARK(1);
        reduce_parts(P.gram_part + (int64_t)grp * GRP * GRAM_STRIDE, members, GRAM_STRIDE, nent, sel, buf,
                     bufn, stash, Gs);
        for (int e = threadIdx.x; e < nent; e += blockDim.x) P.gram_grp[(int64_t)grp * GRAM_STRIDE + e] = Gs[e];
        TR_MARK(2);
        if (!last_cta(P.tickets + T_BWD_G2, ngrp)) return;
        TR_MARK(3);
        reduce_parts(P.gram_grp, ngrp, GRAM_STRIDE, nent, sel, buf, bufn, stash, Gs);
        TR_MARK(4);
    }
    if (P.sharded) {                                         // sharded: local Gram pack
        for (int e = threadIdx.x; e < nent; e += blockDim.x) P.pk_loc[off_gram(P) + e] = Gs[e];
        if (P.p2p) p2p_push(P, XS_GRAM, off_gram(P), GRAM_STRIDE);
        return;
    }
#if RECUR_WARP
    if (threadIdx.x >= 32) return;
    if (E.iter && threadIdx.x == 0) C->rsel = E.rsel ^ 1;
    recur_decide_warp(P, C, Gs, nh, 0, E.tol, E.k);
#else
    if (threadIdx.x != 0) return;
    if (E.iter) C->rsel = E.rsel ^ 1;
    recur_decide_tk(P, C, Gs, nh, 0, E.tol, E.k);
#endif
    TR_MARK(5);
    TR_FLUSH(6, 11, G);
}

// Sharded: reduce the all-gathered Gram packs in rank order, then Alg. 3.
__global__ void __launch_bounds__(NT) k_gram_decide(Prob P, int mode)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    __shared__ double Gs[MAXE + MAXH + 2];
    if (P.p2p) {                                             // P2P exchange: the Gram packs of all ranks
        if (threadIdx.x == 0) p2p_wait_take(P, XS_GRAM, (unsigned long long)P.nranks);
        __syncthreads();
    }
    const int nh = C->nh, nb = 2 * nh + 1, ne = nb * (nb + 1) / 2;
    const int ntot = ne + (P.screen_full ? nh : 0), nent = ntot + 2;
    for (int e = threadIdx.x; e < nent; e += blockDim.x) {
        double s = e == ntot ? -INFINITY : 0.0;
        for (int p = 0; p < P.nranks; ++p) {
            const double v = P.gram_all[(int64_t)p * GRAM_STRIDE + e];
            s = e == ntot ? (v > s ? v : s) : s + v;
        }
        Gs[e] = s;
    }
    __syncthreads();
    if (threadIdx.x >= 32) return;
    const double tol = C->tol;
    const long long k = C->k;
    if (mode == BWD_ITER && threadIdx.x == 0) C->rsel = C->rsel ^ 1;
    recur_decide_warp(P, C, Gs, nh, 0, tol, k);
}

// ---------------------------------------------------------------- k_bwd_s
// Dynamic smem: rs[mpad] (r', later reused as Gram tile / reduce buffer),
// dots[cmax] (column dots of this CTA).
__global__ void __launch_bounds__(NTB, 1) k_bwd_s(Prob P, int mode, const double* rvec, double* gout,
                                                  int64_t mpad, int cmax)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(16) double smd[];
    TR_DECL
    double* rs = smd;
    double* dots = smd + mpad;
    __shared__ double red[NTB / 32 * BWD_NB];
    __shared__ double stash[NTB];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ double gd[BWD_NB];
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t m = P.m, ld = P.ld, ncols = P.ncols;
    const int64_t j0 = (int64_t)cta * ncols / G, j1 = (int64_t)(cta + 1) * ncols / G;
    const int64_t i0 = (int64_t)cta * m / G, i1 = (int64_t)(cta + 1) * m / G;
    const bool iter = mode == BWD_ITER;
    const int rsel = mode == BWD_PLAIN ? 0 : C->rsel;
    const double* rcur = mode == BWD_PLAIN ? rvec : P.rbuf[rsel];
    double* rnext = P.rbuf[rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    // r' once per CTA.  The loads of a batch of RPB rows are issued before any store: a
    // global store between them (rnext may alias rcur / q for the compiler) serialised
    // the 2 x 39 L2 round trips per thread (7% of the kernel's stall samples in ncu);
    // RPB = 20 covers C2's 20000 rows in two batches
    constexpr int RPB = 20;
    for (int64_t ib = threadIdx.x; ib < m; ib += RPB * (int64_t)NTB) {
        double rv[RPB], qv[RPB];
#pragma unroll
        for (int u = 0; u < RPB; ++u) {
            const int64_t i = ib + (int64_t)u * NTB;
            rv[u] = i < m ? __ldcg(rcur + i) : 0.0;
            qv[u] = (iter && i < m) ? __ldcg(P.q + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < RPB; ++u) {
            const int64_t i = ib + (int64_t)u * NTB;
            if (i < m) rs[i] = iter ? fma(alpha, qv[u], rv[u]) : rv[u];     // carried residual (R13)
        }
    }
    __syncthreads();
    TR_MARK(1);
    if (iter)
        for (int64_t i = i0 + threadIdx.x; i < i1; i += NTB) rnext[i] = rs[i];
    for (int64_t jg = j0; jg < j1; jg += BWD_NB) {
        const int nc = (int)(j1 - jg < BWD_NB ? j1 - jg : BWD_NB);
        double acc[BWD_NB];
#pragma unroll
        for (int c = 0; c < BWD_NB; ++c) acc[c] = 0.0;
        const double* M0 = P.M + jg * ld;
        switch (nc) {
            case 8: col_dots_smem<8>(M0, ld, m, rs, acc); break;
            case 7: col_dots_smem<7>(M0, ld, m, rs, acc); break;
            case 6: col_dots_smem<6>(M0, ld, m, rs, acc); break;
            case 5: col_dots_smem<5>(M0, ld, m, rs, acc); break;
            case 4: col_dots_smem<4>(M0, ld, m, rs, acc); break;
            case 3: col_dots_smem<3>(M0, ld, m, rs, acc); break;
            case 2: col_dots_smem<2>(M0, ld, m, rs, acc); break;
            default: col_dots_smem<1>(M0, ld, m, rs, acc); break;
        }
        reduce8(acc, red, gd, nc);
        if ((int)threadIdx.x < nc) dots[jg - j0 + threadIdx.x] = gd[threadIdx.x];
    }
    TR_MARK(2);
    __syncthreads();
    const int ccount = (int)(j1 - j0);
    const int nvg = P.split ? 2 : 1;
    const int nvar = ccount * nvg;
    if (mode == BWD_PLAIN) {
        for (int t = threadIdx.x; t < nvar; t += NTB) {
            const int jj = t % ccount, vv = t / ccount;
            const int64_t j = j0 + jj;
            const double dot = dots[jj];
            double dval = vv ? -dot : dot;
            if (P.colscale) dval = P.colscale[j] * dot;
            gout[j + vv * ncols] = dval;
        }
        return;
    }
    EpiCtx E;
    epi_init(P, C, mode, E);
    GramEnt ent;
    const int ne = E.nb * (E.nb + 1) / 2;
    ent.init(E.nb, ne, ne + (P.screen_full ? E.nh : 0), E.nh);
    double gacc[3] = {0.0, 0.0, 0.0};
    double gmax = 0.0, cnt = 0.0;
    double* tile = rs;                                          // r' no longer needed
    double* mk = rs + (int64_t)EPI_TILE * E.nb;
    for (int vb = 0; vb < nvar; vb += EPI_TILE) {
        const int rows = nvar - vb < EPI_TILE ? nvar - vb : EPI_TILE;
        const int t = threadIdx.x;
        if (t < rows) {
            const int idx = vb + t;
            const int jj = idx % ccount, vv = idx / ccount;
            const int64_t j = j0 + jj;
            const double dot = dots[jj];
            double dval = vv ? -dot : dot;
            if (P.colscale) dval = P.colscale[j] * dot;
            epilogue_var(P, C, E, j + vv * ncols, dval, tile + (int64_t)t * E.nb, mk + t, gmax, cnt);
        }
        if (E.gram) {
            __syncthreads();
            ent.accumulate(tile, mk, rows, E.nb, gacc);
        }
        __syncthreads();
    }
    TR_MARK(3);
    if (!E.gram) return;
    gram_tail(P, C, E, ent, gacc, gmax, cnt, red, rs, (int)(mpad < 4096 ? mpad : 4096), stash, Gs);
    TR_MARK(4);
    TR_FLUSH(5, 1, (int)(j1 - j0));
}

// ---------------------------------------------------------------- k_bwd_w (short columns)
// m < 2048 rows (C1, C4): a whole column is only a few KB, so a CTA-wide
// reduction per column group would dominate.  Each WARP owns WCOL columns
// at a time (lanes stride the rows with WRS row steps = 4 x WCOL 16-byte loads
// in flight per lane, r' from shared memory), reduces with shuffles only, and
// its lanes run the epilogue into the warp's own tile rows.  The masked Gram
// of the next basis is accumulated PER WARP (lane l owns entries l, l+32, ..;
// warp-private smem partials, __syncwarp only), so no CTA barrier interrupts
// the column stream; the CTA sums its warps' partials in warp order once.
#ifndef BWDW_WRS
#define BWDW_WRS 4             // row steps of 64 rows per trip of k_bwd_w's column stream
#endif
#ifndef BWDW_PRED
#define BWDW_PRED 1            // the last partial trip is one predicated batch (zeros beyond m): C4
                               // 1000 x 100000 k_bwd_w 177 -> 162 us with BWDW_MINB 2 (profiles/r02_gemv_ab_c4.txt)
#endif
#ifndef BWDW_MINB
#define BWDW_MINB 2            // resident CTAs per SM of k_bwd_w (128-register cap: no spill in the
                               // predicated trip; 3 CTAs/SM at 80 registers gained nothing)
#endif
#ifndef BWDW_WCOL
#define BWDW_WCOL 4            // columns per warp group of k_bwd_w (4 or 8)
#endif
constexpr int WCOL = BWDW_WCOL;
constexpr int WRS = BWDW_WRS;                   // row steps of 64 rows per trip
constexpr int WROWS = WCOL * 2;                 // tile rows per warp (split: 2 vars per column)
constexpr int WTILE = (NT / 32) * WROWS;        // tile rows per CTA
constexpr int WG_STRIDE = MAXE + MAXH + 1;      // per-warp Gram partial slots (max; launch passes the m_hist size)

template <int NC, int RS = WRS>
__device__ __forceinline__ void warp_col_dots(const double* __restrict__ M0, int64_t ld, int64_t m,
                                              const double* rs, double* acc)
{
    const int lane = threadIdx.x & 31;
    int64_t i = 2 * lane;
    for (; i + 64 * (RS - 1) + 1 < m; i += 64 * RS) {
        double2 av[RS][NC];
#pragma unroll
        for (int u = 0; u < RS; ++u)
#pragma unroll
            for (int c = 0; c < NC; ++c)
                av[u][c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i + 64 * u));
#pragma unroll
        for (int u = 0; u < RS; ++u) {
            const double2 r = *reinterpret_cast<const double2*>(rs + i + 64 * u);
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                acc[c] = fma(av[u][c].x, r.x, acc[c]);
                acc[c] = fma(av[u][c].y, r.y, acc[c]);
            }
        }
    }
#if BWDW_PRED
    // the remaining (< WRS) row steps as ONE batch of loads: rows >= m contribute exact zeros,
    // so every column sees the same additions in the same order as the one-step loop below
    if (i < m) {
        double2 av[RS][NC];
        double2 rv[RS];
#pragma unroll
        for (int u = 0; u < RS; ++u) {
            const int64_t k = i + 64 * u;
            const bool full = k + 1 < m, half = k < m;
            rv[u] = full ? *reinterpret_cast<const double2*>(rs + k) : make_double2(half ? rs[k] : 0.0, 0.0);
#pragma unroll
            for (int c = 0; c < NC; ++c)
                av[u][c] = full ? __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + k))
                                : make_double2(half ? __ldcs(M0 + c * ld + k) : 0.0, 0.0);
        }
#pragma unroll
        for (int u = 0; u < RS; ++u)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                acc[c] = fma(av[u][c].x, rv[u].x, acc[c]);
                acc[c] = fma(av[u][c].y, rv[u].y, acc[c]);
            }
        return;
    }
#endif
    for (; i < m; i += 64) {
        if (i + 1 < m) {
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double2 a = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i));
                acc[c] = fma(a.x, rs[i], acc[c]);
                acc[c] = fma(a.y, rs[i + 1], acc[c]);
            }
        } else {
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = fma(__ldcs(M0 + c * ld + i), rs[i], acc[c]);
        }
    }
}

__global__ void __launch_bounds__(NT, BWDW_MINB) k_bwd_w(Prob P, int mode, const double* rvec, double* gout, int mpad,
                                                int wgs)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(16) double smw[];
    TR_DECL
    double* rs = smw;                               // r' [mpad]
    double* tile = smw + mpad;                      // [WTILE][MAXB]
    double* mk = tile + WTILE * MAXB;               // [WTILE]
    double* wg = mk + WTILE;                        // [NT/32][wgs] per-warp Gram partials
    __shared__ double red[NT / 32 * BWD_NB];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ unsigned char ea[MAXE + MAXH], eb[MAXE + MAXH];   // entry -> basis pair (eb = 255: full norm)
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t m = P.m, ld = P.ld, ncols = P.ncols;
    const int64_t j0 = (int64_t)cta * ncols / G, j1 = (int64_t)(cta + 1) * ncols / G;
    const int64_t i0 = (int64_t)cta * m / G, i1 = (int64_t)(cta + 1) * m / G;
    const bool iter = mode == BWD_ITER;
    const int rsel = mode == BWD_PLAIN ? 0 : C->rsel;
    const double* rcur = mode == BWD_PLAIN ? rvec : P.rbuf[rsel];
    double* rnext = P.rbuf[rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    for (int64_t ib = threadIdx.x; ib < m; ib += 8 * (int64_t)NT) {    // 8 rows' loads before any store
        double rv[8], qv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = ib + (int64_t)u * NT;
            rv[u] = i < m ? rcur[i] : 0.0;
            qv[u] = (iter && i < m) ? P.q[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = ib + (int64_t)u * NT;
            if (i >= m) continue;
            double r = rv[u];
            if (iter) {
                r = fma(alpha, qv[u], r);                       // carried residual (R13)
                if (i >= i0 && i < i1) rnext[i] = r;
            }
            rs[i] = r;
        }
    }
    const bool epi = mode != BWD_PLAIN;
    EpiCtx E;
    if (epi) epi_init(P, C, mode, E);
    const bool gram = epi && E.gram;
    const int nb = epi ? E.nb : 1;
    const int ne = nb * (nb + 1) / 2;
    const int ntot = gram ? ne + (P.screen_full ? E.nh : 0) : 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = NT / 32;
    double* wgw = wg + (int64_t)w * wgs;
    if (gram) {
        for (int e = threadIdx.x; e < ntot; e += NT) {          // upper triangle, row-major; then ||y_i||^2
            if (e < ne) {
                int aa = 0, rem = e;
                while (rem >= nb - aa) { rem -= nb - aa; ++aa; }
                ea[e] = (unsigned char)aa; eb[e] = (unsigned char)(aa + rem);
            } else {
                ea[e] = (unsigned char)(E.nh + (e - ne)); eb[e] = 255;
            }
        }
        for (int e = lane; e < ntot; e += 32) wgw[e] = 0.0;
    }
    __syncthreads();
    TR_MARK(1);
    double gmax = 0.0, cnt = 0.0;
    const int nvg = P.split ? 2 : 1;
    const int64_t ncl = j1 - j0;
    const int64_t ngroups = (ncl + WCOL - 1) / WCOL;
    const int rows_per_warp = WCOL * nvg;
    const int trow0 = w * WROWS;
    for (int64_t grp = w; grp < ngroups; grp += nw) {
        const int64_t jg = j0 + grp * WCOL;
        const int nc = (int)(j1 - jg < WCOL ? j1 - jg : WCOL);
        double acc[WCOL];
#pragma unroll
        for (int c = 0; c < WCOL; ++c) acc[c] = 0.0;
        const double* M0 = P.M + jg * ld;
        switch (nc) {
#if BWDW_WCOL > 4
            case 8: warp_col_dots<8>(M0, ld, m, rs, acc); break;
            case 7: warp_col_dots<7>(M0, ld, m, rs, acc); break;
            case 6: warp_col_dots<6>(M0, ld, m, rs, acc); break;
            case 5: warp_col_dots<5>(M0, ld, m, rs, acc); break;
#endif
            case 4: warp_col_dots<4>(M0, ld, m, rs, acc); break;
            case 3: warp_col_dots<3>(M0, ld, m, rs, acc); break;
            case 2: warp_col_dots<2>(M0, ld, m, rs, acc); break;
            default: warp_col_dots<1>(M0, ld, m, rs, acc); break;
        }
#pragma unroll
        for (int c = 0; c < WCOL; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        // all lanes now hold the column dots (xor butterfly: identical in every lane)
        if (lane < rows_per_warp) {
            const int t = trow0 + lane;
            if (lane < nc * nvg) {
                const int jj = lane % nc, vv = lane / nc;
                double dot = acc[0];
#pragma unroll
                for (int c = 1; c < WCOL; ++c)
                    if (jj == c) dot = acc[c];
                const int64_t j = jg + jj;
                double dval = vv ? -dot : dot;
                if (P.colscale) dval = P.colscale[j] * dot;
                if (!epi) gout[j + vv * ncols] = dval;
                else epilogue_var(P, C, E, j + vv * ncols, dval, tile + (int64_t)t * nb, mk + t, gmax, cnt);
            } else if (gram) {
                for (int b = 0; b < nb; ++b) tile[(int64_t)t * nb + b] = 0.0;
                mk[t] = 0.0;
            }
        }
        if (gram) {
            __syncwarp();
            const double* tw = tile + (int64_t)trow0 * nb;
            const double* mw = mk + trow0;
            for (int e = lane; e < ntot; e += 32) {
                const int aa = ea[e], bb = eb[e];
                double s = 0.0;
                if (bb != 255) {
                    for (int r = 0; r < rows_per_warp; ++r)
                        if (mw[r] != 0.0) s = fma(tw[r * nb + aa], tw[r * nb + bb], s);
                } else {
                    for (int r = 0; r < rows_per_warp; ++r) s = fma(tw[r * nb + aa], tw[r * nb + aa], s);
                }
                wgw[e] += s;
            }
            __syncwarp();                                       // tile rows are rewritten next group
        }
    }
    TR_MARK(2);
    if (!gram) return;
    __syncthreads();
    double* out = P.gram_part + (int64_t)blockIdx.x * GRAM_STRIDE;
    for (int e = threadIdx.x; e < ntot; e += NT) {              // warp partials in warp order
        double s = wg[e];
        for (int k = 1; k < nw; ++k) s += wg[(int64_t)k * wgs + e];
        out[e] = s;
    }
    gram_tail_after(P, C, E, gmax, cnt, red, rs, mpad < 4096 ? mpad : 4096, stash, Gs);
    TR_MARK(3);
    TR_FLUSH(4, 2, (int)(j1 - j0));
}

// ---------------------------------------------------------------- k_bwd_wd (short columns, deferred epilogue)
// k_bwd_w's per-warp column stream (WCOL columns per warp group, shuffle
// reductions, r' in shared memory) with the epilogue taken OUT of the stream:
// the warps only stream and park the column dots in shared memory, so no warp
// stalls on the epilogue's dependent loads while the others stream; then the
// whole CTA runs k_bwd_s's epilogue (one variable per thread, NT-row Gram
// tiles) and the same 2-level tail.  A/B against k_bwd_w: BWDW_DEFER.
#ifndef BWDW_DEFER
#define BWDW_DEFER 1
#endif
#ifndef BWDWD_MINB
#define BWDWD_MINB 2
#endif
__global__ void __launch_bounds__(NT, BWDWD_MINB) k_bwd_wd(Prob P, int mode, const double* rvec, double* gout,
                                                         int mpad, int cpad)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(16) double smw[];
    TR_DECL
    double* rs = smw;                               // r' [mpad]; later the tail's reduce buffer
    double* dots = smw + mpad;                      // [cpad] column dots of this CTA
    double* tile = dots + cpad;                     // [NT][nb] epilogue Gram tile, then mk[NT]
    __shared__ double red[NT / 32 * BWD_NB];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ int s_next;                          // next column unit
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t m = P.m, ld = P.ld, ncols = P.ncols;
    const int64_t j0 = (int64_t)cta * ncols / G, j1 = (int64_t)(cta + 1) * ncols / G;
    const int64_t i0 = (int64_t)cta * m / G, i1 = (int64_t)(cta + 1) * m / G;
    const bool iter = mode == BWD_ITER;
    const int rsel = mode == BWD_PLAIN ? 0 : C->rsel;
    const double* rcur = mode == BWD_PLAIN ? rvec : P.rbuf[rsel];
    double* rnext = P.rbuf[rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    if (threadIdx.x == 0) s_next = 0;
    for (int64_t ib = threadIdx.x; ib < m; ib += 8 * (int64_t)NT) {    // 8 rows' loads before any store
        double rv[8], qv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = ib + (int64_t)u * NT;
            rv[u] = i < m ? rcur[i] : 0.0;
            qv[u] = (iter && i < m) ? P.q[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = ib + (int64_t)u * NT;
            if (i >= m) continue;
            double r = rv[u];
            if (iter) {
                r = fma(alpha, qv[u], r);                       // carried residual (R13)
                if (i >= i0 && i < i1) rnext[i] = r;
            }
            rs[i] = r;
        }
    }
    __syncthreads();
    TR_MARK(1);
    const int lane = threadIdx.x & 31;
    const int64_t ncl = j1 - j0;
    // Units of WCOL columns go to the warps dynamically (a shared-memory counter), so
    // the warps of a CTA finish their streams within about one unit of each other
    // (C4 shape: 3126 -> 3297 solver iterations / s against round-robin units).  A
    // unit's dots do not depend on the warp that streams it: deterministic.  A tail of
    // single-column units (16 row steps per trip) was measured slower (3190-3231).
    const int64_t nbulk = ncl;
    const int nunits = (int)((nbulk + WCOL - 1) / WCOL);
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&s_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= nunits) break;
        const int64_t jg = j0 + (int64_t)u * WCOL;
        const int nc = (int)(nbulk - (int64_t)u * WCOL < WCOL ? nbulk - (int64_t)u * WCOL : WCOL);
        double acc[WCOL];
#pragma unroll
        for (int c = 0; c < WCOL; ++c) acc[c] = 0.0;
        const double* M0 = P.M + jg * ld;
        switch (nc) {
#if BWDW_WCOL > 4
            case 8: warp_col_dots<8>(M0, ld, m, rs, acc); break;
            case 7: warp_col_dots<7>(M0, ld, m, rs, acc); break;
            case 6: warp_col_dots<6>(M0, ld, m, rs, acc); break;
            case 5: warp_col_dots<5>(M0, ld, m, rs, acc); break;
#endif
            case 4: warp_col_dots<4>(M0, ld, m, rs, acc); break;
            case 3: warp_col_dots<3>(M0, ld, m, rs, acc); break;
            case 2: warp_col_dots<2>(M0, ld, m, rs, acc); break;
            default: warp_col_dots<1>(M0, ld, m, rs, acc); break;
        }
#pragma unroll
        for (int c = 0; c < WCOL; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        if (lane < nc) {
            double dot = acc[0];
#pragma unroll
            for (int c = 1; c < WCOL; ++c)
                if (lane == c) dot = acc[c];
            dots[jg - j0 + lane] = dot;
        }
    }
    TR_MARK(2);
    __syncthreads();
    TR_MARK(3);
    const int ccount = (int)ncl;
    const int nvg = P.split ? 2 : 1;
    const int nvar = ccount * nvg;
    if (mode == BWD_PLAIN) {
        for (int t = threadIdx.x; t < nvar; t += NT) {
            const int jj = t % ccount, vv = t / ccount;
            const int64_t j = j0 + jj;
            const double dot = dots[jj];
            double dval = vv ? -dot : dot;
            if (P.colscale) dval = P.colscale[j] * dot;
            gout[j + vv * ncols] = dval;
        }
        return;
    }
    EpiCtx E;
    epi_init(P, C, mode, E);
    GramEnt ent;
    const int ne = E.nb * (E.nb + 1) / 2;
    ent.init(E.nb, ne, ne + (P.screen_full ? E.nh : 0), E.nh);
    double gacc[3] = {0.0, 0.0, 0.0};
    double gmax = 0.0, cnt = 0.0;
    double* mk = tile + (int64_t)NT * E.nb;
    for (int vb = 0; vb < nvar; vb += NT) {
        const int rows = nvar - vb < NT ? nvar - vb : NT;
        const int t = threadIdx.x;
        if (t < rows) {
            const int idx = vb + t;
            const int jj = idx % ccount, vv = idx / ccount;
            const int64_t j = j0 + jj;
            const double dot = dots[jj];
            double dval = vv ? -dot : dot;
            if (P.colscale) dval = P.colscale[j] * dot;
            epilogue_var(P, C, E, j + vv * ncols, dval, tile + (int64_t)t * E.nb, mk + t, gmax, cnt);
        }
        if (E.gram) {
            __syncthreads();
            ent.accumulate(tile, mk, rows, E.nb, gacc);
        }
        __syncthreads();
    }
    TR_MARK(4);
    if (!E.gram) return;
    gram_tail(P, C, E, ent, gacc, gmax, cnt, red, rs, mpad < 4096 ? mpad : 4096, stash, Gs);
    TR_MARK(5);
    TR_FLUSH(6, 3, (int)ncl);
}

// ---------------------------------------------------------------- k_bwd_wo (short columns, overlapped epilogue)
// k_bwd_wd's dynamic column units, with the epilogue cut into mini-tiles of MT
// columns run by the warp that completes a mini-tile's last unit (a shared
// counter per mini-tile) right away, while the other warps keep streaming: the
// epilogue of its columns (one lane per column; the two halves of a split
// operator in turn) into a warp-private tile, and the mini-tile's masked-Gram
// partial into shared memory; the CTA sums the partials in mini-tile order.  The dependent loads of the epilogue then overlap the other
// warps' column streams instead of following them (k_bwd_wd: 14.6 us of its
// 142 us at the C4 shape).  A partial does not depend on the warp that computes
// it: deterministic.  BWDW_OVL selects it over k_bwd_wd (A/B).
#ifndef BWDW_OVL
#define BWDW_OVL 1
#endif
constexpr int MT = 32;                          // columns per epilogue mini-tile
__global__ void __launch_bounds__(NT, BWDWD_MINB) k_bwd_wo(Prob P, int mode, const double* rvec, double* gout,
                                                         int mpad, int cpad, int pstride)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(16) double smw[];
    TR_DECL
    const int nw = NT / 32, w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nbm = 2 * P.mh + 1;
    const int nmt_max = (cpad + MT - 1) / MT;
    double* rs = smw;                                           // r' [mpad]; later the tail's reduce buffer
    double* dots = smw + mpad;                                  // [cpad]
    double* wtile = dots + cpad + (int64_t)w * MT * (nbm + 1);  // this warp's [MT][nbm] rows, then mk[MT]
    double* part = dots + cpad + (int64_t)nw * MT * (nbm + 1);  // [2 nmt_max][pstride] mini-tile partials
    int* mt_done = reinterpret_cast<int*>(part + (int64_t)2 * nmt_max * pstride);   // [nmt_max]
    __shared__ double red[NT / 32 * BWD_NB];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ int s_next;
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t m = P.m, ld = P.ld, ncols = P.ncols;
    const int64_t j0 = (int64_t)cta * ncols / G, j1 = (int64_t)(cta + 1) * ncols / G;
    const int64_t i0 = (int64_t)cta * m / G, i1 = (int64_t)(cta + 1) * m / G;
    const bool iter = mode == BWD_ITER;
    const int rsel = mode == BWD_PLAIN ? 0 : C->rsel;
    const double* rcur = mode == BWD_PLAIN ? rvec : P.rbuf[rsel];
    double* rnext = P.rbuf[rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    const int ccount = (int)(j1 - j0);
    const int nmt = (ccount + MT - 1) / MT;
    LB_CHECK(ccount >= 1 && ccount <= cpad && nmt <= nmt_max);
    if (threadIdx.x == 0) s_next = 0;
    for (int i = threadIdx.x; i < nmt; i += NT) mt_done[i] = 0;
    for (int64_t ib = threadIdx.x; ib < m; ib += 8 * (int64_t)NT) {    // 8 rows' loads before any store
        double rv[8], qv[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = ib + (int64_t)u * NT;
            rv[u] = i < m ? rcur[i] : 0.0;
            qv[u] = (iter && i < m) ? P.q[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int64_t i = ib + (int64_t)u * NT;
            if (i >= m) continue;
            double r = rv[u];
            if (iter) {
                r = fma(alpha, qv[u], r);                       // carried residual (R13)
                if (i >= i0 && i < i1) rnext[i] = r;
            }
            rs[i] = r;
        }
    }
    __syncthreads();
    TR_MARK(1);
    const bool epi = mode != BWD_PLAIN;
    EpiCtx E;
    if (epi) epi_init(P, C, mode, E);                           // first needed after a warp's first mini-tile
    const bool gram = epi && E.gram;
    const int nb = epi ? E.nb : 1;
    const int ne = nb * (nb + 1) / 2;
    const int ntot = gram ? ne + (P.screen_full ? E.nh : 0) : 0;
    // Gram entry -> basis pair for this lane's entries e = lane + 32 k (upper triangle, row-major,
    // then ||y_i||^2 with b = 255); registers for k < 4, computed on the fly beyond
    auto entry = [&](int e, int& aa, int& bb) {
        if (e < ne) {
            int rem = e;
            aa = 0;
            while (rem >= nb - aa) { rem -= nb - aa; ++aa; }
            bb = aa + rem;
        } else {
            aa = E.nh + (e - ne);
            bb = 255;
        }
    };
    int eaa[4], ebb[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) entry(lane + 32 * q, eaa[q], ebb[q]);
    const int nunits = (ccount + WCOL - 1) / WCOL;
    const int nvg = P.split ? 2 : 1;
    double gmax = 0.0, cnt = 0.0;
    double* mkw = wtile + MT * nbm;
    // epilogue + Gram partial of mini-tile i (its dots are complete); whole warp
    auto do_mt = [&](int i) {
        const int c0 = i * MT, cn = ccount - c0 < MT ? ccount - c0 : MT;
        for (int vv = 0; vv < nvg; ++vv) {
            double* tr = wtile + lane * nbm;
            if (lane < cn) {
                const int jj = c0 + lane;
                const int64_t j = j0 + jj;
                const double dot = dots[jj];
                double dval = vv ? -dot : dot;
                if (P.colscale) dval = P.colscale[j] * dot;
                epilogue_var(P, C, E, j + vv * ncols, dval, tr, mkw + lane, gmax, cnt);
            } else if (gram) {
                for (int b = 0; b < nb; ++b) tr[b] = 0.0;
                mkw[lane] = 0.0;
            }
            __syncwarp();
            if (gram) {
                double* po = part + (int64_t)(i * nvg + vv) * pstride;
                LB_CHECK(i * nvg + vv < 2 * nmt_max && ntot <= pstride && nb <= nbm);
                for (int e = lane; e < ntot; e += 32) {
                    int aa, bb;
                    if (e < 128) {
                        const int q = e >> 5;
                        aa = q == 0 ? eaa[0] : q == 1 ? eaa[1] : q == 2 ? eaa[2] : eaa[3];
                        bb = q == 0 ? ebb[0] : q == 1 ? ebb[1] : q == 2 ? ebb[2] : ebb[3];
                    } else {
                        entry(e, aa, bb);
                    }
                    double sacc = 0.0;
                    if (bb != 255) {
                        for (int r0 = 0; r0 < MT; r0 += 8) {
                            double m8[8], a8[8], b8[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                m8[q] = mkw[r0 + q];
                                a8[q] = wtile[(r0 + q) * nbm + aa];
                                b8[q] = wtile[(r0 + q) * nbm + bb];
                            }
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                if (m8[q] != 0.0) sacc = fma(a8[q], b8[q], sacc);
                        }
                    } else {
                        for (int r0 = 0; r0 < MT; r0 += 8) {
                            double a8[8];
#pragma unroll
                            for (int q = 0; q < 8; ++q) a8[q] = wtile[(r0 + q) * nbm + aa];
#pragma unroll
                            for (int q = 0; q < 8; ++q) sacc = fma(a8[q], a8[q], sacc);
                        }
                    }
                    po[e] = sacc;
                }
            }
            __syncwarp();                                       // the tile rows are rewritten next
        }
    };
    for (;;) {
        int u = 0;
        if (lane == 0) u = atomicAdd(&s_next, 1);
        u = __shfl_sync(0xffffffffu, u, 0);
        if (u >= nunits) break;
        const int64_t jg = j0 + (int64_t)u * WCOL;
        const int nc = ccount - u * WCOL < WCOL ? ccount - u * WCOL : WCOL;
        double acc[WCOL];
#pragma unroll
        for (int c = 0; c < WCOL; ++c) acc[c] = 0.0;
        const double* M0 = P.M + jg * ld;
        switch (nc) {
#if BWDW_WCOL > 4
            case 8: warp_col_dots<8>(M0, ld, m, rs, acc); break;
            case 7: warp_col_dots<7>(M0, ld, m, rs, acc); break;
            case 6: warp_col_dots<6>(M0, ld, m, rs, acc); break;
            case 5: warp_col_dots<5>(M0, ld, m, rs, acc); break;
#endif
            case 4: warp_col_dots<4>(M0, ld, m, rs, acc); break;
            case 3: warp_col_dots<3>(M0, ld, m, rs, acc); break;
            case 2: warp_col_dots<2>(M0, ld, m, rs, acc); break;
            default: warp_col_dots<1>(M0, ld, m, rs, acc); break;
        }
#pragma unroll
        for (int c = 0; c < WCOL; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        if (lane < nc) {
            double dot = acc[0];
#pragma unroll
            for (int c = 1; c < WCOL; ++c)
                if (lane == c) dot = acc[c];
            LB_CHECK(u * WCOL + lane < ccount);
            dots[u * WCOL + lane] = dot;
        }
        __syncwarp();
        const int mt = (u * WCOL) / MT;
        LB_CHECK(mt < nmt);
        int prev = 0;
        if (lane == 0) {                                        // release the unit to its mini-tile
            __threadfence_block();
            prev = atomicAdd(&mt_done[mt], 1);
            __threadfence_block();
        }
        prev = __shfl_sync(0xffffffffu, prev, 0);
        const int cmt = ccount - mt * MT < MT ? ccount - mt * MT : MT;
        if (epi && prev + 1 == (cmt + WCOL - 1) / WCOL) {          // this warp completed the mini-tile
            __syncwarp();                                       // lane 0's acquire before every lane's reads
            do_mt(mt);
        }
    }
    TR_MARK(2);
    TR_MARK(3);
    __syncthreads();
    TR_MARK(4);
    if (!epi) {
        for (int t = threadIdx.x; t < ccount * nvg; t += NT) {
            const int jj = t % ccount, vv = t / ccount;
            const int64_t j = j0 + jj;
            const double dot = dots[jj];
            double dval = vv ? -dot : dot;
            if (P.colscale) dval = P.colscale[j] * dot;
            gout[j + vv * ncols] = dval;
        }
        return;
    }
    if (!gram) return;
    double* out = P.gram_part + (int64_t)cta * GRAM_STRIDE;
    for (int e = threadIdx.x; e < ntot; e += NT) {              // mini-tile partials in mini-tile order
        double sacc = 0.0;
        for (int k = 0; k < nmt * nvg; ++k) sacc += part[(int64_t)k * pstride + e];
        out[e] = sacc;
    }
    gram_tail_after(P, C, E, gmax, cnt, red, rs, mpad < 4096 ? mpad : 4096, stash, Gs);
    TR_MARK(5);
    TR_FLUSH(6, 3, ccount);
}

// ---------------------------------------------------------------- TMA / mbarrier helpers (k_qepi_t, k_qepi_d)
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned cnt)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(cnt));
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* b, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b)
{
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned parity)
{
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
                 ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// ---------------------------------------------------------------- k_qpu (QP objective)
// QP objective (the kernel dual SVM): f = 1/2 x^T Q~ x + ..., the
// gradient is carried as w = Q~ x (like the LSQ residual, R13): w' =
// fma(alpha, q, w) with q = Q~ p from k_fwd, so an iteration needs ONE pass
// over Q.  This elementwise kernel is the "a3" step of the QP: w', then the
// same per-variable epilogue, Gram and Alg. 3 tail as k_bwd.
__global__ void __launch_bounds__(NT) k_qpu(Prob P, int mode, int bufn)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(16) double smq[];
    __shared__ double red[NT / 32 * BWD_NB];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    const bool iter = mode == BWD_ITER;
    const int rsel = C->rsel;
    const double* wcur = P.rbuf[rsel];
    double* wnext = P.rbuf[rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    EpiCtx E;
    epi_init(P, C, mode, E);
    double* tile = smq;
    double* mk = smq + (size_t)NT * E.nb;
    GramEnt ent;
    const int ne = E.nb * (E.nb + 1) / 2;
    ent.init(E.nb, ne, ne + (P.screen_full ? E.nh : 0), E.nh);
    double gacc[3] = {0.0, 0.0, 0.0};
    double gmax = 0.0, cnt = 0.0;
    const int64_t n = P.n;
    const double rho = C->rho;
    if (P.tp && iter) {                                         // carried h' = h + alpha A p (N2)
        const int64_t K = P.tm + P.tn;
        for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < K; k += (int64_t)gridDim.x * NT)
            wnext[k] = fma(alpha, P.tap[k], wcur[k]);
    }
    const bool small = n < (1LL << 31);
    for (int64_t base = (int64_t)blockIdx.x * NT; base < n; base += (int64_t)gridDim.x * NT) {
        const int64_t v = base + threadIdx.x;
        if (v < n) {
            double w;
            if (P.tp) {
                // marginal multipliers of row i and column j: (rho h + lam)_i + (rho h + lam)_{tm+j}
                int64_t i, j;
                if (small) {
                    const unsigned vv = (unsigned)v, tmu = (unsigned)P.tm;
                    j = vv / tmu; i = vv - (unsigned)j * tmu;
                } else {
                    j = v / P.tm; i = v - j * P.tm;
                }
                const int64_t kj = P.tm + j;
                double hi = wcur[i], hj = wcur[kj];
                if (iter) { hi = fma(alpha, P.tap[i], hi); hj = fma(alpha, P.tap[kj], hj); }
                w = (rho * hi + P.tlam[i]) + (rho * hj + P.tlam[kj]);
            } else {
                w = wcur[v];
                if (iter) {
                    w = fma(alpha, P.q[v], w);                  // carried w' = Q~ x'
                    wnext[v] = w;
                }
            }
            epilogue_var(P, C, E, v, w, tile + (int64_t)threadIdx.x * E.nb, mk + threadIdx.x, gmax, cnt);
        } else if (E.gram) {
            for (int b = 0; b < E.nb; ++b) tile[(int64_t)threadIdx.x * E.nb + b] = 0.0;
            mk[threadIdx.x] = 0.0;
        }
        if (E.gram) {
            __syncthreads();
            ent.accumulate(tile, mk, NT, E.nb, gacc);
            __syncthreads();
        }
    }
    if (!E.gram) return;
    gram_tail(P, C, E, ent, gacc, gmax, cnt, red, smq, bufn, stash, Gs);
}

// ---------------------------------------------------------------- k_qepi (register Gram)
// QP / transport epilogue for m_hist <= (NBX - 1) / 2: each thread keeps the
// variable's Gram row (S, Y, g) in registers and accumulates the upper
// triangle of B^T diag(mask) B and the unmasked ||B_b||^2 in NBX (NBX + 1) / 2
// + NBX register accumulators over a grid-stride loop (fixed order per
// thread), reduced once per CTA (warp shuffles, then warps in order).  No
// shared-memory tile, no per-tile barriers: for n in the millions (N2) the
// Gram costs ~66 DFMA per variable, well under the epilogue's HBM time.
template <int NBX>
__global__ void __launch_bounds__(NT, 1) k_qepi(Prob P, int mode)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    constexpr int NE = NBX * (NBX + 1) / 2, NA = NE + NBX;
    __shared__ double red[NT / 32];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ double buf[NT / 32 * NA > 4096 ? NT / 32 * NA : 4096];
    const bool iter = mode == BWD_ITER;
    const double* wcur = P.rbuf[C->rsel];
    double* wnext = P.rbuf[C->rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    const double rho = C->rho;
    EpiCtx E;
    epi_init(P, C, mode, E);
    const int64_t n = P.n;
    if (P.tp && iter) {                                         // carried h' = h + alpha A p (N2)
        const int64_t K = P.tm + P.tn;
        for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < K; k += (int64_t)gridDim.x * NT)
            wnext[k] = fma(alpha, P.tap[k], wcur[k]);
    }
    double acc[NA];
#pragma unroll
    for (int k = 0; k < NA; ++k) acc[k] = 0.0;
    double gmax = 0.0, cnt = 0.0;
    const bool small = n < (1LL << 31);
    const int nh = E.nh;
    for (int64_t v = (int64_t)blockIdx.x * NT + threadIdx.x; v < n; v += (int64_t)gridDim.x * NT) {
        // ---- every load of the variable first (memory-level parallelism: the
        // stores below may alias nothing we read later, but the compiler
        // cannot prove it)
        const double xo = P.x[v], lv = P.l[v], uv = P.u[v];
        const double pv = E.iter ? (E.branch ? P.pp[v] : P.pt[v]) : 0.0;
        const double cv = P.c ? P.c[v] : 0.0;
        const double go = E.iter ? P.g[v] : 0.0;
        double bv[NBX];
#pragma unroll
        for (int b = 0; b < NBX; ++b) {
            double val = 0.0;
            if (E.gram && b < 2 * nh) {
                const int bb = b < nh ? b : b - nh;
                const bool cur = E.iter && ring_slot(E.head, nh, bb, E.mh) == E.slot;
                if (!cur) val = __ldcs(E.bptr[b] + v);
            }
            bv[b] = val;
        }
        double w;
        if (P.tp) {
            int64_t i, j;
            if (small) {
                const unsigned vv = (unsigned)v, tmu = (unsigned)P.tm;
                j = vv / tmu; i = vv - (unsigned)j * tmu;
            } else {
                j = v / P.tm; i = v - j * P.tm;
            }
            const int64_t kj = P.tm + j;
            double hi = wcur[i], hj = wcur[kj];
            if (iter) { hi = fma(alpha, P.tap[i], hi); hj = fma(alpha, P.tap[kj], hj); }
            w = (rho * hi + P.tlam[i]) + (rho * hj + P.tlam[kj]);
        } else {
            w = wcur[v];
            if (iter) {
                w = fma(alpha, P.q[v], w);                      // carried w' = Q~ x'
                wnext[v] = w;
            }
        }
        // ---- epilogue (the arithmetic of epi_core, on the preloaded values)
        const double xn = E.iter ? clipd(fma(E.alpha, pv, xo), lv, uv) : xo;   // Alg. 1 line 7
        double gn = w;
        if (P.c) gn = gn + cv;
        gn = gn + P.delta * xn;
        if (P.ent != 0.0) gn = gn + P.ent * (log(xn) + 1.0);
        for (int k = 0; k < E.ncons; ++k) gn = gn + C->ccoef[k] * P.Ecol[k][v];
        double sv = 0.0, yv = 0.0;
        if (E.iter) {
            const int64_t so = (int64_t)E.slot * n + v;
            sv = xn - xo;                                       // s^k
            yv = gn - go;                                       // y^k
            P.S[so] = sv;
            P.Y[so] = yv;
        }
        P.x[v] = xn;
        P.g[v] = gn;
        const bool fixed = (xn <= lv + P.eps && gn >= 0.0) || (xn >= uv - P.eps && gn <= 0.0);
        P.mask[v] = fixed ? 0 : 1;                              // S^{k+1}, Eq. (1)
        if (!fixed) {
            const double ag = fabs(gn);
            gmax = ag > gmax ? ag : gmax;
            cnt += 1.0;
        }
        if (!E.gram) continue;
#pragma unroll
        for (int b = 0; b < NBX; ++b) {
            if (b < 2 * nh) {
                const int bb = b < nh ? b : b - nh;
                const bool cur = E.iter && ring_slot(E.head, nh, bb, E.mh) == E.slot;
                if (cur) bv[b] = b < nh ? sv : yv;
            } else if (b == 2 * nh) {
                bv[b] = gn;
            }
        }
        int idx = 0;
#pragma unroll
        for (int a = 0; a < NBX; ++a) {
            const double ma = fixed ? 0.0 : bv[a];
#pragma unroll
            for (int b = a; b < NBX; ++b) {
                acc[idx] = fma(ma, bv[b], acc[idx]);
                ++idx;
            }
        }
#pragma unroll
        for (int b = 0; b < NBX; ++b) acc[NE + b] = fma(bv[b], bv[b], acc[NE + b]);
    }
    if (!E.gram) return;
    // CTA reduction of the NA accumulators (warps in order)
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NA; ++k) {
        const double s = warp_red<0>(acc[k]);
        if (lane == 0) buf[wid * NA + k] = s;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < NA; k += NT) {
        double s = buf[k];
        for (int w = 1; w < NT / 32; ++w) s += buf[w * NA + k];
        stash[k] = s;                                           // NA <= NT
    }
    __syncthreads();
    // this CTA's partial in the runtime enumeration of gram_tail (a <= b < nb, then
    // the unmasked ||y_k||^2 when screen_full)
    const int nb = E.nb, ne = nb * (nb + 1) / 2;
    const int ntot = ne + (P.screen_full ? nh : 0);
    double* out = P.gram_part + (int64_t)blockIdx.x * GRAM_STRIDE;
    for (int e = threadIdx.x; e < ntot; e += NT) {
        int k;
        if (e < ne) {
            int aa = 0, rem = e;
            while (rem >= nb - aa) { rem -= nb - aa; ++aa; }
            const int bb = aa + rem;
            k = aa * NBX - aa * (aa - 1) / 2 + (bb - aa);
        } else {
            k = NE + nh + (e - ne);
        }
        out[e] = stash[k];
    }
    __syncthreads();
    gram_tail_after(P, C, E, gmax, cnt, red, buf, 4096, stash, Gs);
}

// ---------------------------------------------------------------- k_bwd (generic)
template <bool VEC>
__global__ void __launch_bounds__(NT, BWD_MINB) k_bwd(Prob P, int mode, const double* rvec, double* gout)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t m = P.m, ld = P.ld, ncols = P.ncols;
    const int64_t j0 = (int64_t)cta * ncols / G, j1 = (int64_t)(cta + 1) * ncols / G;
    const int64_t i0 = (int64_t)cta * m / G, i1 = (int64_t)(cta + 1) * m / G;
    const bool iter = mode == BWD_ITER;
    const int rsel = mode == BWD_PLAIN ? 0 : C->rsel;
    const double* rcur = mode == BWD_PLAIN ? rvec : P.rbuf[rsel];
    double* rnext = P.rbuf[rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;

    __shared__ double red[NT / 32 * BWD_NB];
    __shared__ double gd[BWD_NB];
    __shared__ double tile[BWD_TILE * MAXB];
    __shared__ double mk[BWD_TILE];
    __shared__ double buf[BWD_BUF];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];

    EpiCtx E;
    if (mode != BWD_PLAIN) epi_init(P, C, mode, E);
    GramEnt ent;
    const int nb = mode != BWD_PLAIN ? E.nb : 1;
    const int ne = nb * (nb + 1) / 2;
    ent.init(nb, ne, ne + (P.screen_full && mode != BWD_PLAIN ? E.nh : 0), mode != BWD_PLAIN ? E.nh : 0);
    double gacc[3] = {0.0, 0.0, 0.0};
    double gmax = 0.0, cnt = 0.0;
    const int nvg = P.split ? 2 : 1;

    for (int64_t jg = j0; jg < j1; jg += BWD_NB) {
        const int nc = (int)(j1 - jg < BWD_NB ? j1 - jg : BWD_NB);
        const bool wr = iter && jg == j0;
        double acc[BWD_NB];
#pragma unroll
        for (int c = 0; c < BWD_NB; ++c) acc[c] = 0.0;
        const double* M0 = P.M + jg * ld;
        switch (nc) {
            case 8: col_dots_glob<8, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
            case 7: col_dots_glob<7, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
            case 6: col_dots_glob<6, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
            case 5: col_dots_glob<5, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
            case 4: col_dots_glob<4, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
            case 3: col_dots_glob<3, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
            case 2: col_dots_glob<2, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
            default: col_dots_glob<1, VEC>(M0, ld, m, rcur, P.q, alpha, iter, wr, rnext, i0, i1, acc); break;
        }
        reduce8(acc, red, gd, nc);
        const int nvar = nc * nvg;
        if ((int)threadIdx.x < nvar) {
            const int jj = threadIdx.x % nc, vv = threadIdx.x / nc;
            const int64_t j = jg + jj;
            const double dot = gd[jj];
            double dval = vv ? -dot : dot;
            if (P.colscale) dval = P.colscale[j] * dot;
            if (mode == BWD_PLAIN) gout[j + vv * ncols] = dval;
            else epilogue_var(P, C, E, j + vv * ncols, dval, tile + threadIdx.x * nb, mk + threadIdx.x, gmax, cnt);
        }
        if (mode != BWD_PLAIN && E.gram) {
            __syncthreads();
            ent.accumulate(tile, mk, nvar, nb, gacc);
        }
        __syncthreads();
    }
    if (mode == BWD_PLAIN || !E.gram) return;
    gram_tail(P, C, E, ent, gacc, gmax, cnt, red, buf, BWD_BUF, stash, Gs);
}

// ---------------------------------------------------------------- k_qepi_t (TMA-staged)
// Same epilogue and register Gram as k_qepi, with every per-variable input
// streamed into shared memory by cp.async.bulk: persistent CTAs walk tiles
// of QT variables; thread 0 issues one bulk copy per input vector per tile
// into a 2-stage ring (mbarrier complete_tx), so ~QT * nvec * 8 bytes per SM
// are in flight independently of the (register-heavy) consumer threads.
// The body is instantiated per history length NH = C->nh (0..5, a uniform
// switch at kernel entry): the Gram basis (S_0..S_{NH-1}, Y_0..Y_{NH-1}, g)
// and its (2NH+1)(2NH+2)/2 + 2NH+1 accumulators are compile-time, and in an
// iteration the newest pair (basis NH-1 and 2NH-1, the ring slot this
// iteration writes) comes from registers.  Staged slots: 0 x, 1 l, 2 u, 3 g,
// 4 p, 5 c, 6 w, 7 q (QP), 8 + b the b-th Gram basis vector.  The partial
// last tile (n % QT variables) is read directly from global memory.
constexpr int QT = 512;                      // variables per tile (2 per thread)
constexpr int QMH = 5;                       // largest m_hist with a k_qepi_t instance
constexpr int QV = 8 + 2 * QMH;              // staged vector slots per tile

struct QCtx {
    const double* wcur;
    double* wnext;
    double alpha, rho;
    bool small;
};

template <int NH, bool GRAM, bool ITER, bool STAGED>
__device__ __forceinline__ void qepi_elem(const Prob& P, const Ctrl* C, const EpiCtx& E, const QCtx& Q,
                                          const double* base, const double* const* vsrc, int e,
                                          int64_t v, double* acc, double& gmax, double& cnt)
{
    constexpr int NB = 2 * NH + 1, NE = NB * (NB + 1) / 2;
    auto ld = [&](int k) -> double { return STAGED ? base[k * QT + e] : vsrc[k][v]; };
    const double xo = ld(0), lv = ld(1), uv = ld(2);
    const double go = ITER ? ld(3) : 0.0;
    const double pv = ITER ? ld(4) : 0.0;
    const double cv = P.c ? ld(5) : 0.0;
    double bv[NB];
    if (GRAM) {
#pragma unroll
        for (int b = 0; b < 2 * NH; ++b)
            if (!(ITER && (b == NH - 1 || b == 2 * NH - 1))) bv[b] = ld(8 + b);
    }
    double w;
    if (P.tp) {
        int64_t i, j;
        if (Q.small) {
            const unsigned vv = (unsigned)v, tmu = (unsigned)P.tm;
            j = vv / tmu; i = vv - (unsigned)j * tmu;
        } else {
            j = v / P.tm; i = v - j * P.tm;
        }
        const int64_t kj = P.tm + j;
        double hi = Q.wcur[i], hj = Q.wcur[kj];
        if (ITER) { hi = fma(Q.alpha, P.tap[i], hi); hj = fma(Q.alpha, P.tap[kj], hj); }
        w = (Q.rho * hi + P.tlam[i]) + (Q.rho * hj + P.tlam[kj]);
    } else {
        w = ld(6);
        if (ITER) {
            w = fma(Q.alpha, ld(7), w);                         // carried w' = Q~ x'
            Q.wnext[v] = w;
        }
    }
    const double xn = ITER ? clipd(fma(Q.alpha, pv, xo), lv, uv) : xo;   // Alg. 1 line 7
    double gn = w;
    if (P.c) gn = gn + cv;
    gn = gn + P.delta * xn;
    if (P.ent != 0.0) gn = gn + P.ent * (log(xn) + 1.0);
    for (int k = 0; k < E.ncons; ++k) gn = gn + C->ccoef[k] * P.Ecol[k][v];
    double sv = 0.0, yv = 0.0;
    if (ITER) {
        const int64_t so = (int64_t)E.slot * P.n + v;
        sv = xn - xo;                                           // s^k
        yv = gn - go;                                           // y^k
        P.S[so] = sv;
        P.Y[so] = yv;
    }
    P.x[v] = xn;
    P.g[v] = gn;
    const bool fixed = (xn <= lv + P.eps && gn >= 0.0) || (xn >= uv - P.eps && gn <= 0.0);
    P.mask[v] = fixed ? 0 : 1;                                  // S^{k+1}, Eq. (1)
    if (!fixed) {
        const double ag = fabs(gn);
        gmax = ag > gmax ? ag : gmax;
        cnt += 1.0;
    }
    if (!GRAM) return;
    if (ITER && NH > 0) { bv[NH - 1] = sv; bv[2 * NH - 1] = yv; }
    bv[2 * NH] = gn;
    int idx = 0;
#pragma unroll
    for (int a = 0; a < NB; ++a) {
        const double ma = fixed ? 0.0 : bv[a];
#pragma unroll
        for (int b = a; b < NB; ++b) {
            acc[idx] = fma(ma, bv[b], acc[idx]);
            ++idx;
        }
    }
    if (P.screen_full) {
#pragma unroll
        for (int k = 0; k < NH; ++k) acc[NE + k] = fma(bv[NH + k], bv[NH + k], acc[NE + k]);
    }
}

template <int NH, bool GRAM>
__device__ __forceinline__ void qepi_body(const Prob& P, Ctrl* C, const EpiCtx& E, const QCtx& Q,
                                          double* stg, uint64_t* full_bar, const double* const* vsrc,
                                          bool iter, double* buf, double* stash, double& gmax,
                                          double& cnt)
{
    constexpr int NB = 2 * NH + 1, NE = NB * (NB + 1) / 2, NA = NE + NH;
    double acc[NA];
#pragma unroll
    for (int k = 0; k < NA; ++k) acc[k] = 0.0;
    const int64_t n = P.n;
    const int64_t nfull = n / QT, ntiles = (n + QT - 1) / QT;
    unsigned bytes_tile = 0;
    for (int k = 0; k < QV; ++k) if (vsrc[k]) bytes_tile += QT * 8;
    auto issue = [&](int64_t t, int sidx) {                  // thread 0 only
        double* base = stg + (size_t)sidx * QV * QT;
        mbar_arrive_tx(&full_bar[sidx], bytes_tile);
        for (int k = 0; k < QV; ++k)
            if (vsrc[k]) bulk_g2s(base + (size_t)k * QT, vsrc[k] + t * QT, QT * 8, &full_bar[sidx]);
    };
    if (threadIdx.x == 0 && (int64_t)blockIdx.x < nfull) issue(blockIdx.x, 0);
    int li = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++li) {
        const int sidx = li & 1;
        const double* base = stg + (size_t)sidx * QV * QT;
        if (t < nfull) {
            const int64_t tn = t + gridDim.x;                   // prefetch the next tile
            if (threadIdx.x == 0 && tn < nfull) issue(tn, sidx ^ 1);
            mbar_wait(&full_bar[sidx], (unsigned)((li >> 1) & 1));
#pragma unroll 1
            for (int e = threadIdx.x; e < QT; e += NT) {
                const int64_t v = t * QT + e;
                if (iter) qepi_elem<NH, GRAM, true, true>(P, C, E, Q, base, vsrc, e, v, acc, gmax, cnt);
                else qepi_elem<NH, GRAM, false, true>(P, C, E, Q, base, vsrc, e, v, acc, gmax, cnt);
            }
        } else {
#pragma unroll 1
            for (int e = threadIdx.x; e < QT; e += NT) {
                const int64_t v = t * QT + e;
                if (v >= n) break;
                if (iter) qepi_elem<NH, GRAM, true, false>(P, C, E, Q, base, vsrc, e, v, acc, gmax, cnt);
                else qepi_elem<NH, GRAM, false, false>(P, C, E, Q, base, vsrc, e, v, acc, gmax, cnt);
            }
        }
        // every thread is done with this stage before it is refilled (two tiles on)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
    if (!GRAM) return;
    // CTA reduction (warps in order) and this CTA's partial in gram_tail's
    // enumeration: (a <= b < NB) row-major, then the unmasked ||y_k||^2
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NA; ++k) {
        const double s = warp_red<0>(acc[k]);
        if (lane == 0) buf[wid * NA + k] = s;
    }
    __syncthreads();
    const int ntot = NE + (P.screen_full ? NH : 0);
    double* out = P.gram_part + (int64_t)blockIdx.x * GRAM_STRIDE;
    for (int k = threadIdx.x; k < ntot; k += NT) {
        double s = buf[k];
        for (int w = 1; w < NT / 32; ++w) s += buf[w * NA + k];
        out[k] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(NT, 1) k_qepi_t(Prob P, int mode)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(128) double stg[];           // [2][QV][QT]
    __shared__ double red[NT / 32];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ double buf[4096];
    __shared__ const double* vsrc[QV];
    __shared__ __align__(8) uint64_t full_bar[2];
    const bool iter = mode == BWD_ITER;
    QCtx Q;
    Q.wcur = P.rbuf[C->rsel];
    Q.wnext = P.rbuf[C->rsel ^ 1];
    Q.alpha = iter ? C->alpha : 0.0;
    Q.rho = C->rho;
    Q.small = P.n < (1LL << 31);
    EpiCtx E;
    epi_init(P, C, mode, E);
    const int nh = E.nh;
    if (threadIdx.x == 0) {
        vsrc[0] = P.x; vsrc[1] = P.l; vsrc[2] = P.u;
        vsrc[3] = iter ? P.g : nullptr;
        vsrc[4] = iter ? (E.branch ? P.pp : P.pt) : nullptr;
        vsrc[5] = P.c;
        vsrc[6] = P.qp ? Q.wcur : nullptr;
        vsrc[7] = (P.qp && iter) ? P.q : nullptr;
        for (int b = 0; b < 2 * QMH; ++b) {
            const bool cur = iter && (b == nh - 1 || b == 2 * nh - 1);
            vsrc[8 + b] = (E.gram && b < 2 * nh && !cur) ? E.bptr[b] : nullptr;
        }
        mbar_init(&full_bar[0], 1);
        mbar_init(&full_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (P.tp && iter) {                                         // carried h' = h + alpha A p (N2)
        const int64_t K = P.tm + P.tn;
        for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < K; k += (int64_t)gridDim.x * NT)
            Q.wnext[k] = fma(Q.alpha, P.tap[k], Q.wcur[k]);
    }
    double gmax = 0.0, cnt = 0.0;
    if (!E.gram) {
        qepi_body<0, false>(P, C, E, Q, stg, full_bar, vsrc, iter, buf, stash, gmax, cnt);
        return;
    }
    switch (nh) {
        case 0: qepi_body<0, true>(P, C, E, Q, stg, full_bar, vsrc, iter, buf, stash, gmax, cnt); break;
        case 1: qepi_body<1, true>(P, C, E, Q, stg, full_bar, vsrc, iter, buf, stash, gmax, cnt); break;
        case 2: qepi_body<2, true>(P, C, E, Q, stg, full_bar, vsrc, iter, buf, stash, gmax, cnt); break;
        case 3: qepi_body<3, true>(P, C, E, Q, stg, full_bar, vsrc, iter, buf, stash, gmax, cnt); break;
        case 4: qepi_body<4, true>(P, C, E, Q, stg, full_bar, vsrc, iter, buf, stash, gmax, cnt); break;
        default: qepi_body<5, true>(P, C, E, Q, stg, full_bar, vsrc, iter, buf, stash, gmax, cnt); break;
    }
    gram_tail_after(P, C, E, gmax, cnt, red, buf, 4096, stash, Gs);
}

// ---------------------------------------------------------------- k_qepi_d (TMA + DMMA Gram)
// The QP / transport epilogue with the masked Gram on the FP64 tensor cores.
// Tiles of QD = 256 variables (one per thread) are staged by cp.async.bulk
// into a 2-stage ring exactly as in k_qepi_t (slot stride QDP = QD + 4
// doubles: the 8 basis rows a warp reads per k-step fall on distinct bank
// groups); the epilogue writes the tile's new s, y, g and the Eq. (1) mask to
// shared memory; then each warp accumulates the Gram of its 32 variables with
// mma.sync.m8n8k4 f64 (DMMA): the basis {S_0..S_{NH-1}, Y_0..Y_{NH-1}, g} is
// padded to 16 rows (two 8-blocks), A = (mask * B)^T, B = B, and the three
// upper blocks (0,0), (0,1), (1,1) take 3 DMMA per 4 variables.  Accumulators
// are 6 doubles per lane, so two CTAs fit per SM.  The partial last tile is
// copied to the same shared layout by the threads (zero-filled beyond n).
constexpr int QD = 256;
constexpr int QDP = QD + 4;
constexpr int QDV = 8 + 2 * QMH;             // staged slots (same map as k_qepi_t)

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b)
{
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(NT, 2) k_qepi_d(Prob P, int mode)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(128) double stg[];           // [2][QDV][QDP] | new[3][QD] | mk[QD]
    __shared__ double red[NT / 32];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ double gw[NT / 32][3][64];                    // per-warp Gram blocks
    __shared__ const double* vsrc[QDV];
    __shared__ __align__(8) uint64_t full_bar[2];
    double* nw = stg + 2 * (size_t)QDV * QDP;                // new s | new y | g
    double* mkv = nw + 3 * QD;
    const bool iter = mode == BWD_ITER;
    const double* wcur = P.rbuf[C->rsel];
    double* wnext = P.rbuf[C->rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    const double rho = C->rho;
    EpiCtx E;
    epi_init(P, C, mode, E);
    const int nh = E.nh;
    const int64_t n = P.n;
    const bool gram = E.gram;
    if (threadIdx.x == 0) {
        vsrc[0] = P.x; vsrc[1] = P.l; vsrc[2] = P.u;
        vsrc[3] = iter ? P.g : nullptr;
        vsrc[4] = iter ? (E.branch ? P.pp : P.pt) : nullptr;
        vsrc[5] = P.c;
        vsrc[6] = P.qp ? wcur : nullptr;
        vsrc[7] = (P.qp && iter) ? P.q : nullptr;
        for (int b = 0; b < 2 * QMH; ++b) {
            const bool cur = iter && (b == nh - 1 || b == 2 * nh - 1);
            vsrc[8 + b] = (gram && b < 2 * nh && !cur) ? E.bptr[b] : nullptr;
        }
        mbar_init(&full_bar[0], 1);
        mbar_init(&full_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (P.tp && iter) {                                         // carried h' = h + alpha A p (N2)
        const int64_t K = P.tm + P.tn;
        for (int64_t k = (int64_t)blockIdx.x * NT + threadIdx.x; k < K; k += (int64_t)gridDim.x * NT)
            wnext[k] = fma(alpha, P.tap[k], wcur[k]);
    }
    const int64_t nfull = n / QD, ntiles = (n + QD - 1) / QD;
    unsigned bytes_tile = 0;
    for (int k = 0; k < QDV; ++k) if (vsrc[k]) bytes_tile += QD * 8;
    auto issue = [&](int64_t t, int sidx) {                  // thread 0 only
        double* base = stg + (size_t)sidx * QDV * QDP;
        mbar_arrive_tx(&full_bar[sidx], bytes_tile);
        for (int k = 0; k < QDV; ++k)
            if (vsrc[k]) bulk_g2s(base + (size_t)k * QDP, vsrc[k] + t * QD, QD * 8, &full_bar[sidx]);
    };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    // this lane's two basis rows (block 0: j0 = lane/4, block 1: j1 = 8 + lane/4)
    const int j0 = lane >> 2, j1 = 8 + (lane >> 2);
    auto src_of = [&](int j, const double* base) -> const double* {   // nullptr = padding row
        if (j >= 2 * nh + 1) return nullptr;
        if (j == 2 * nh) return nw + 2 * QD;                              // g
        if (iter && j == nh - 1) return nw;                               // newest s
        if (iter && j == 2 * nh - 1) return nw + QD;                      // newest y
        return base + (size_t)(8 + j) * QDP;
    };
    double a00 = 0.0, a01 = 0.0, b00 = 0.0, b01 = 0.0, c00 = 0.0, c01 = 0.0;  // blocks (0,0) (0,1) (1,1)
    double fullacc[QMH];
#pragma unroll
    for (int k = 0; k < QMH; ++k) fullacc[k] = 0.0;
    double gmax = 0.0, cnt = 0.0;
    const bool small = n < (1LL << 31);
    if (threadIdx.x == 0 && (int64_t)blockIdx.x < nfull) issue(blockIdx.x, 0);
    int li = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++li) {
        const int sidx = li & 1;
        double* base = stg + (size_t)sidx * QDV * QDP;
        const int e = threadIdx.x;
        const int64_t v = t * QD + e;
        if (t < nfull) {
            const int64_t tn = t + gridDim.x;
            if (threadIdx.x == 0 && tn < nfull) issue(tn, sidx ^ 1);
            mbar_wait(&full_bar[sidx], (unsigned)((li >> 1) & 1));
        } else {                                                // partial tile: threads fill the stage
            for (int k = 0; k < QDV; ++k)
                if (vsrc[k]) base[(size_t)k * QDP + e] = v < n ? vsrc[k][v] : 0.0;
            __syncthreads();
        }
        // ---- epilogue (one variable per thread)
        double sv = 0.0, yv = 0.0, gn = 0.0;
        bool fixed = true;
        if (v < n) {
            auto ld = [&](int k) -> double { return base[(size_t)k * QDP + e]; };
            const double xo = ld(0), lv = ld(1), uv = ld(2);
            const double go = iter ? ld(3) : 0.0;
            const double pv = iter ? ld(4) : 0.0;
            const double cv = P.c ? ld(5) : 0.0;
            double w;
            if (P.tp) {
                int64_t i, j;
                if (small) {
                    const unsigned vv = (unsigned)v, tmu = (unsigned)P.tm;
                    j = vv / tmu; i = vv - (unsigned)j * tmu;
                } else {
                    j = v / P.tm; i = v - j * P.tm;
                }
                const int64_t kj = P.tm + j;
                double hi = wcur[i], hj = wcur[kj];
                if (iter) { hi = fma(alpha, P.tap[i], hi); hj = fma(alpha, P.tap[kj], hj); }
                w = (rho * hi + P.tlam[i]) + (rho * hj + P.tlam[kj]);
            } else {
                w = ld(6);
                if (iter) {
                    w = fma(alpha, ld(7), w);                   // carried w' = Q~ x'
                    wnext[v] = w;
                }
            }
            const double xn = iter ? clipd(fma(alpha, pv, xo), lv, uv) : xo;   // Alg. 1 line 7
            gn = w;
            if (P.c) gn = gn + cv;
            gn = gn + P.delta * xn;
            if (P.ent != 0.0) gn = gn + P.ent * (log(xn) + 1.0);
            for (int k = 0; k < E.ncons; ++k) gn = gn + C->ccoef[k] * P.Ecol[k][v];
            if (iter) {
                const int64_t so = (int64_t)E.slot * n + v;
                sv = xn - xo;                                   // s^k
                yv = gn - go;                                   // y^k
                P.S[so] = sv;
                P.Y[so] = yv;
            }
            P.x[v] = xn;
            P.g[v] = gn;
            fixed = (xn <= lv + P.eps && gn >= 0.0) || (xn >= uv - P.eps && gn <= 0.0);
            P.mask[v] = fixed ? 0 : 1;                          // S^{k+1}, Eq. (1)
            if (!fixed) {
                const double ag = fabs(gn);
                gmax = ag > gmax ? ag : gmax;
                cnt += 1.0;
            }
            if (gram && P.screen_full) {                        // unmasked ||y_k||^2 (R3 option)
#pragma unroll
                for (int k = 0; k < QMH; ++k) {
                    if (k >= nh) break;
                    const double yk = (iter && k == nh - 1) ? yv : ld(8 + nh + k);
                    fullacc[k] = fma(yk, yk, fullacc[k]);
                }
            }
        }
        if (gram) {
            nw[e] = sv; nw[QD + e] = yv; nw[2 * QD + e] = gn;
            mkv[e] = fixed ? 0.0 : 1.0;
            __syncthreads();
            // ---- warp Gram of variables [32 wid, 32 wid + 32) on DMMA
            const double* r0 = src_of(j0, base);
            const double* r1 = src_of(j1, base);
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
                const int vv = wid * 32 + ks * 4 + (lane & 3);
                const double m = mkv[vv];
                const double x0 = r0 ? r0[vv] : 0.0, x1 = r1 ? r1[vv] : 0.0;
                const double m0 = m * x0, m1 = m * x1;
                dmma884(a00, a01, m0, x0);                      // block (0,0)
                dmma884(b00, b01, m0, x1);                      // block (0,1)
                dmma884(c00, c01, m1, x1);                      // block (1,1)
            }
        }
        // every thread is done with this stage before it is refilled (two tiles on)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
    }
    if (!gram) return;
    // ---- CTA reduction: warps' blocks in order, then the enumeration of gram_tail
    {
        const int ra = lane >> 2, cb = 2 * (lane & 3);
        gw[wid][0][ra * 8 + cb] = a00; gw[wid][0][ra * 8 + cb + 1] = a01;
        gw[wid][1][ra * 8 + cb] = b00; gw[wid][1][ra * 8 + cb + 1] = b01;
        gw[wid][2][ra * 8 + cb] = c00; gw[wid][2][ra * 8 + cb + 1] = c01;
    }
    double fr[QMH];
#pragma unroll
    for (int k = 0; k < QMH; ++k) fr[k] = P.screen_full ? block_reduce<0>(fullacc[k], red) : 0.0;
    __syncthreads();
    const int nb = E.nb, ne = nb * (nb + 1) / 2;
    const int ntot = ne + (P.screen_full ? nh : 0);
    double* out = P.gram_part + (int64_t)blockIdx.x * GRAM_STRIDE;
    for (int q = threadIdx.x; q < ntot; q += NT) {
        double sum = 0.0;
        if (q < ne) {
            int aa = 0, rem = q;
            while (rem >= nb - aa) { rem -= nb - aa; ++aa; }
            const int bb = aa + rem;                                  // aa <= bb
            const int blk = aa < 8 ? (bb < 8 ? 0 : 1) : 2;
            const int r = aa & 7, c = bb & 7;
            for (int w = 0; w < NT / 32; ++w) sum += gw[w][blk][r * 8 + c];
        } else {
            sum = fr[q - ne];
        }
        out[q] = sum;
    }
    __syncthreads();
    gram_tail_after(P, C, E, gmax, cnt, red, &gw[0][0][0], NT / 32 * 3 * 64, stash, Gs);
}

// ---------------------------------------------------------------- launch
static int g_bwd_occ = 0, g_bwdw_occ = 0;
// k_qepi (register Gram) is the QP / transport epilogue for m_hist <= 5; LBFGSB_NO_QEPI=1
// selects the shared-memory tile kernel k_qpu instead (A/B experiments)
static bool g_no_qepi = getenv("LBFGSB_NO_QEPI") != nullptr;
static bool g_no_qepi_t = getenv("LBFGSB_NO_QEPI_T") != nullptr;   // register-Gram kernel without TMA staging
static bool g_qepi_reg = getenv("LBFGSB_QEPI_REG") != nullptr;      // k_qepi_t (register Gram) instead of k_qepi_d (DMMA)
constexpr int BWD_W_MAXM = 2048;
constexpr int BWD_W_SMEM_MAX = (int)sizeof(double) * (BWD_W_MAXM + WTILE * (MAXB + 1) + (NT / 32) * WG_STRIDE + 64);
static bool g_bwd_init = false;

static void bwd_init()
{
    if (g_bwd_init) return;
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_bwd<true>, NT, 0);
    g_bwd_occ = o > 0 ? o : 1;
    cudaFuncSetAttribute(k_bwd_s, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_SMEM_MAX);
    cudaFuncSetAttribute(k_qpu, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(double) * (NT * (MAXB + 1) > 4096 ? NT * (MAXB + 1) : 4096)));
    cudaFuncSetAttribute(k_bwd_w, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_W_SMEM_MAX);
    o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_bwd_w, NT, BWD_W_SMEM_MAX);
    g_bwdw_occ = o > 0 ? o : 1;
    cudaGetLastError();
    g_bwd_init = true;
}

int bwd_ctas_per_sm() { bwd_init(); return g_bwd_occ; }

void launch_gram_decide(const Prob& P, cudaStream_t st, int bwd_mode)
{
    k_gram_decide<<<1, NT, 0, st>>>(P, bwd_mode);
}

// smem bytes k_bwd_s needs for this problem (0 = does not fit)
static size_t bwd_s_smem(const Prob& P, int G)
{
    const int64_t cmax = (P.ncols + G - 1) / G;
    const int nbmax = 2 * P.mh + 1;
    int64_t mpad = P.m + (P.m & 1);
    const int64_t need_tile = (int64_t)EPI_TILE * (nbmax + 1);
    if (mpad < need_tile) mpad = need_tile;
    if (mpad < 4096) mpad = 4096;
    const size_t bytes = sizeof(double) * (size_t)(mpad + cmax + 1);
    return bytes <= (size_t)BWD_SMEM_MAX ? bytes : 0;
}

void launch_bwd(const Prob& P, cudaStream_t st, int mode, const double* rvec, double* gout)
{
    bwd_init();
    if ((P.qp || P.tp) && mode != BWD_PLAIN && P.mh <= 5 && !g_no_qepi) {
        static int occ = 0;
        if (!occ) {
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_qepi<11>, NT, 0);
            if (occ < 1) occ = 1;
        }
        // staged (TMA) variant when every staged vector is 16-byte aligned
        bool al16 = true;
        const void* ptrs[] = {P.x, P.l, P.u, P.g, P.pp, P.pt, P.c, P.rbuf[0], P.rbuf[1], P.q, P.S, P.Y};
        for (const void* p : ptrs) al16 = al16 && ((reinterpret_cast<uintptr_t>(p) & 15u) == 0);
        al16 = al16 && (P.n % 2 == 0);                          // S / Y slot starts stay aligned
        if (al16 && !g_no_qepi_t && !g_qepi_reg && P.n >= QD && 2 * P.mh + 1 <= 16) {
            const size_t smem = sizeof(double) * (2 * (size_t)QDV * QDP + 4 * (size_t)QD);
            static bool smem_set_d = false;
            if (!smem_set_d) {
                cudaFuncSetAttribute(k_qepi_d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                smem_set_d = true;
            }
            int64_t g = (P.n + QD - 1) / QD;
            if (g > 2LL * sm_count()) g = 2LL * sm_count();
            k_qepi_d<<<(int)g, NT, smem, st>>>(P, mode);
            return;
        }
        if (al16 && !g_no_qepi_t && P.n >= QT) {
            const size_t smem = sizeof(double) * 2 * (size_t)QV * QT;
            static bool smem_set = false;
            if (!smem_set) {
                cudaFuncSetAttribute(k_qepi_t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                smem_set = true;
            }
            int64_t g = (P.n + QT - 1) / QT;
            if (g > sm_count()) g = sm_count();
            k_qepi_t<<<(int)g, NT, smem, st>>>(P, mode);
            return;
        }
        int64_t g = (P.n + NT - 1) / NT;
        const int64_t cap = (int64_t)sm_count() * occ;
        if (g > cap) g = cap;
        k_qepi<11><<<(int)g, NT, 0, st>>>(P, mode);
        return;
    }
    if ((P.qp || P.tp) && mode != BWD_PLAIN) {
        const int sms = sm_count();
        int64_t g = (P.n + NT - 1) / NT;
        if (g > 2LL * sms) g = 2LL * sms;
        const int nbmax = 2 * P.mh + 1;
        int bufn = NT * (nbmax + 1);
        if (bufn < 4096) bufn = 4096;
        k_qpu<<<(int)g, NT, sizeof(double) * (size_t)bufn, st>>>(P, mode, bufn);
        return;
    }
    const double* r = mode == BWD_PLAIN ? rvec : P.rbuf[0];
    const bool aligned = (P.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(P.M) & 15u) == 0) &&
                         (reinterpret_cast<uintptr_t>(r) & 15u) == 0 &&
                         (reinterpret_cast<uintptr_t>(P.rbuf[1]) & 15u) == 0 &&
                         (mode != BWD_ITER || (reinterpret_cast<uintptr_t>(P.q) & 15u) == 0);
    const int sms = sm_count();
    const int Gs_ = (int)(P.ncols < sms ? P.ncols : sms);
    const size_t smem = aligned ? bwd_s_smem(P, Gs_) : 0;
    if (aligned && P.m < BWD_W_MAXM) {
        int mpad = (int)(P.m + (P.m & 1));
        if (mpad < 4096 / 2) mpad = 4096 / 2;     // tail reduce buffer reuses r' space
        const int nbm = 2 * P.mh + 1;
        const int wgs = nbm * (nbm + 1) / 2 + P.mh + 1;            // Gram entries + full norms for m_hist
        const size_t sm = sizeof(double) * ((size_t)mpad + WTILE * (MAXB + 1) + (NT / 32) * (size_t)wgs);
        static size_t occ_sm = 0;
        static int occ_w = 1;
        if (sm != occ_sm) {
            int o = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_bwd_w, NT, sm);
            occ_w = o > 0 ? o : 1;
            occ_sm = sm;
        }
        // grid = sms * BWDWD_MINB CTAs (fewer only when ncols is smaller), so cpad covers
        // every CTA's column range; k_bwd_w when that many CTAs do not fit an SM
        const int Gd = (int)(P.ncols < (int64_t)sms * BWDWD_MINB ? P.ncols : (int64_t)sms * BWDWD_MINB);
        const int64_t cmax = (P.ncols + Gd - 1) / Gd;
        const int cpad = (int)(cmax + (cmax & 1));
        const size_t smd = sizeof(double) * ((size_t)mpad + cpad + (size_t)NT * (nbm + 1));
        static size_t occ_dsm = 0;
        static int occ_d = 0;
        if (BWDW_DEFER && smd <= (size_t)BWD_SMEM_MAX && smd != occ_dsm) {
            cudaFuncSetAttribute(k_bwd_wd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smd);
            int o = 0;
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_bwd_wd, NT, smd);
            occ_d = o;
            occ_dsm = smd;
        }
        if (BWDW_OVL && cmax >= 2 * MT) {                       // mini-tiles pay off from 2 per CTA (C1: k_bwd_wd)
            const int nmt_max = (cpad + MT - 1) / MT;
            const int pst = nbm * (nbm + 1) / 2 + P.mh;             // Gram entries + full norms for m_hist
            const size_t smo = sizeof(double) * ((size_t)mpad + cpad + (size_t)(NT / 32) * MT * (nbm + 1) +
                                                 (size_t)2 * nmt_max * pst) + sizeof(int) * (size_t)nmt_max;
            static size_t occ_osm = 0;
            static int occ_o = 0;
            if (smo <= (size_t)BWD_SMEM_MAX && smo != occ_osm) {
                cudaFuncSetAttribute(k_bwd_wo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smo);
                int o = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_bwd_wo, NT, smo);
                occ_o = o;
                occ_osm = smo;
            }
            if (smo == occ_osm && occ_o >= BWDWD_MINB) {
                k_bwd_wo<<<Gd, NT, smo, st>>>(P, mode, rvec, gout, mpad, cpad, pst);
                return;
            }
        }
        if (BWDW_DEFER && smd == occ_dsm && occ_d >= BWDWD_MINB) {
            k_bwd_wd<<<Gd, NT, smd, st>>>(P, mode, rvec, gout, mpad, cpad);
            return;
        }
        const int Gw = (int)(P.ncols < (int64_t)sms * occ_w ? P.ncols : (int64_t)sms * occ_w);
        k_bwd_w<<<Gw, NT, sm, st>>>(P, mode, rvec, gout, mpad, wgs);
        return;
    }
#ifndef BWD_S_ENABLE
#define BWD_S_ENABLE 1         // 0: the generic k_bwd also for 2048 <= m <= ~24K (A/B builds)
#endif
    if (BWD_S_ENABLE && smem && P.m >= 2048) {
        const int64_t cmax = (P.ncols + Gs_ - 1) / Gs_;
        const int64_t mpad = (int64_t)(smem / sizeof(double)) - cmax - 1;
        k_bwd_s<<<Gs_, NTB, smem, st>>>(P, mode, rvec, gout, mpad, (int)cmax);
        return;
    }
    if (aligned) k_bwd<true><<<P.GB, NT, 0, st>>>(P, mode, rvec, gout);
    else k_bwd<false><<<P.GB, NT, 0, st>>>(P, mode, rvec, gout);
}

}  // namespace lb
