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
#include "common.cuh"

namespace lb {

constexpr int NTB = 512;                // threads of k_bwd_s
constexpr int BWD_SMEM_MAX = 210 * 1024;   // dynamic; + ~10 KB static <= 227 KB per CTA

// ---------------------------------------------------------------- column dots
// acc[c] += sum over this thread's rows of M[i, jg + c] * r'_i, rows
// i = 2 tid + 2 blockDim k (row pairs), two row pairs per loop trip.
template <int NC>
__device__ __forceinline__ void col_dots_smem(const double* __restrict__ M0, int64_t ld, int64_t m,
                                              const double* rs, double* acc)
{
    const int64_t step = 2 * (int64_t)blockDim.x;
    int64_t i = 2 * (int64_t)threadIdx.x;
    for (; i + step + 1 < m; i += 2 * step) {
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
    for (int64_t i = 2 * (int64_t)threadIdx.x; i < m; i += 2 * (int64_t)blockDim.x) {
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
    int nh, head, slot, mh, nb, ncons, branch;
    const double* bptr[2 * MAXH];
};

// Per-variable epilogue; writes the variable's row of the Gram tile.
__device__ __forceinline__ void epilogue_var(const Prob& P, const Ctrl* C, const EpiCtx& E, int64_t v,
                                             double dval, double* trow, double* mkv, double& gmax,
                                             double& cnt)
{
    const double xo = P.x[v], lv = P.l[v], uv = P.u[v];
    double xn = xo;
    if (E.iter) {
        const double pv = E.branch ? P.pp[v] : P.pt[v];
        xn = clipd(fma(E.alpha, pv, xo), lv, uv);               // Alg. 1 line 7
    }
    double gn = dval;
    if (P.c) gn = gn + P.c[v];
    gn = gn + P.delta * xn;
    for (int k = 0; k < E.ncons; ++k) gn = gn + C->ccoef[k] * P.Ecol[k][v];
    double sv = 0.0, yv = 0.0;
    if (E.iter) {
        const int64_t so = (int64_t)E.slot * P.n + v;
        sv = xn - xo;                                           // s^k
        yv = gn - P.g[v];                                       // y^k
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
    for (int b = 0; b < E.nh; ++b) {
        const int sl = ring_slot(E.head, E.nh, b, E.mh);
        const bool cur = E.iter && sl == E.slot;
        trow[b] = cur ? sv : E.bptr[b][v];
        trow[E.nh + b] = cur ? yv : E.bptr[E.nh + b][v];
    }
    trow[2 * E.nh] = gn;
    *mkv = fixed ? 0.0 : 1.0;
}

__device__ __forceinline__ void epi_init(const Prob& P, const Ctrl* C, int mode, EpiCtx& E)
{
    E.iter = mode == BWD_ITER;
    E.gram = mode == BWD_ITER || mode == BWD_SETUP;
    E.alpha = E.iter ? C->alpha : 0.0;
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

// Per-CTA Gram partial -> 2-level deterministic tail -> Alg. 3 (thread 0).
__device__ void gram_tail(const Prob& P, Ctrl* C, const EpiCtx& E, const double* gacc, double gmax,
                          double cnt, double* red, double* buf, int bufn, double* stash, double* Gs)
{
    const int G = gridDim.x, cta = blockIdx.x;
    const int nh = E.nh, nb = E.nb, ne = nb * (nb + 1) / 2;
    const int ntot = ne + (P.screen_full ? nh : 0);
    double* out = P.gram_part + (int64_t)cta * GRAM_STRIDE;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int e = threadIdx.x + k * (int)blockDim.x;
        if (e < ntot) out[e] = gacc[k];
    }
    const double bm = block_reduce<1>(gmax, red);
    const double bc = block_reduce<0>(cnt, red);
    if (threadIdx.x == 0) { out[ntot] = bm; out[ntot + 1] = bc; }
    const int nent = ntot + 2;
    auto sel = [ntot](int e) { return e == ntot ? 1 : 0; };
    const int grp = cta / GRP, ngrp = (G + GRP - 1) / GRP;
    const int members = G - grp * GRP < GRP ? G - grp * GRP : GRP;
    if (!last_cta(P.tickets + T_BWD_G1 + grp, members)) return;
    reduce_parts(P.gram_part + (int64_t)grp * GRP * GRAM_STRIDE, members, GRAM_STRIDE, nent, sel, buf,
                 bufn, stash, Gs);
    for (int e = threadIdx.x; e < nent; e += blockDim.x) P.gram_grp[(int64_t)grp * GRAM_STRIDE + e] = Gs[e];
    if (!last_cta(P.tickets + T_BWD_G2, ngrp)) return;
    reduce_parts(P.gram_grp, ngrp, GRAM_STRIDE, nent, sel, buf, bufn, stash, Gs);
    if (P.sharded) {                                         // sharded: local Gram pack
        for (int e = threadIdx.x; e < nent; e += blockDim.x) P.pk_loc[off_gram(P) + e] = Gs[e];
        return;
    }
    if (threadIdx.x != 0) return;
    if (E.iter) C->rsel = C->rsel ^ 1;
    recur_decide(P, C, Gs, nh, 0);
}

// Sharded: reduce the all-gathered Gram packs in rank order, then Alg. 3.
__global__ void __launch_bounds__(NT) k_gram_decide(Prob P, int mode)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    __shared__ double Gs[MAXE + MAXH + 2];
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
    if (threadIdx.x != 0) return;
    if (mode == BWD_ITER) C->rsel = C->rsel ^ 1;
    recur_decide(P, C, Gs, nh, 0);
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
    // r' once per CTA
    for (int64_t i = threadIdx.x; i < m; i += NTB) {
        double r = rcur[i];
        if (iter) {
            r = fma(alpha, P.q[i], r);                          // carried residual (R13)
            if (i >= i0 && i < i1) rnext[i] = r;
        }
        rs[i] = r;
    }
    __syncthreads();
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
    double* mk = rs + (int64_t)NTB * E.nb;
    for (int vb = 0; vb < nvar; vb += NTB) {
        const int rows = nvar - vb < NTB ? nvar - vb : NTB;
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
    if (!E.gram) return;
    gram_tail(P, C, E, gacc, gmax, cnt, red, rs, (int)(mpad < 4096 ? mpad : 4096), stash, Gs);
}

// ---------------------------------------------------------------- k_bwd_w (short columns)
// m < 2048 rows (C1, C4): a whole column is only a few KB, so a CTA-wide
// reduction per column group would dominate.  Each WARP owns WCOL columns
// at a time (lanes stride the rows, r' from shared memory), reduces with
// shuffles only, and its lanes run the epilogue; the CTA syncs once per
// round of 8 warp-groups to accumulate the Gram tile.
constexpr int WCOL = 4;
constexpr int WTILE = (NT / 32) * WCOL * 2;     // tile rows per round (split: 2 vars per column)

template <int NC>
__device__ __forceinline__ void warp_col_dots(const double* __restrict__ M0, int64_t ld, int64_t m,
                                              const double* rs, double* acc)
{
    const int lane = threadIdx.x & 31;
    int64_t i = 2 * lane;
    for (; i + 64 + 1 < m; i += 128) {
        double2 a0[NC], a1[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            a0[c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i));
            a1[c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i + 64));
        }
        const double2 r0 = *reinterpret_cast<const double2*>(rs + i);
        const double2 r1 = *reinterpret_cast<const double2*>(rs + i + 64);
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            acc[c] = fma(a0[c].x, r0.x, acc[c]);
            acc[c] = fma(a0[c].y, r0.y, acc[c]);
            acc[c] = fma(a1[c].x, r1.x, acc[c]);
            acc[c] = fma(a1[c].y, r1.y, acc[c]);
        }
    }
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

__global__ void __launch_bounds__(NT, 3) k_bwd_w(Prob P, int mode, const double* rvec, double* gout, int mpad)
{
    Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    extern __shared__ __align__(16) double smw[];
    double* rs = smw;                               // r' [mpad]
    double* tile = smw + mpad;                      // [WTILE][MAXB]
    double* mk = tile + WTILE * MAXB;               // [WTILE]
    __shared__ double red[NT / 32 * BWD_NB];
    __shared__ double stash[NT];
    __shared__ double Gs[MAXE + MAXH + 2];
    const int G = gridDim.x, cta = blockIdx.x;
    const int64_t m = P.m, ld = P.ld, ncols = P.ncols;
    const int64_t j0 = (int64_t)cta * ncols / G, j1 = (int64_t)(cta + 1) * ncols / G;
    const int64_t i0 = (int64_t)cta * m / G, i1 = (int64_t)(cta + 1) * m / G;
    const bool iter = mode == BWD_ITER;
    const int rsel = mode == BWD_PLAIN ? 0 : C->rsel;
    const double* rcur = mode == BWD_PLAIN ? rvec : P.rbuf[rsel];
    double* rnext = P.rbuf[rsel ^ 1];
    const double alpha = iter ? C->alpha : 0.0;
    for (int64_t i = threadIdx.x; i < m; i += NT) {
        double r = rcur[i];
        if (iter) {
            r = fma(alpha, P.q[i], r);                          // carried residual (R13)
            if (i >= i0 && i < i1) rnext[i] = r;
        }
        rs[i] = r;
    }
    __syncthreads();
    const bool epi = mode != BWD_PLAIN;
    EpiCtx E;
    if (epi) epi_init(P, C, mode, E);
    const int nb = epi ? E.nb : 1;
    const int ne = nb * (nb + 1) / 2;
    GramEnt ent;
    ent.init(nb, ne, ne + (epi && P.screen_full ? E.nh : 0), epi ? E.nh : 0);
    double gacc[3] = {0.0, 0.0, 0.0};
    double gmax = 0.0, cnt = 0.0;
    const int nvg = P.split ? 2 : 1;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = NT / 32;
    const int64_t ncl = j1 - j0;
    const int64_t ngroups = (ncl + WCOL - 1) / WCOL;
    const int64_t rounds = (ngroups + nw - 1) / nw;
    const int rows_per_warp = WCOL * nvg;
    for (int64_t rd = 0; rd < rounds; ++rd) {
        const int64_t grp = rd * nw + w;
        const int64_t jg = j0 + grp * WCOL;
        const int nc = jg < j1 ? (int)(j1 - jg < WCOL ? j1 - jg : WCOL) : 0;
        double acc[WCOL] = {0.0, 0.0, 0.0, 0.0};
        const double* M0 = P.M + jg * ld;
        switch (nc) {
            case 4: warp_col_dots<4>(M0, ld, m, rs, acc); break;
            case 3: warp_col_dots<3>(M0, ld, m, rs, acc); break;
            case 2: warp_col_dots<2>(M0, ld, m, rs, acc); break;
            case 1: warp_col_dots<1>(M0, ld, m, rs, acc); break;
            default: break;
        }
#pragma unroll
        for (int c = 0; c < WCOL; ++c)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
        // all lanes now hold the column dots (xor butterfly: identical in every lane)
        const int trow0 = w * rows_per_warp;
        if (lane < rows_per_warp) {
            const int t = trow0 + lane;
            if (lane < nc * nvg) {
                const int jj = lane % nc, vv = lane / nc;
                double dot = acc[0];
                if (jj == 1) dot = acc[1];
                if (jj == 2) dot = acc[2];
                if (jj == 3) dot = acc[3];
                const int64_t j = jg + jj;
                double dval = vv ? -dot : dot;
                if (P.colscale) dval = P.colscale[j] * dot;
                if (!epi) gout[j + vv * ncols] = dval;
                else epilogue_var(P, C, E, j + vv * ncols, dval, tile + (int64_t)t * nb, mk + t, gmax, cnt);
            } else if (epi) {
                for (int b = 0; b < nb; ++b) tile[(int64_t)t * nb + b] = 0.0;
                mk[t] = 0.0;
            }
        }
        if (epi && E.gram) {
            __syncthreads();
            ent.accumulate(tile, mk, nw * rows_per_warp, nb, gacc);
            __syncthreads();
        }
    }
    if (!epi || !E.gram) return;
    gram_tail(P, C, E, gacc, gmax, cnt, red, rs, mpad < 4096 ? mpad : 4096, stash, Gs);
}

// ---------------------------------------------------------------- k_bwd (generic)
template <bool VEC>
__global__ void __launch_bounds__(NT, 4) k_bwd(Prob P, int mode, const double* rvec, double* gout)
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
    gram_tail(P, C, E, gacc, gmax, cnt, red, buf, BWD_BUF, stash, Gs);
}

// ---------------------------------------------------------------- launch
static int g_bwd_occ = 0, g_bwdw_occ = 0;
constexpr int BWD_W_MAXM = 2048;
constexpr int BWD_W_SMEM_MAX = (int)sizeof(double) * (BWD_W_MAXM + WTILE * (MAXB + 1) + 64);
static bool g_bwd_init = false;

static void bwd_init()
{
    if (g_bwd_init) return;
    int o = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_bwd<true>, NT, 0);
    g_bwd_occ = o > 0 ? o : 1;
    cudaFuncSetAttribute(k_bwd_s, cudaFuncAttributeMaxDynamicSharedMemorySize, BWD_SMEM_MAX);
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
    const int64_t need_tile = (int64_t)NTB * (nbmax + 1);
    if (mpad < need_tile) mpad = need_tile;
    if (mpad < 4096) mpad = 4096;
    const size_t bytes = sizeof(double) * (size_t)(mpad + cmax + 1);
    return bytes <= (size_t)BWD_SMEM_MAX ? bytes : 0;
}

void launch_bwd(const Prob& P, cudaStream_t st, int mode, const double* rvec, double* gout)
{
    bwd_init();
    const double* r = mode == BWD_PLAIN ? rvec : P.rbuf[0];
    const bool aligned = (P.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(P.M) & 15u) == 0) &&
                         (reinterpret_cast<uintptr_t>(r) & 15u) == 0 &&
                         (reinterpret_cast<uintptr_t>(P.rbuf[1]) & 15u) == 0 &&
                         (mode != BWD_ITER || (reinterpret_cast<uintptr_t>(P.q) & 15u) == 0);
    const int sms = sm_count();
    const int Gs_ = (int)(P.ncols < sms ? P.ncols : sms);
    const size_t smem = aligned ? bwd_s_smem(P, Gs_) : 0;
    if (aligned && P.m < BWD_W_MAXM) {
        const int G = (int)(P.ncols < (int64_t)sms * g_bwdw_occ ? P.ncols : (int64_t)sms * g_bwdw_occ);
        int mpad = (int)(P.m + (P.m & 1));
        if (mpad < 4096 / 2) mpad = 4096 / 2;     // tail reduce buffer reuses r' space
        const size_t sm = sizeof(double) * ((size_t)mpad + WTILE * (MAXB + 1));
        k_bwd_w<<<G, NT, sm, st>>>(P, mode, rvec, gout, mpad);
        return;
    }
    if (smem && P.m >= 2048) {
        const int64_t cmax = (P.ncols + Gs_ - 1) / Gs_;
        const int64_t mpad = (int64_t)(smem / sizeof(double)) - cmax - 1;
        k_bwd_s<<<Gs_, NTB, smem, st>>>(P, mode, rvec, gout, mpad, (int)cmax);
        return;
    }
    if (aligned) k_bwd<true><<<P.GB, NT, 0, st>>>(P, mode, rvec, gout);
    else k_bwd<false><<<P.GB, NT, 0, st>>>(P, mode, rvec, gout);
}

}  // namespace lb
