// kernels.cu -- sm_100a fp64 kernels of the modified L-BFGS-B hot path
// (arXiv 2203.16340, Alg. 1-3) for the least-squares objective family.
//
// Compiled with -fmad=false: no implicit contraction, every fused
// multiply-add is an explicit fma() (reading R12), so that elementwise
// results (clip, Alg. 2 candidates, x' = clip(fma(alpha, p, x)), s, y) are
// bit-identical to the CPU oracle on identical inputs.  All reductions are
// deterministic: fixed thread->data assignment, fixed shuffle trees, partials
// summed by a single thread in block order.
//
// Citations: PAPER.md:N (paper LaTeX line), R<k>.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include "impl.cuh"

namespace lb {

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double clipd(double v, double lo, double hi)
{
    // clip(v) = min(max(v, l), u) with the comparison order of the oracle
    if (v < lo) v = lo;
    if (v > hi) v = hi;
    return v;
}

__device__ __forceinline__ double warp_sum(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    return v;   // lane 0 holds the sum
}

__device__ __forceinline__ double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_down_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

__device__ __forceinline__ double warp_min(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double w = __shfl_down_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// Deterministic block reduction; result valid in thread 0.  sh: >= NT/32.
template <int OP>  // 0 sum, 1 max, 2 min
__device__ __forceinline__ double block_reduce(double v, double* sh)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = OP == 0 ? warp_sum(v) : (OP == 1 ? warp_max(v) : warp_min(v));
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
        r = sh[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) {
            if (OP == 0) r += sh[i];
            else if (OP == 1) r = sh[i] > r ? sh[i] : r;
            else r = sh[i] < r ? sh[i] : r;
        }
    }
    return r;
}

__device__ __forceinline__ bool halted(const Ctrl* C) { return (C->done | C->stall) != 0; }

// upper-triangle index of (a, b), a <= b, in an nb x nb symmetric matrix
__host__ __device__ __forceinline__ int tri(int a, int b, int nb)
{
    return a * nb - (a * (a - 1)) / 2 + (b - a);
}

__device__ __forceinline__ int ring_slot(int head, int nh, int i, int mh)
{
    // basis index i (0 = oldest) -> physical ring slot; head = newest
    return ((head - (nh - 1) + i) % mh + mh) % mh;
}

// ------------------------------------------------------------------ clip
__global__ void k_clip(Prob P)
{
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P.n;
         j += (int64_t)gridDim.x * blockDim.x)
        P.x[j] = clipd(P.x[j], P.l[j], P.u[j]);          // feasible x^0
}

// ------------------------------------------------------------------ a4 + a5 (Gram)
// Working set Eq. (1) and the masked Gram matrix
// G_ab = sum_{j in S} B_a[j] B_b[j] of the basis B = {s_0..s_{nh-1},
// y_0..y_{nh-1}, g} (oldest pair first), from which Alg. 3 is evaluated in
// vector-free form by k_recur.  Per-CTA partials, summed in block order.
__global__ void __launch_bounds__(NT) k_gram(Prob P, int op_mode)
{
    const Ctrl* C = P.ctrl;
    if (!op_mode && halted(C)) return;
    const int nh = C->fallback ? 0 : C->nh;
    const int head = C->head, mh = P.mh;
    const int nb = 2 * nh + 1;
    const int ne = nb * (nb + 1) / 2;
    const int nfull = P.screen_full ? nh : 0;
    const int ntot = ne + nfull;
    const int64_t n = P.n;
    const double eps = P.eps;

    extern __shared__ double sm[];
    double* Bt = sm;                    // [TILE][nb]
    double* mk = sm + TILE * nb;        // [TILE]
    __shared__ double red[NT / 32];
    __shared__ const double* bptr[MAXB];
    if (threadIdx.x < nb) {
        const int b = threadIdx.x;
        const double* p;
        if (b < nh) p = P.S + (int64_t)ring_slot(head, nh, b, mh) * n;
        else if (b < 2 * nh) p = P.Y + (int64_t)ring_slot(head, nh, b - nh, mh) * n;
        else p = P.g;
        bptr[b] = p;
    }
    // entries handled by this thread (ntot <= 561 + 16 < 3 * NT)
    int ea[3], eb[3];
    bool full[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int e = threadIdx.x + k * NT;
        ea[k] = -1; eb[k] = -1; full[k] = false;
        if (e < ne) {
            int a = 0, rem = e;
            while (rem >= nb - a) { rem -= nb - a; ++a; }
            ea[k] = a; eb[k] = a + rem;
        } else if (e < ntot) {
            ea[k] = eb[k] = nh + (e - ne); full[k] = true;
        }
    }
    double acc[3] = {0.0, 0.0, 0.0};
    double gmax = 0.0, cnt = 0.0;
    __syncthreads();

    for (int64_t base = (int64_t)blockIdx.x * TILE; base < n; base += (int64_t)gridDim.x * TILE) {
        const int64_t j = base + threadIdx.x;
        double msk = 0.0;
        if (j < n) {
            const double xj = P.x[j], gj = P.g[j], lj = P.l[j], uj = P.u[j];
            const bool fixed = (xj <= lj + eps && gj >= 0.0) || (xj >= uj - eps && gj <= 0.0);
            P.mask[j] = fixed ? 0 : 1;
            if (!fixed) {
                msk = 1.0;
                const double ag = fabs(gj);
                gmax = ag > gmax ? ag : gmax;
                cnt += 1.0;
            }
            for (int b = 0; b < nb; ++b) Bt[threadIdx.x * nb + b] = bptr[b][j];
        } else {
            for (int b = 0; b < nb; ++b) Bt[threadIdx.x * nb + b] = 0.0;
        }
        mk[threadIdx.x] = msk;
        __syncthreads();
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (ea[k] < 0) continue;
            const int a = ea[k], b = eb[k];
            double s = 0.0;
            if (!full[k]) {
                for (int jj = 0; jj < TILE; ++jj)
                    if (mk[jj] != 0.0) s = fma(Bt[jj * nb + a], Bt[jj * nb + b], s);
            } else {
                for (int jj = 0; jj < TILE; ++jj) s = fma(Bt[jj * nb + a], Bt[jj * nb + a], s);
            }
            acc[k] += s;
        }
        __syncthreads();
    }
    double* out = P.gram_part + (int64_t)blockIdx.x * GRAM_STRIDE;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int e = threadIdx.x + k * NT;
        if (e < ntot) out[e] = acc[k];
    }
    const double bm = block_reduce<1>(gmax, red);
    const double bc = block_reduce<0>(cnt, red);
    if (threadIdx.x == 0) {
        out[GRAM_STRIDE - 2] = bm;
        out[GRAM_STRIDE - 1] = bc;
    }
}

// ------------------------------------------------------------------ a5 + a7
// Reduce the Gram partials, test convergence (R15: ||g[S]||_inf <= tol or
// S empty) and run Alg. 3 on the
// coefficient vector w of q = sum_b w_b B_b:
//   newest..oldest: rho_i = <s_i,y_i>_S, nu_i = ||y_i||^2_S (R3), ok_i = rho_i > eps nu_i,
//                   a_i = <s_i, q>_S / rho_i, q -= a_i y_i
//   q *= rho_{k-1}/nu_{k-1} if pair k-1 passes (R4)
//   oldest..newest: beta = <y_i, q>_S / rho_i, q += (a_i - beta) s_i
// and d = -q on S (R5).  Inner products of q are sum_b w_b G(., b).
__global__ void __launch_bounds__(NT) k_recur(Prob P, int op_mode)
{
    Ctrl* C = P.ctrl;
    if (!op_mode && halted(C)) return;
    const int nh = C->fallback ? 0 : C->nh;
    const int nb = 2 * nh + 1;
    const int ne = nb * (nb + 1) / 2;
    const int nfull = P.screen_full ? nh : 0;
    __shared__ double G[MAXE + MAXH];
    for (int e = threadIdx.x; e < ne + nfull; e += NT) {
        double s = 0.0;
        for (int b = 0; b < P.G1; ++b) s += P.gram_part[(int64_t)b * GRAM_STRIDE + e];
        G[e] = s;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    double gm = 0.0, cnt = 0.0;
    for (int b = 0; b < P.G1; ++b) {
        const double v = P.gram_part[(int64_t)b * GRAM_STRIDE + GRAM_STRIDE - 2];
        gm = v > gm ? v : gm;
        cnt += P.gram_part[(int64_t)b * GRAM_STRIDE + GRAM_STRIDE - 1];
    }
    C->gfree = gm;
    C->nfree = (long long)cnt;
    if (!op_mode) {
        if (cnt == 0.0 || gm <= C->tol) { C->done = 1; C->status = S_CONVERGED; return; }
        if (C->k >= P.max_iters) { C->done = 1; C->status = S_MAX_ITERS; return; }
    }
    double w[MAXB], al[MAXH], rho[MAXH], nu[MAXH];
    bool ok[MAXH];
    for (int b = 0; b < nb; ++b) w[b] = 0.0;
    w[2 * nh] = 1.0;                                             // q = grad[S]
    auto Gv = [&](int a, int b) { return a <= b ? G[tri(a, b, nb)] : G[tri(b, a, nb)]; };
    for (int i = nh - 1; i >= 0; --i) {
        rho[i] = Gv(i, nh + i);
        nu[i] = P.screen_full ? G[ne + i] : Gv(nh + i, nh + i);
        ok[i] = rho[i] > P.eps * nu[i];
        al[i] = 0.0;
        if (ok[i]) {
            double t = 0.0;
            for (int b = 0; b < nb; ++b) t += w[b] * Gv(i, b);     // <s_i, q>_S
            al[i] = t / rho[i];
            w[nh + i] = w[nh + i] - al[i];                       // q -= a_i y_i
        }
    }
    if (nh > 0 && ok[nh - 1]) {
        const double gam = rho[nh - 1] / nu[nh - 1];
        for (int b = 0; b < nb; ++b) w[b] = gam * w[b];
    }
    for (int i = 0; i < nh; ++i) {
        if (!ok[i]) continue;
        double t = 0.0;
        for (int b = 0; b < nb; ++b) t += w[b] * Gv(nh + i, b);  // <y_i, q>_S
        const double beta = t / rho[i];
        w[i] = w[i] + (al[i] - beta);                           // q += (a_i - beta) s_i
    }
    for (int b = 0; b < nb; ++b) C->coef[b] = -w[b];
}

// ------------------------------------------------------------------ a6
// d = sum_b coef_b B_b on S, 0 off S; Alg. 2:
// projected candidate pp = clip(x + d) - x, truncated candidate pt = d with
// eps-active outward components zeroed; partial sums <pp,g>, ||pp||^2,
// <pt,g> and the minimum blocking ratio of pt (R10).
__global__ void __launch_bounds__(NT) k_dir(Prob P, int op_mode)
{
    const Ctrl* C = P.ctrl;
    if (!op_mode && halted(C)) return;
    const int nh = C->fallback ? 0 : C->nh;
    const int head = C->head, mh = P.mh;
    const int64_t n = P.n;
    const double eps = P.eps;
    __shared__ double cf[MAXB];
    __shared__ const double* sp[MAXH];
    __shared__ const double* yp[MAXH];
    __shared__ double red[NT / 32];
    if (threadIdx.x < 2 * nh + 1) cf[threadIdx.x] = C->coef[threadIdx.x];
    if (threadIdx.x < nh) {
        const int s = ring_slot(head, nh, threadIdx.x, mh);
        sp[threadIdx.x] = P.S + (int64_t)s * n;
        yp[threadIdx.x] = P.Y + (int64_t)s * n;
    }
    __syncthreads();
    double spg = 0.0, spp = 0.0, stg = 0.0, amin = INFINITY;
    for (int64_t j = blockIdx.x * (int64_t)NT + threadIdx.x; j < n; j += (int64_t)gridDim.x * NT) {
        const double xj = P.x[j], gj = P.g[j], lj = P.l[j], uj = P.u[j];
        double d = 0.0;
        if (P.mask[j]) {
            double a = cf[2 * nh] * gj;
            for (int i = 0; i < nh; ++i) {
                a = fma(cf[i], sp[i][j], a);
                a = fma(cf[nh + i], yp[i][j], a);
            }
            d = a;
        }
        P.d[j] = d;
        const double z = clipd(xj + d, lj, uj);                 // Alg. 2 line 1
        const double pp = z - xj;                               // line 2
        double pt = d;                                          // lines 6-8
        if (d < 0.0 && xj <= lj + eps) pt = 0.0;
        if (d > 0.0 && xj >= uj - eps) pt = 0.0;
        P.pp[j] = pp;
        P.pt[j] = pt;
        spg += pp * gj;
        spp += pp * pp;
        stg += pt * gj;
        double t = INFINITY;
        if (pt < 0.0) t = (lj - xj) / pt;
        else if (pt > 0.0) t = (uj - xj) / pt;
        amin = t < amin ? t : amin;
    }
    const double a0 = block_reduce<0>(spg, red);
    const double a1 = block_reduce<0>(spp, red);
    const double a2 = block_reduce<0>(stg, red);
    const double a3 = block_reduce<2>(amin, red);
    if (threadIdx.x == 0) {
        double* o = P.dir_part + (int64_t)blockIdx.x * 4;
        o[0] = a0; o[1] = a1; o[2] = a2; o[3] = a3;
    }
}

// Alg. 2 line 3 decision (R9) and the line-search bound (R10).
__global__ void k_branch(Prob P, int op_mode)
{
    Ctrl* C = P.ctrl;
    if (!op_mode && halted(C)) return;
    if (threadIdx.x != 0) return;
    double spg = 0.0, spp = 0.0, stg = 0.0, amin = INFINITY;
    for (int b = 0; b < P.G1; ++b) {
        const double* o = P.dir_part + (int64_t)b * 4;
        spg += o[0]; spp += o[1]; stg += o[2];
        amin = o[3] < amin ? o[3] : amin;
    }
    const int projected = (spg <= -P.eps * spp && spp >= P.eps) ? 1 : 0;
    double amax = projected ? 1.0 : amin;
    if (amax < 0.0) amax = 0.0;
    const double gp = projected ? spg : stg;
    C->branch = projected;
    C->gp = gp;
    C->amax = amax;
    C->alpha0 = amax < 1.0 ? amax : 1.0;                        // R10
    C->ls_batch = 0;
    if (op_mode) return;
    if (!(gp < 0.0)) {                                          // guard (R14)
        if (C->fallback) { C->done = 1; C->status = S_LS_FAIL; }
        else C->stall = ST_FALLBACK;
    }
}

// ------------------------------------------------------------------ a1
// q partials: qpart[chunk][i] = sum over active columns j of the chunk, in
// ascending j, of M[i,j] * peff_j, peff = (split ? p_j - p_{ncols+j} : p_j)
// * colscale_j.  Only columns with peff != 0 are read: p[S-bar] = 0 in both
// Alg. 2 branches, so fixed variables cost no HBM traffic.
template <bool VEC>
__global__ void __launch_bounds__(NT) k_fwd(Prob P, int mode, const double* pvec)
{
    const Ctrl* C = P.ctrl;
    if (mode == FWD_ITER && halted(C)) return;
    const double* pv = mode == FWD_ITER ? (C->branch ? P.pp : P.pt) : pvec;
    const int64_t m = P.m, ncols = P.ncols, ld = P.ld;
    const int64_t row = (int64_t)blockIdx.x * FWD_ROWS + 2 * threadIdx.x;
    const int64_t c0 = (int64_t)blockIdx.y * P.fwd_chunk;
    const int64_t c1 = c0 + P.fwd_chunk < ncols ? c0 + P.fwd_chunk : ncols;
    __shared__ int lidx[FWD_SUB];
    __shared__ double lval[FWD_SUB];
    __shared__ int wcnt[NT / 32];
    __shared__ int nact_s;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const bool r0ok = row < m, r1ok = row + 1 < m;
    double acc0 = 0.0, acc1 = 0.0;

    for (int64_t sb = c0; sb < c1; sb += FWD_SUB) {
        const int64_t se = sb + FWD_SUB < c1 ? sb + FWD_SUB : c1;
        if (threadIdx.x == 0) nact_s = 0;
        __syncthreads();
        for (int rd = 0; rd < FWD_SUB; rd += NT) {
            const int64_t j = sb + rd + threadIdx.x;
            double v = 0.0;
            if (j < se) {
                v = P.split ? pv[j] - pv[ncols + j] : pv[j];
                if (P.colscale) v = P.colscale[j] * v;
            }
            const bool act = v != 0.0;
            const unsigned bal = __ballot_sync(0xffffffffu, act);
            if (lane == 0) wcnt[wid] = __popc(bal);
            __syncthreads();
            int off = nact_s;
            for (int w = 0; w < wid; ++w) off += wcnt[w];
            if (act) {
                const int pos = off + __popc(bal & ((1u << lane) - 1u));
                lidx[pos] = (int)(j - c0);
                lval[pos] = v;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int t = 0;
                for (int w = 0; w < NT / 32; ++w) t += wcnt[w];
                nact_s += t;
            }
            __syncthreads();
        }
        const int nact = nact_s;
        const double* Mc = P.M + c0 * ld + row;
        int a = 0;
        for (; a + 8 <= nact; a += 8) {
            double2 v2[8];
            double s2[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                const double* ptr = Mc + (int64_t)lidx[a + e] * ld;
                if (VEC && r1ok) {
                    v2[e] = __ldcs(reinterpret_cast<const double2*>(ptr));
                } else {
                    v2[e].x = r0ok ? __ldcs(ptr) : 0.0;
                    v2[e].y = r1ok ? __ldcs(ptr + 1) : 0.0;
                }
                s2[e] = lval[a + e];
            }
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                acc0 = fma(v2[e].x, s2[e], acc0);
                acc1 = fma(v2[e].y, s2[e], acc1);
            }
        }
        for (; a < nact; ++a) {
            const double* ptr = Mc + (int64_t)lidx[a] * ld;
            const double s = lval[a];
            double vx = 0.0, vy = 0.0;
            if (VEC && r1ok) {
                const double2 t = __ldcs(reinterpret_cast<const double2*>(ptr));
                vx = t.x; vy = t.y;
            } else {
                vx = r0ok ? __ldcs(ptr) : 0.0;
                vy = r1ok ? __ldcs(ptr + 1) : 0.0;
            }
            acc0 = fma(vx, s, acc0);
            acc1 = fma(vy, s, acc1);
        }
        __syncthreads();
    }
    double* out = P.qpart + (int64_t)blockIdx.y * m;
    if (r0ok) out[row] = acc0;
    if (r1ok) out[row + 1] = acc1;
}

// out_i = sum_cc qpart[cc][i] (chunk order) - b_i   (r = M~x - b at setup)
__global__ void k_resid(Prob P, int subtract_b, double* out)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.m;
         i += (int64_t)gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int c = 0; c < P.fwd_cc; ++c) s += P.qpart[(int64_t)c * P.m + i];
        if (subtract_b && P.b) s = s - P.b[i];
        out[i] = s;
    }
}

// ------------------------------------------------------------------ a2
// One batch of KT Armijo trials (R10, R11, R13): alpha_t = alpha0 shrink^t,
//   f_t = 1/2 ||fma(alpha_t, q, r)||^2 + phi(clip(fma(alpha_t, p, x))).
// CTAs [0, GL) reduce the m-part (and, in LS_ITER0, finish q from its
// partials); CTAs [GL, GL+GS) the separable part phi (c, delta, AL rows).
__global__ void __launch_bounds__(NT) k_ls(Prob P, int mode, const double* pvec)
{
    const Ctrl* C = P.ctrl;
    if ((mode == LS_ITER0 || mode == LS_ITER_NEXT) && halted(C)) return;
    __shared__ double red[NT / 32];
    double al[KT];
    const int ntr = mode == LS_SETUP ? 1 : KT;
    al[0] = mode == LS_SETUP ? 0.0 : C->alpha0;
#pragma unroll
    for (int t = 1; t < KT; ++t) al[t] = al[t - 1] * P.shrink;
    const double* pv = (mode == LS_ITER0 || mode == LS_ITER_NEXT)
                           ? (C->branch ? P.pp : P.pt) : pvec;

    if ((int)blockIdx.x < P.GL) {
        double acc[KT];
#pragma unroll
        for (int t = 0; t < KT; ++t) acc[t] = 0.0;
        for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < P.m;
             i += (int64_t)P.GL * NT) {
            double qi = 0.0;
            if (mode == LS_ITER0) {
                for (int c = 0; c < P.fwd_cc; ++c) qi += P.qpart[(int64_t)c * P.m + i];
                P.q[i] = qi;
            } else if (mode != LS_SETUP) {
                qi = P.q[i];
            }
            const double ri = P.r[i];
#pragma unroll
            for (int t = 0; t < KT; ++t) {
                if (t < ntr) {
                    const double v = fma(al[t], qi, ri);
                    acc[t] += v * v;
                }
            }
        }
        for (int t = 0; t < ntr; ++t) {
            const double s = block_reduce<0>(acc[t], red);
            if (threadIdx.x == 0) P.ls_part[(int64_t)blockIdx.x * KT + t] = s;
        }
        return;
    }
    // separable part
    const int sb = blockIdx.x - P.GL;
    const int ncons = P.n_eq + P.n_in;
    for (int t0 = 0; t0 < ntr; t0 += 4) {
        double a[4][NSEP];
#pragma unroll
        for (int tt = 0; tt < 4; ++tt)
#pragma unroll
            for (int s = 0; s < NSEP; ++s) a[tt][s] = 0.0;
        for (int64_t j = sb * (int64_t)NT + threadIdx.x; j < P.n; j += (int64_t)P.GS * NT) {
            const double xj = P.x[j], pj = pv[j], lj = P.l[j], uj = P.u[j];
            const double cj = P.c ? P.c[j] : 0.0;
#pragma unroll
            for (int tt = 0; tt < 4; ++tt) {
                if (t0 + tt >= ntr) break;
                const double xt = clipd(fma(al[t0 + tt], pj, xj), lj, uj);
                if (P.c) a[tt][0] += cj * xt;
                a[tt][1] += xt * xt;
                for (int k = 0; k < ncons; ++k) a[tt][2 + k] += P.Ecol[k][j] * xt;
            }
        }
        for (int tt = 0; tt < 4; ++tt) {
            if (t0 + tt >= ntr) break;
            for (int s = 0; s < 2 + ncons; ++s) {
                const double v = block_reduce<0>(a[tt][s], red);
                if (threadIdx.x == 0)
                    P.sep_part[((int64_t)sb * KT + t0 + tt) * NSEP + s] = v;
            }
        }
    }
}

// Evaluate trial t's objective from the partials (oracle order: 1/2 S + phi,
// phi = c^T x + delta/2 ||x||^2, then the AL terms of Eq. (3)).
__device__ double trial_value(const Prob& P, const Ctrl* C, int t, double* ccoef, double* hval,
                               double* fbase = nullptr)
{
    double S = 0.0;
    for (int b = 0; b < P.GL; ++b) S += P.ls_part[(int64_t)b * KT + t];
    const int ncons = P.n_eq + P.n_in;
    double sums[NSEP];
    for (int s = 0; s < NSEP; ++s) sums[s] = 0.0;
    for (int b = 0; b < P.GS; ++b)
        for (int s = 0; s < 2 + ncons; ++s) sums[s] += P.sep_part[((int64_t)b * KT + t) * NSEP + s];
    double phi = sums[0] + 0.5 * P.delta * sums[1];
    if (fbase) *fbase = 0.5 * S + phi;
    for (int k = 0; k < ncons; ++k) {
        const double hv = sums[2 + k] - C->rhs[k];
        hval[k] = hv;
        if (k < P.n_eq) {
            const double tt = hv + C->lam[k] / C->rho;
            phi += 0.5 * C->rho * tt * tt;
            ccoef[k] = C->rho * hv + C->lam[k];
        } else {
            double tt = hv + C->lam[k] / C->rho;
            if (tt < 0.0) tt = 0.0;
            phi += 0.5 * C->rho * tt * tt;
            ccoef[k] = C->rho * tt;
        }
    }
    return 0.5 * S + phi;
}

__global__ void k_ls_decide(Prob P, int mode, double* f_out, int ntr_op)
{
    Ctrl* C = P.ctrl;
    if ((mode == LS_ITER0 || mode == LS_ITER_NEXT) && halted(C)) return;
    if (threadIdx.x != 0) return;
    double cc[MAXC], hv[MAXC];
    const int ncons = P.n_eq + P.n_in;
    if (mode == LS_SETUP) {
        double fb = 0.0;
        const double f = trial_value(P, C, 0, cc, hv, &fb);
        C->f = f;
        C->f_base = fb;
        for (int k = 0; k < ncons; ++k) { C->ccoef[k] = cc[k]; C->hval[k] = hv[k]; }
        C->nonfinite = isfinite(f) ? 0 : 1;
        return;
    }
    if (mode == LS_OP) {
        for (int t = 0; t < ntr_op; ++t) f_out[t] = trial_value(P, C, t, cc, hv);
        return;
    }
    double a = C->alpha0;
    int tried = 0;
    for (int t = 0; t < KT; ++t) {
        if (t > 0) a = a * P.shrink;
        const int gidx = C->ls_batch * KT + t;
        if (gidx > P.max_bt) break;
        ++tried;
        const double ft = trial_value(P, C, t, cc, hv);
        if (ft <= C->f + P.c1 * a * C->gp) {                    // Armijo
            C->alpha = a;
            C->f_new = ft;
            C->f = ft;
            for (int k = 0; k < ncons; ++k) { C->ccoef[k] = cc[k]; C->hval[k] = hv[k]; }
            C->n_fg += t + 1;
            C->n_bt += t;
            const int head = (C->head + 1) % P.mh;              // store pair
            C->head = head;
            C->slot = head;
            C->nh = C->nh + 1 < P.mh ? C->nh + 1 : P.mh;
            C->k += 1;
            C->fallback = 0;
            return;
        }
    }
    C->n_fg += tried;
    C->n_bt += tried;
    if ((C->ls_batch + 1) * KT > P.max_bt) {                    // trials exhausted
        if (C->fallback) { C->done = 1; C->status = S_LS_FAIL; }
        else C->stall = ST_FALLBACK;
    } else {
        C->alpha0 = a * P.shrink;
        C->ls_batch += 1;
        C->stall = ST_LS_CONT;
    }
}

// r <- fma(alpha, q, r)  (carried residual, R13)
__global__ void k_rupd(Prob P)
{
    const Ctrl* C = P.ctrl;
    if (halted(C)) return;
    const double a = C->alpha;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P.m;
         i += (int64_t)gridDim.x * blockDim.x)
        P.r[i] = fma(a, P.q[i], P.r[i]);
}

// ------------------------------------------------------------------ a3
// g' = M~^T r (full pass over M) with the iteration epilogue fused per column:
// x' = clip(fma(alpha, p, x)), g' = dot + c + delta x' + sum_k ccoef_k E_k,
// s = x' - x and y = g' - g written into the ring slot.
template <bool VEC>
__global__ void __launch_bounds__(NT) k_bwd(Prob P, int mode, const double* rvec, double* gout)
{
    const Ctrl* C = P.ctrl;
    if (mode == BWD_ITER && halted(C)) return;
    const double* r = mode == BWD_PLAIN ? rvec : P.r;
    const int64_t m = P.m, ld = P.ld, ncols = P.ncols;
    const int64_t j0 = (int64_t)blockIdx.x * BWD_NB;
    const int nc = (int)(ncols - j0 < BWD_NB ? ncols - j0 : BWD_NB);
    __shared__ double red[NT / 32];
    __shared__ double dots[BWD_NB];
    double acc[BWD_NB];
#pragma unroll
    for (int c = 0; c < BWD_NB; ++c) acc[c] = 0.0;
    const double* M0 = P.M + j0 * ld;
    if (nc == BWD_NB) {
        for (int64_t i = 2 * threadIdx.x; i < m; i += 2 * NT) {
            if (VEC && i + 1 < m) {
                const double2 rr = *reinterpret_cast<const double2*>(r + i);
                double2 av[BWD_NB];
#pragma unroll
                for (int c = 0; c < BWD_NB; ++c)
                    av[c] = __ldcs(reinterpret_cast<const double2*>(M0 + c * ld + i));
#pragma unroll
                for (int c = 0; c < BWD_NB; ++c) {
                    acc[c] = fma(av[c].x, rr.x, acc[c]);
                    acc[c] = fma(av[c].y, rr.y, acc[c]);
                }
            } else {
                const double r0 = r[i];
                const double r1 = i + 1 < m ? r[i + 1] : 0.0;
#pragma unroll
                for (int c = 0; c < BWD_NB; ++c) {
                    acc[c] = fma(__ldcs(M0 + c * ld + i), r0, acc[c]);
                    if (i + 1 < m) acc[c] = fma(__ldcs(M0 + c * ld + i + 1), r1, acc[c]);
                }
            }
        }
    } else {
        for (int64_t i = 2 * threadIdx.x; i < m; i += 2 * NT) {
            const double r0 = r[i];
            const double r1 = i + 1 < m ? r[i + 1] : 0.0;
            for (int c = 0; c < nc; ++c) {
                acc[c] = fma(__ldcs(M0 + c * ld + i), r0, acc[c]);
                if (i + 1 < m) acc[c] = fma(__ldcs(M0 + c * ld + i + 1), r1, acc[c]);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < BWD_NB; ++c) {
        const double s = block_reduce<0>(acc[c], red);
        if (threadIdx.x == 0) dots[c] = s;
    }
    __syncthreads();
    if (threadIdx.x >= nc) return;
    const int64_t j = j0 + threadIdx.x;
    const double dot = dots[threadIdx.x];
    const int ncons = P.n_eq + P.n_in;
    const int nv = P.split ? 2 : 1;
    for (int vv = 0; vv < nv; ++vv) {
        const int64_t v = j + vv * ncols;
        double dval = vv ? -dot : dot;
        if (P.colscale) dval = P.colscale[j] * dot;
        if (mode == BWD_PLAIN) { gout[v] = dval; continue; }
        const double xo = P.x[v];
        double xn = xo;
        if (mode == BWD_ITER) {
            const double pv = C->branch ? P.pp[v] : P.pt[v];
            xn = clipd(fma(C->alpha, pv, xo), P.l[v], P.u[v]);   // Alg. 1 line 7
        }
        double gn = dval;
        if (P.c) gn = gn + P.c[v];
        gn = gn + P.delta * xn;
        for (int k = 0; k < ncons; ++k) gn = gn + C->ccoef[k] * P.Ecol[k][v];
        if (mode == BWD_ITER) {
            const int64_t so = (int64_t)C->slot * P.n + v;
            P.S[so] = xn - xo;                                   // s^k
            P.Y[so] = gn - P.g[v];                               // y^k
        }
        P.x[v] = xn;
        P.g[v] = gn;
    }
}

// ------------------------------------------------------------------ KKT report
__global__ void __launch_bounds__(NT) k_kkt(Prob P)
{
    __shared__ double red[NT / 32];
    double pg = 0.0, gm = 0.0, cnt = 0.0;
    for (int64_t j = blockIdx.x * (int64_t)NT + threadIdx.x; j < P.n; j += (int64_t)gridDim.x * NT) {
        const double xj = P.x[j], gj = P.g[j], lj = P.l[j], uj = P.u[j];
        const double v = fabs(clipd(xj - gj, lj, uj) - xj);
        pg = v > pg ? v : pg;
        const bool fixed = (xj <= lj + P.eps && gj >= 0.0) || (xj >= uj - P.eps && gj <= 0.0);
        if (!fixed) { cnt += 1.0; gm = fabs(gj) > gm ? fabs(gj) : gm; }
    }
    const double a = block_reduce<1>(pg, red);
    const double b = block_reduce<1>(gm, red);
    const double c = block_reduce<0>(cnt, red);
    if (threadIdx.x == 0) {
        double* o = P.kkt_part + (int64_t)blockIdx.x * 3;
        o[0] = a; o[1] = b; o[2] = c;
    }
}

__global__ void k_kkt_decide(Prob P)
{
    if (threadIdx.x != 0) return;
    double pg = 0.0, gm = 0.0, cnt = 0.0;
    for (int b = 0; b < P.G1; ++b) {
        const double* o = P.kkt_part + (int64_t)b * 3;
        pg = o[0] > pg ? o[0] : pg;
        gm = o[1] > gm ? o[1] : gm;
        cnt += o[2];
    }
    P.ctrl->pg = pg;
    P.ctrl->gfree = gm;
    P.ctrl->nfree = (long long)cnt;
}

// ------------------------------------------------------------------ op / callback helpers
__global__ void k_ring_load(Prob P, int nh, const double* S, const double* Y)
{
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < (int64_t)nh * P.n;
         t += (int64_t)gridDim.x * blockDim.x) {
        P.S[t] = S[t];
        P.Y[t] = Y[t];
    }
}

__global__ void k_cb_trial(Prob P, double alpha, double* xt)
{
    const Ctrl* C = P.ctrl;
    const double* pv = C->branch ? P.pp : P.pt;
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P.n;
         j += (int64_t)gridDim.x * blockDim.x)
        xt[j] = clipd(fma(alpha, pv[j], P.x[j]), P.l[j], P.u[j]);
}

__global__ void k_cb_commit(Prob P, const double* xt, const double* gt, int slot)
{
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < P.n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t so = (int64_t)slot * P.n + j;
        P.S[so] = xt[j] - P.x[j];
        P.Y[so] = gt[j] - P.g[j];
        P.x[j] = xt[j];
        P.g[j] = gt[j];
    }
}

// ------------------------------------------------------------------ launchers
static int g_sms = 0;
int sm_count()
{
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

static int grid_for(int64_t n, int per)
{
    int64_t g = (n + per - 1) / per;
    const int64_t cap = 4LL * sm_count();
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

static bool vec_ok(const Prob& P)
{
    return (P.ld % 2 == 0) && ((reinterpret_cast<uintptr_t>(P.M) & 15u) == 0);
}

void launch_clip(const Prob& P, cudaStream_t st) { k_clip<<<grid_for(P.n, NT), NT, 0, st>>>(P); }

static const size_t kGramSmem = sizeof(double) * (size_t)TILE * (MAXB + 1);
void init_kernels()
{
    static bool done = false;
    if (done) return;
    cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kGramSmem);
    sm_count();
    done = true;
}

void launch_gram(const Prob& P, cudaStream_t st, int op_mode)
{
    // dynamic smem sized for the maximal basis: the actual nb is read on device
    k_gram<<<P.G1, NT, kGramSmem, st>>>(P, op_mode);
}
void launch_recur(const Prob& P, cudaStream_t st, int op_mode) { k_recur<<<1, NT, 0, st>>>(P, op_mode); }
void launch_dir(const Prob& P, cudaStream_t st, int op_mode) { k_dir<<<P.G1, NT, 0, st>>>(P, op_mode); }
void launch_branch(const Prob& P, cudaStream_t st, int op_mode) { k_branch<<<1, 32, 0, st>>>(P, op_mode); }

void launch_fwd(const Prob& P, cudaStream_t st, int mode, const double* pvec)
{
    dim3 grid(P.fwd_rb, P.fwd_cc);
    if (vec_ok(P)) k_fwd<true><<<grid, NT, 0, st>>>(P, mode, pvec);
    else k_fwd<false><<<grid, NT, 0, st>>>(P, mode, pvec);
}
void launch_resid(const Prob& P, cudaStream_t st, int subtract_b, double* out)
{
    k_resid<<<grid_for(P.m, NT), NT, 0, st>>>(P, subtract_b, out);
}
void launch_ls(const Prob& P, cudaStream_t st, int mode, const double* pvec)
{
    k_ls<<<P.GL + P.GS, NT, 0, st>>>(P, mode, pvec);
}
void launch_ls_decide(const Prob& P, cudaStream_t st, int mode, double* f_out_dev, int ntr)
{
    k_ls_decide<<<1, 32, 0, st>>>(P, mode, f_out_dev, ntr);
}
void launch_rupd(const Prob& P, cudaStream_t st) { k_rupd<<<grid_for(P.m, NT), NT, 0, st>>>(P); }
void launch_bwd(const Prob& P, cudaStream_t st, int mode, const double* rvec, double* gout)
{
    const double* r = mode == BWD_PLAIN ? rvec : P.r;
    if (vec_ok(P) && (reinterpret_cast<uintptr_t>(r) & 15u) == 0) k_bwd<true><<<P.bwd_blocks, NT, 0, st>>>(P, mode, rvec, gout);
    else k_bwd<false><<<P.bwd_blocks, NT, 0, st>>>(P, mode, rvec, gout);
}
void launch_kkt(const Prob& P, cudaStream_t st)
{
    k_kkt<<<P.G1, NT, 0, st>>>(P);
    k_kkt_decide<<<1, 32, 0, st>>>(P);
}
void launch_ring_load(const Prob& P, cudaStream_t st, int nh, const double* S, const double* Y)
{
    if (nh > 0) k_ring_load<<<grid_for((int64_t)nh * P.n, NT), NT, 0, st>>>(P, nh, S, Y);
}
void launch_cb_trial(const Prob& P, cudaStream_t st, double alpha, double* xt)
{
    k_cb_trial<<<grid_for(P.n, NT), NT, 0, st>>>(P, alpha, xt);
}
void launch_cb_commit(const Prob& P, cudaStream_t st, const double* xt, const double* gt, int slot)
{
    k_cb_commit<<<grid_for(P.n, NT), NT, 0, st>>>(P, xt, gt, slot);
}

}  // namespace lb
