// batch.cu -- SURVEY.md 8(f) N4 "replicas": many independent small
// least-squares problems of one shape solved at once, ONE CTA PER PROBLEM.
// Each CTA runs the whole of Alg. 1 -- Eq. (1), the
// vector-free Alg. 3 on the masked Gram, Alg. 2
// (PAPER.md:86-101), the carried-residual Armijo search (R10-R14) and the
// final refresh -- with the problem's A (m x n, column-major) resident in
// shared memory when it fits (C1: 200 x 100 = 160 KB) and every vector in
// shared memory.  The scalar decisions are the same device functions the
// large path uses (dir_decide, recur_decide, armijo_decide), on a per-CTA
// Ctrl in shared memory; all reductions are fixed-order, so every problem's
// trajectory is the one lbfgsb_solve takes on it alone, up to summation order.
#include "impl.cuh"
#include "common.cuh"

namespace lb {

constexpr int BT = 256;                      // threads per problem

struct BatchArgs {
    int64_t m, n;
    const double* M; const double* b; const double* lo; const double* up;
    double* x;
    int mh;
    double eps, c1, shrink, tol;
    int max_bt, screen_full, no_projection;
    long long max_iters;
    int a_in_smem;
    lbfgsb_result* res;                      // device, one per problem
};

__device__ __forceinline__ double bsum(double v, double* red) { return block_reduce<0>(v, red); }

__global__ void __launch_bounds__(BT) k_batch(BatchArgs B)
{
    extern __shared__ __align__(16) double sm[];
    __shared__ Ctrl Cs;
    __shared__ Prob Ps;
    __shared__ double red[BT / 32];
    __shared__ double msh[BT / 32 * KT];
    __shared__ double Ssum[KT];
    __shared__ double Gs[MAXE + MAXH + 2];
    __shared__ double res4[4];
    const int64_t m = B.m, n = B.n;
    const int k = blockIdx.x, tid = threadIdx.x;
    const int mh = B.mh;
    const double* Ag = B.M + (int64_t)k * m * n;
    const double* bg = B.b + (int64_t)k * m;
    // shared layout: [A (if resident)] x g l u d pp pt mk(n) S Y (mh x n) r q (m)
    double* p0 = sm;
    const double* A = Ag;
    if (B.a_in_smem) {
        for (int64_t i = tid; i < m * n; i += BT) p0[i] = Ag[i];
        A = p0;
        p0 += m * n;
    }
    double* x = p0; double* g = x + n; double* l = g + n; double* u = l + n; double* d = u + n;
    double* pp = d + n; double* pt = pp + n; double* mk = pt + n;
    double* S = mk + n; double* Y = S + (int64_t)mh * n; double* r = Y + (int64_t)mh * n; double* q = r + m;
    Ctrl* C = &Cs;
    if (tid == 0) {
        memset(&Ps, 0, sizeof(Prob));
        Ps.n = n; Ps.m = m; Ps.eps = B.eps; Ps.c1 = B.c1; Ps.shrink = B.shrink; Ps.max_bt = B.max_bt;
        Ps.tpp = KT;                                    // the batched kernel decides KT trials per batch
        Ps.screen_full = B.screen_full; Ps.mh = mh; Ps.no_projection = B.no_projection;
        Ps.max_iters = B.max_iters;
        memset(C, 0, sizeof(Ctrl));
        C->head = mh - 1;
        C->tol = B.tol;
        C->rho = 1.0;
        C->n_fg = 1;
    }
    for (int64_t j = tid; j < n; j += BT) {
        const double lj = B.lo ? B.lo[(int64_t)k * n + j] : -INFINITY;
        const double uj = B.up ? B.up[(int64_t)k * n + j] : INFINITY;
        l[j] = lj; u[j] = uj;
        x[j] = clipd(B.x[(int64_t)k * n + j], lj, uj);          // feasible x^0
    }
    __syncthreads();
    const Prob& P = Ps;
    const int lane = tid & 31, wid = tid >> 5;

    // r = A x - b and f (R13 / R16)
    auto residual = [&]() {
        double s = 0.0;
        for (int64_t i = tid; i < m; i += BT) {
            double a = 0.0;
            for (int64_t j = 0; j < n; ++j) a += A[i + j * m] * x[j];
            const double ri = a - bg[i];
            r[i] = ri;
            s += ri * ri;
        }
        return bsum(s, red);
    };
    // g = A^T r (warp per column, fixed lane order), Eq. (1) mask, max|g_S|, |S|
    auto gradient = [&](double* gmax_out, double* cnt_out) {
        for (int64_t j = wid; j < n; j += BT / 32) {
            double a = 0.0;
            for (int64_t i = lane; i < m; i += 32) a += A[i + j * m] * r[i];
            a = warp_red<0>(a);
            if (lane == 0) g[j] = a;
        }
        __syncthreads();
        double gm = 0.0, cnt = 0.0;
        for (int64_t j = tid; j < n; j += BT) {
            const double xj = x[j], gj = g[j];
            const bool fixed = (xj <= l[j] + P.eps && gj >= 0.0) || (xj >= u[j] - P.eps && gj <= 0.0);
            mk[j] = fixed ? 0.0 : 1.0;
            if (!fixed) { const double ag = fabs(gj); gm = ag > gm ? ag : gm; cnt += 1.0; }
        }
        *gmax_out = block_reduce<1>(gm, red);
        *cnt_out = bsum(cnt, red);
    };
    // masked Gram of the basis {s_0..s_{nh-1}, y_0..y_{nh-1}, g} (+ full ||y_i||^2), then Alg. 3
    auto gram_recur = [&](double gm, double cnt) {
        const int nh = C->nh, head = C->head, nb = 2 * nh + 1, ne = nb * (nb + 1) / 2;
        const int ntot = ne + (P.screen_full ? nh : 0);
        auto vec = [&](int bidx) -> const double* {
            if (bidx == 2 * nh) return g;
            const int i = bidx < nh ? bidx : bidx - nh;
            const int sl = ring_slot(head, nh, i, mh);
            return (bidx < nh ? S : Y) + (int64_t)sl * n;
        };
        for (int e = wid; e < ntot; e += BT / 32) {
            int a, bb;
            bool full = false;
            if (e < ne) {
                int aa = 0, rem = e;
                while (rem >= nb - aa) { rem -= nb - aa; ++aa; }
                a = aa; bb = aa + rem;
            } else {
                a = bb = nh + (e - ne); full = true;
            }
            const double* va = vec(a); const double* vb = vec(bb);
            double s = 0.0;
            for (int64_t j = lane; j < n; j += 32)
                if (full || mk[j] != 0.0) s = fma(va[j], vb[j], s);
            s = warp_red<0>(s);
            if (lane == 0) Gs[e] = s;
        }
        if (tid == 0) { Gs[ntot] = gm; Gs[ntot + 1] = cnt; }
        __syncthreads();
        if (tid == 0) recur_decide(P, C, Gs, nh, 0);
        __syncthreads();
    };

    // ---- setup
    {
        const double s = residual();
        if (tid == 0) C->f = 0.5 * s;
        __syncthreads();
        double gm, cnt;
        gradient(&gm, &cnt);
        gram_recur(gm, cnt);
    }
    long long guard = 0;
    while (!C->done && ++guard < 4 * (B.max_iters + 16)) {
        // ---- direction: d = sum_b coef_b B_b on S; Alg. 2 candidates and sums
        {
            const int nh = C->fallback ? 0 : C->nh, head = C->head;
            double spg = 0.0, spp = 0.0, stg = 0.0, amin = INFINITY;
            for (int64_t j = tid; j < n; j += BT) {
                const double xj = x[j], gj = g[j], lj = l[j], uj = u[j];
                double dj = 0.0;
                if (mk[j] != 0.0) {
                    double a = C->coef[2 * nh] * gj;
                    for (int i = 0; i < nh; ++i) {
                        const int sl = ring_slot(head, nh, i, mh);
                        a = fma(C->coef[i], S[(int64_t)sl * n + j], a);
                        a = fma(C->coef[nh + i], Y[(int64_t)sl * n + j], a);
                    }
                    dj = a;
                }
                d[j] = dj;
                const double z = clipd(xj + dj, lj, uj);        // Alg. 2 line 1
                const double ppj = z - xj;                       // line 2
                double ptj = dj;                                 // lines 6-8
                if (dj < 0.0 && xj <= lj + P.eps) ptj = 0.0;
                if (dj > 0.0 && xj >= uj - P.eps) ptj = 0.0;
                pp[j] = ppj; pt[j] = ptj;
                spg += ppj * gj; spp += ppj * ppj; stg += ptj * gj;
                double t = INFINITY;
                if (ptj < 0.0) t = (lj - xj) / ptj;
                else if (ptj > 0.0) t = (uj - xj) / ptj;
                amin = t < amin ? t : amin;
            }
            const double v3[3] = {spg, spp, stg};
            block_sum_multi<3>(v3, msh, res4);
            const double a3 = block_reduce<2>(amin, red);
            if (tid == 0) { res4[3] = a3; dir_decide(P, C, res4, 0); }
            __syncthreads();
        }
        {
            // every thread reads the flags BEFORE thread 0 may reset them (the barrier
            // between the reads and the reset keeps all warps on the same path)
            const int st = C->stall, dn = C->done;
            __syncthreads();
            if (dn) break;
            if (st == ST_FALLBACK) {
                if (tid == 0) { C->stall = 0; C->fallback = 1; C->nh = 0; C->n_fallbacks += 1; C->coef[0] = -1.0; }
                __syncthreads();
                continue;
            }
        }
        const double* pv = C->branch ? pp : pt;
        // ---- q = A p over the active columns
        for (int64_t i = tid; i < m; i += BT) {
            double a = 0.0;
            for (int64_t j = 0; j < n; ++j) {
                const double pj = pv[j];
                if (pj != 0.0) a = fma(A[i + j * m], pj, a);
            }
            q[i] = a;
        }
        __syncthreads();
        // ---- Armijo batches of KT trials on the carried residual (R13)
        for (;;) {
            double acc[KT];
            double al = C->alpha0;
#pragma unroll
            for (int t = 0; t < KT; ++t) acc[t] = 0.0;
            for (int64_t i = tid; i < m; i += BT) {
                const double ri = r[i], qi = q[i];
                double a = al;
#pragma unroll
                for (int t = 0; t < KT; ++t) {
                    if (t > 0) a = a * P.shrink;
                    const double v = fma(a, qi, ri);
                    acc[t] += v * v;
                }
            }
            block_sum_multi<KT>(acc, msh, Ssum);
            if (tid == 0) {
                double quad[KT];
                quad_values(P, C, Ssum, quad);
                armijo_decide(P, C, quad, nullptr);
            }
            __syncthreads();
            const int st = C->stall;
            __syncthreads();                                     // all reads before the reset
            if (st == ST_LS_CONT) {
                if (tid == 0) C->stall = 0;
                __syncthreads();
                continue;
            }
            break;
        }
        {
            const int st = C->stall, dn = C->done;
            __syncthreads();
            if (dn) break;
            if (st == ST_FALLBACK) {
                if (tid == 0) { C->stall = 0; C->fallback = 1; C->nh = 0; C->n_fallbacks += 1; C->coef[0] = -1.0; }
                __syncthreads();
                continue;
            }
        }
        // ---- step (Alg. 1 line 7), r' = fma(alpha, q, r), g', s, y into the ring
        {
            const double alpha = C->alpha;
            const int slot = C->slot;
            for (int64_t i = tid; i < m; i += BT) r[i] = fma(alpha, q[i], r[i]);
            for (int64_t j = tid; j < n; j += BT) {
                const double xo = x[j];
                const double xn = clipd(fma(alpha, pv[j], xo), l[j], u[j]);
                x[j] = xn;
                S[(int64_t)slot * n + j] = xn - xo;              // s^k
                Y[(int64_t)slot * n + j] = -g[j];                // y^k = g' - g (completed below)
            }
            __syncthreads();
            double gm, cnt;
            gradient(&gm, &cnt);
            for (int64_t j = tid; j < n; j += BT) Y[(int64_t)slot * n + j] += g[j];
            __syncthreads();
            gram_recur(gm, cnt);
        }
    }
    // ---- final refresh (R13): r = A x - b, f, g, KKT report
    const double s = residual();
    __syncthreads();
    double gm, cnt;
    gradient(&gm, &cnt);
    double pg = 0.0;
    for (int64_t j = tid; j < n; j += BT) {
        const double v = fabs(clipd(x[j] - g[j], l[j], u[j]) - x[j]);
        pg = v > pg ? v : pg;
        B.x[(int64_t)k * n + j] = x[j];
    }
    pg = block_reduce<1>(pg, red);
    if (tid == 0) {
        lbfgsb_result R;
        memset(&R, 0, sizeof R);
        R.f = 0.5 * s;
        R.pg_inf = pg;
        R.gfree_inf = gm;
        R.n_free = (int64_t)cnt;
        R.iters = C->k;
        R.n_fg = C->n_fg;
        R.n_backtracks = C->n_bt;
        R.n_fallbacks = C->n_fallbacks;
        R.status = C->done ? C->status : S_MAX_ITERS;
        R.last_branch = C->branch;
        B.res[k] = R;
    }
}

size_t batch_smem(int64_t m, int64_t n, int mh, bool a_in_smem)
{
    return sizeof(double) * ((a_in_smem ? (size_t)(m * n) : 0) + (size_t)n * (8 + 2 * mh) + 2 * (size_t)m);
}

int launch_batch(int32_t batch, int64_t m, int64_t n, const double* M, const double* b, const double* lo,
                 const double* up, double* x, int mh, const lbfgsb_opts& o, double tol, lbfgsb_result* res,
                 cudaStream_t st)
{
    BatchArgs A;
    A.m = m; A.n = n; A.M = M; A.b = b; A.lo = lo; A.up = up; A.x = x; A.mh = mh;
    A.eps = o.eps; A.c1 = o.c1; A.shrink = o.shrink; A.tol = tol; A.max_bt = o.max_backtracks;
    A.screen_full = o.screen_full_norm; A.no_projection = o.no_projection; A.max_iters = o.max_iters;
    A.res = res;
    const size_t cap = 200 * 1024;
    size_t smem = batch_smem(m, n, mh, true);
    A.a_in_smem = smem <= cap ? 1 : 0;
    if (!A.a_in_smem) smem = batch_smem(m, n, mh, false);
    if (smem > cap) return 1;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap);
        attr = true;
    }
    k_batch<<<batch, BT, smem, st>>>(A);
    return 0;
}

}  // namespace lb
