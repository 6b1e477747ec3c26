// transport.cu -- joint probability / regularised optimal transport objective
// (PAPER.md:393-402):
//     min_P <M, P> + lam r(P)   s.t.  P 1 = u,  P^T 1 = v,  P >= 0,
// r = sum P log P (entropy) or 1/2 ||P||_F^2 (Gaussian), solved with Alg. 4
// around Alg. 1.  x = vec(P), P tm x tn column-major.
//
// One iteration = k_dir (Alg. 2 / 3, unchanged) -> k_tsum -> k_qpu (epilogue).
// k_tsum reads the direction p once and produces, in one pass,
//   * a = A p = [p 1; p^T 1] (row sums: per-chunk partials reduced by the
//     row block's last CTA; column sums: smem tile transpose + per-row-block
//     partials reduced by the column chunk's last CTA), fixed order;
//   * c^T p, x^T p, p^T p and, for the entropy, the per-element differences
//     y log y - x log x at the TT clipped trial points y = clip(x + a_t p);
//   * sum t_k a_k and sum a_k^2 with t = h + lam / rho (the AL terms);
// and the last finisher takes the Armijo decision in the difference form of
// reading R29 (the AL term of a linear equality is exactly quadratic in the
// step, so only the entropy needs per-trial sums).  The epilogue then updates
// the carried h' = h + alpha a (reading R13 for the constraint residual), and
// forms g = c + lam r'(x) + (rho h_i + lam_i) + (rho h_{tm+j} + lam_{tm+j}).
#include "impl.cuh"
#include "common.cuh"

namespace lb {

__device__ __forceinline__ double xlogx_d(double x) { return x > 0.0 ? x * log(x) : 0.0; }

// sum_{c < cnt} p[c * stride] in ascending c, 8 loads in flight (L2-resident partials)
__device__ __forceinline__ double sum_strided(const double* p, int64_t stride, int cnt)
{
    double a = 0.0;
    int c = 0;
    for (; c + 8 <= cnt; c += 8) {
        double t[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) t[q] = __ldcg(p + (int64_t)(c + q) * stride);
#pragma unroll
        for (int q = 0; q < 8; ++q) a += t[q];
    }
    for (; c < cnt; ++c) a += __ldcg(p + (int64_t)c * stride);
    return a;
}

// last of `total` arrivals where this CTA contributes `nf` arrivals
__device__ __forceinline__ bool last_of(unsigned* ticket, unsigned total, unsigned nf)
{
    __shared__ int s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ticket, nf);
        s_last = (t + nf == total) ? 1 : 0;
        if (s_last) *ticket = 0u;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// Armijo decision in the difference form (R29) for the transport objective;
// S = (c^T p, x^T p, p^T p, E_0..E_{ntr-1}) and Sta, Saa the AL sums.  The
// Gaussian case is closed form in alpha: all max_bt + 1 trials at once.  The
// entropy needs per-trial sums: ntr of them per pass (1 in the iteration's
// pass, TT in a continuation pass); a failed pass continues on the device
// (cont = 1: the graph's k_tsum(TS_CONT) runs next) or through the host
// (stall), until max_bt + 1 trials have failed (R14 fallback).
__device__ void transport_decide(const Prob& P, Ctrl* C, const double* S, double Sta, double Saa,
                                 int ntr, bool allow_cont)
{
    const double rho = C->rho;
    const double lin = S[0] + P.delta * S[1] + rho * Sta;
    const double qua = P.delta * S[2] + rho * Saa;
    double a = C->alpha0;
    const bool ent = P.ent != 0.0;
    if (!ent) ntr = P.max_bt + 1;
    int tried = 0;
    for (int t = 0; t < ntr; ++t) {
        if (t > 0) a = a * P.shrink;
        if (C->ls_tried + t > P.max_bt) break;
        ++tried;
        double dl = a * lin + 0.5 * a * a * qua;
        if (ent) dl += P.ent * S[3 + t];
        if (dl <= P.c1 * a * C->gp) {
            C->alpha = a;
            C->f = C->f + dl;
            C->f_new = C->f;
            C->n_fg += C->ls_tried;
            C->n_bt += C->ls_tried;
            accept_step(P, C, t);
            return;
        }
    }
    C->ls_tried += tried;
    if (ent && C->ls_tried <= P.max_bt) {                    // more trials remain
        C->alpha0 = a * P.shrink;
        C->ls_batch += 1;
        if (allow_cont) C->cont = 1;
        else C->stall = ST_LS_CONT;
        return;
    }
    C->n_fg += C->ls_tried;
    C->n_bt += C->ls_tried;
    if (C->fallback) { C->done = 1; C->status = S_LS_FAIL; }
    else C->stall = ST_FALLBACK;
}

__global__ void __launch_bounds__(NT) k_tsum(Prob P, int mode)
{
    Ctrl* C = P.ctrl;
    const bool setup = mode == TS_SETUP;
    if (!setup && halted(C)) return;
    if (mode == TS_CONT && !C->cont) return;                  // no device-side continuation pending
    // trials this pass: 1 in the iteration (usually accepted), TT in a continuation
    const int ntr = mode == TS_ITER ? 1 : TT;
    __shared__ double tile[TCOLS][NT + 1];
    constexpr int NPART = NT / TCOLS, PROWS = NT / NPART;     // column reduction split
    __shared__ double cpart[NPART][TCOLS];
    __shared__ double msh[NT / 32 * TNS];
    __shared__ double sums[TNS];
    __shared__ double stash[NT];
    const double* pv = setup ? P.x : (C->branch ? P.pp : P.pt);
    const int64_t tm = P.tm, tn = P.tn;
    const int rb = blockIdx.x, cb = blockIdx.y;
    const int64_t i = (int64_t)rb * NT + threadIdx.x;
    const bool rok = i < tm;
    const int64_t j0 = (int64_t)cb * TCOLS;
    const int ncol = (int)(tn - j0 < TCOLS ? tn - j0 : TCOLS);
    const bool ent = P.ent != 0.0;
    double al[TT];
    al[0] = setup ? 0.0 : C->alpha0;
#pragma unroll
    for (int t = 1; t < TT; ++t) al[t] = al[t - 1] * P.shrink;
    double acc[TNS];
#pragma unroll
    for (int k = 0; k < TNS; ++k) acc[k] = 0.0;
    double racc = 0.0;
    for (int jj = 0; jj < ncol; ++jj) {
        double pj = 0.0;
        if (rok) {
            const int64_t v = i + (j0 + jj) * tm;
            pj = pv[v];
            const double cv = P.c[v];
            if (setup) {                                        // f(x): c^T x, ||x||^2, sum x log x
                acc[0] += cv * pj;
                acc[1] += pj * pj;
                if (ent) acc[2] += xlogx_d(pj);
            } else {
                const double xv = P.x[v];
                acc[0] += cv * pj;
                acc[1] += xv * pj;
                acc[2] += pj * pj;
                if (ent) {
                    const double lv = P.l[v], uv = P.u[v];
                    const double lx = xv > 0.0 ? log(xv) : 0.0;
#pragma unroll
                    for (int t = 0; t < TT; ++t) {
                        if (t >= ntr) break;
                        // y log y - x log x = d log x + y log(y/x) (oracle armijo_delta)
                        const double y = clipd(fma(al[t], pj, xv), lv, uv), d = y - xv;
                        if (xv > 0.0 && y > 0.0) {
                            const double lr = fabs(d) < 0.5 * xv ? log1p(d / xv) : log(y / xv);
                            acc[3 + t] += d * lx + y * lr;
                        } else {
                            acc[3 + t] += xlogx_d(y) - xlogx_d(xv);
                        }
                    }
                }
            }
            racc += pj;
        }
        tile[jj][threadIdx.x] = pj;
    }
    if (rok) P.trow[(int64_t)cb * tm + i] = racc;
    __syncthreads();
    {   // column partials of this row block: thread (col, part) sums PROWS rows
        const int col = threadIdx.x % TCOLS, part = threadIdx.x / TCOLS;
        double s = 0.0;
        if (col < ncol)
            for (int k = 0; k < PROWS; ++k) s += tile[col][part * PROWS + k];
        cpart[part][col] = s;
    }
    __syncthreads();
    if ((int)threadIdx.x < ncol) {
        double s = cpart[0][threadIdx.x];
        for (int w = 1; w < NPART; ++w) s += cpart[w][threadIdx.x];
        P.tcol[(int64_t)rb * tn + j0 + threadIdx.x] = s;
    }
    block_sum_multi<TNS>(acc, msh, sums);
    if ((int)threadIdx.x < TNS) P.tsp[((int64_t)rb * P.TCB + cb) * TNS + threadIdx.x] = sums[threadIdx.x];

    const double rho = C->rho;
    const double* hcur = P.rbuf[C->rsel];
    double* buf = &tile[0][0];
    constexpr int BUFN = TCOLS * (NT + 1);
    // ---- row block finisher: a_i (or h_i at setup) and its AL partial sums
    const bool fr = last_cta(P.tticket + rb, (unsigned)P.TCB);
    if (fr) {
        double v2[2] = {0.0, 0.0};
        if (rok) {
            const double a = sum_strided(P.trow + i, tm, P.TCB);
            if (setup) {
                const double hk = a - P.te[i];
                P.rbuf[C->rsel][i] = hk;
                const double t = hk + P.tlam[i] / rho;
                v2[0] = t * t;
            } else {
                P.tap[i] = a;
                const double t = hcur[i] + P.tlam[i] / rho;
                v2[0] = t * a;
                v2[1] = a * a;
            }
        }
        double o2[2];
        block_sum_multi<2>(v2, msh, o2);
        if (threadIdx.x < 2) P.tspr[rb * 2 + threadIdx.x] = o2[threadIdx.x];
    }
    // ---- column chunk finisher
    const bool fc = last_cta(P.tticket + P.TRB + cb, (unsigned)P.TRB);
    if (fc) {
        double v2[2] = {0.0, 0.0};
        if ((int)threadIdx.x < ncol) {
            const int64_t j = j0 + threadIdx.x, k = tm + j;
            const double a = sum_strided(P.tcol + j, tn, P.TRB);
            if (setup) {
                const double hk = a - P.te[k];
                P.rbuf[C->rsel][k] = hk;
                const double t = hk + P.tlam[k] / rho;
                v2[0] = t * t;
            } else {
                P.tap[k] = a;
                const double t = hcur[k] + P.tlam[k] / rho;
                v2[0] = t * a;
                v2[1] = a * a;
            }
        }
        double o2[2];
        block_sum_multi<2>(v2, msh, o2);
        if (threadIdx.x < 2) P.tspc[cb * 2 + threadIdx.x] = o2[threadIdx.x];
    }
    const unsigned nf = (fr ? 1u : 0u) + (fc ? 1u : 0u);
    if (nf == 0) return;
    if (!last_of(P.tticket + P.TRB + P.TCB, (unsigned)(P.TRB + P.TCB), nf)) return;
    // ---- global finisher: fixed-order reductions, then f (setup) or the decision
    __shared__ double S[TNS], R2[2], Q2[2];
    reduce_parts(P.tsp, P.TRB * P.TCB, TNS, TNS, [](int) { return 0; }, buf, BUFN, stash, S);
    reduce_parts(P.tspr, P.TRB, 2, 2, [](int) { return 0; }, buf, BUFN, stash, R2);
    reduce_parts(P.tspc, P.TCB, 2, 2, [](int) { return 0; }, buf, BUFN, stash, Q2);
    if (threadIdx.x != 0) return;
    if (setup) {
        const double f0 = S[0] + 0.5 * P.delta * S[1] + P.ent * S[2];
        const double f = f0 + 0.5 * rho * (R2[0] + Q2[0]);
        C->f = f;
        C->f_base = f0;
        C->nonfinite = isfinite(f) ? 0 : 1;
        return;
    }
    if (mode == TS_CONT) C->cont = 0;                         // every CTA has read it by now
    transport_decide(P, C, S, R2[0] + Q2[0], R2[1] + Q2[1], ntr, mode == TS_ITER);
}

// AL bookkeeping on the device residual h = rbuf[rsel] (Alg. 4 line 6):
// out = ||h||_inf (the violation, R21 for equalities), then, if update,
// lam += rho h.  One CTA, fixed order.
__global__ void __launch_bounds__(1024) k_tviol(Prob P, double rho, int update, double* out)
{
    __shared__ double red[32];
    const Ctrl* C = P.ctrl;
    const double* h = P.rbuf[C->rsel];
    const int64_t K = P.tm + P.tn;
    double vmax = 0.0;
    for (int64_t k = threadIdx.x; k < K; k += blockDim.x) {
        const double hk = h[k];
        const double a = fabs(hk);
        vmax = a > vmax ? a : vmax;
        if (update) P.tlam[k] = P.tlam[k] + rho * hk;
    }
    const double v = block_reduce<1>(vmax, red);
    if (threadIdx.x == 0) *out = v;
}

void launch_tsum(const Prob& P, cudaStream_t st, int mode)
{
    k_tsum<<<dim3((unsigned)P.TRB, (unsigned)P.TCB), NT, 0, st>>>(P, mode);
}

void launch_tviol(const Prob& P, cudaStream_t st, double rho, int update, double* out_dev)
{
    k_tviol<<<1, 1024, 0, st>>>(P, rho, update, out_dev);
}

}  // namespace lb
