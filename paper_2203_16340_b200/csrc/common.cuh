// common.cuh -- device helpers shared by the kernel translation units of
// liblbfgsb (deterministic reductions, last-CTA tickets, Gram entry layout,
// the vector-free Alg. 3 recurrence and the Armijo decision).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include "impl.cuh"

namespace lb {

// ticket indices
constexpr int T_DIR = 0, T_FWD_ALL = 1, T_LS = 2, T_KKT = 3, T_BWD_G2 = 4, T_GRAM = 5, T_SEP = 6;
constexpr int T_FWD_RB = 64;            // + row block (<= 8192)
constexpr int T_BWD_G1 = 64 + 8192;     // + group (<= 8000)
constexpr int T_FWD_G = T_BWD_G1 + 8000; // + row block * FWD_MAXCG + chunk group (<= 4096)
static_assert(T_FWD_G + 4096 <= NTICKETS + TICKETS_EXTRA, "ticket space");

constexpr int BWD_BUF = 2048;           // smem doubles for the k_bwd tail reduction
constexpr int BWD_TILE = 2 * BWD_NB;    // variables per epilogue group (split: 2 per column)

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ double clipd(double v, double lo, double hi)
{
    // clip(v) = min(max(v, l), u) with the comparison order of the oracle
    if (v < lo) v = lo;
    if (v > hi) v = hi;
    return v;
}

template <int OP>
__device__ __forceinline__ double opf(double a, double b)
{
    if (OP == 0) return a + b;
    if (OP == 1) return b > a ? b : a;
    return b < a ? b : a;
}

template <int OP>
__device__ __forceinline__ double warp_red(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = opf<OP>(v, __shfl_down_sync(0xffffffffu, v, o));
    return v;   // lane 0
}

// Deterministic block reduction; result valid in thread 0.  sh: >= blockDim.x/32.
template <int OP>
__device__ __forceinline__ double block_reduce(double v, double* sh)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    v = warp_red<OP>(v);
    __syncthreads();
    if (lane == 0) sh[w] = v;
    __syncthreads();
    double r = 0.0;
    if (threadIdx.x == 0) {
        r = sh[0];
        for (int i = 1; i < (int)(blockDim.x >> 5); ++i) r = opf<OP>(r, sh[i]);
    }
    return r;
}

// N block-wide sums with a single barrier: warp shuffles, one smem stage
// (sh >= N * warps doubles), threads k < N sum the warp partials in warp
// order.  out[k] valid for all threads after the call (trailing barrier).
template <int N>
__device__ __forceinline__ void block_sum_multi(const double* v, double* sh, double* out)
{
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const double s = warp_red<0>(v[k]);
        if (lane == 0) sh[w * N + k] = s;
    }
    __syncthreads();
    if ((int)threadIdx.x < N) {
        double s = sh[threadIdx.x];
        for (int i = 1; i < nw; ++i) s += sh[i * N + threadIdx.x];
        out[threadIdx.x] = s;
    }
    __syncthreads();
}

__device__ __forceinline__ bool halted(const Ctrl* C) { return (C->done | C->stall) != 0; }

// ---- P2P exchange: the fused "collective" half of a
// producing kernel's tail.  Every thread of the calling CTA takes part:
// this rank's pack section pk_loc[off .. off + cnt) is stored into slot
// [rank_id] of section `sec` of EVERY rank's mailbox (peer memory over
// NVLink, or own memory), then one system-scope release per peer bumps that
// peer's section counter.  The consuming kernel on the peer waits for the count
// in its prologue (p2p_wait_take / p2p_wait_for below).
__device__ __forceinline__ void p2p_signal(const Prob& P, int sec)
{
    for (int r = 0; r < P.nranks; ++r) {
        unsigned long long* c = reinterpret_cast<unsigned long long*>(P.peer_mb[r]) + sec;
        atomicAdd_system(c, 1ULL);
    }
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p)
{
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
// ---- LB_CHECK (debug variant builds only): device-side bounds / invariant checks that trap;
// compute-sanitizer's stand-in where it is not available.  The default library compiles none of this.
#ifdef LB_CHECK_ON
#define LB_CHECK(c) do { if (!(c)) { printf("LB_CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #c); __trap(); } } while (0)
#else
#define LB_CHECK(c) do {} while (0)
#endif

// ---- LB_TRACE (A/B variant builds only, tools/trace_phases.py): per-CTA
// phase timestamps (%globaltimer) appended as one record per CTA per launch.
// The default library compiles none of this.
#ifdef LB_TRACE
struct TraceRec { unsigned long long t[6]; int kid, cta, smid, aux; };
constexpr unsigned TRACE_CAP = 1u << 20;
static __device__ TraceRec* g_trace_buf;
static __device__ unsigned* g_trace_cnt;
__device__ __forceinline__ void trace_flush(const unsigned long long* ts, int nts, int kid, int aux)
{
    TraceRec* b = g_trace_buf;
    if (!b) return;
    const unsigned k = atomicAdd(g_trace_cnt, 1u);
    if (k >= TRACE_CAP) return;
    unsigned sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    for (int i = 0; i < 6; ++i) b[k].t[i] = i < nts ? ts[i] : 0ULL;
    b[k].kid = kid; b[k].cta = (int)(blockIdx.x + blockIdx.y * gridDim.x); b[k].smid = (int)sm; b[k].aux = aux;
}
static inline void trace_set_tu(void* buf, void* cnt)
{
    cudaMemcpyToSymbol(g_trace_buf, &buf, sizeof(void*));
    cudaMemcpyToSymbol(g_trace_cnt, &cnt, sizeof(void*));
}
// thread 0 stamps into a shared array (no per-thread registers)
#define TR_DECL __shared__ unsigned long long _trs[6]; if (threadIdx.x == 0) _trs[0] = lb::globaltimer_ns();
#define TR_MARK(i) do { if (threadIdx.x == 0) _trs[i] = lb::globaltimer_ns(); } while (0)
#define TR_FLUSH(n, kid, aux) do { if (threadIdx.x == 0) lb::trace_flush(_trs, n, kid, aux); } while (0)
#else
#define TR_DECL
#define TR_MARK(i) do {} while (0)
#define TR_FLUSH(n, kid, aux) do {} while (0)
#endif
// Consumer side (one thread): spin until section `sec` of the own mailbox has
// received `tgt` signals in total.  A peer that never signals trips the
// timeout flag in the header after 60 s instead of hanging the GPU.
__device__ __forceinline__ void p2p_wait_for(const Prob& P, int sec, unsigned long long tgt)
{
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(P.mb_hdr + sec) < tgt) {
        __nanosleep(100);
        if (globaltimer_ns() - t0 > 60000000000ULL) { atomicExch(P.mb_hdr + 4, 1ULL); break; }
    }
}
// ... and account for them (single-CTA consumers: the *_decide kernels)
__device__ __forceinline__ void p2p_wait_take(const Prob& P, int sec, unsigned long long inc)
{
    const unsigned long long tgt = P.p2p_tgt[sec] + inc;
    p2p_wait_for(P, sec, tgt);
    P.p2p_tgt[sec] = tgt;
}
__device__ __forceinline__ void p2p_push(const Prob& P, int sec, int64_t off, int64_t cnt)
{
    __syncthreads();                                    // pk_loc section written by this CTA
    for (int r = 0; r < P.nranks; ++r) {
        double* dst = P.peer_mb[r] + mb_off(P, sec) + (int64_t)P.rank_id * cnt;
        for (int64_t i = threadIdx.x; i < cnt; i += blockDim.x) dst[i] = P.pk_loc[off + i];
    }
    __syncthreads();                                    // CTA's stores ordered before thread 0's fence
    if (threadIdx.x == 0) {
        __threadfence_system();                         // one system-scope release per CTA (cumulative)
        p2p_signal(P, sec);
    }
}

// Last-CTA ticket: true in every thread of the last of `total` CTAs to arrive.
// Partials written before the call by the other CTAs are visible afterwards.
// The CTA barrier orders every thread's partial writes before thread 0's
// acq_rel ticket increment (release, cumulative over the barrier), and the
// same increment's acquire plus the second barrier orders the last CTA's
// reads of the other CTAs' partials after it: one gpu-scope fence by one
// thread instead of a sequentially consistent fence by every thread
// (LASTCTA_AR 0: the __threadfence() form, A/B).
#ifndef LASTCTA_AR
#define LASTCTA_AR 1
#endif
__device__ __forceinline__ bool last_cta(unsigned* ticket, unsigned total)
{
    __shared__ int s_last;
#if LASTCTA_AR
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned t;
        asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(t) : "l"(ticket) : "memory");
        s_last = (t == total - 1u) ? 1 : 0;
        if (s_last) *ticket = 0u;           // everyone else has arrived: reset for the next launch
    }
    __syncthreads();
#else
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned t = atomicAdd(ticket, 1u);
        s_last = (t == total - 1u) ? 1 : 0;
        if (s_last) *ticket = 0u;           // everyone else has arrived: reset for the next launch
    }
    __syncthreads();
    if (s_last) __threadfence();
#endif
    return s_last != 0;
}

// out[e] = reduction over parts p = 0..nparts-1 of src[p * stride + e], for
// e < nent, in a fixed tree order (per pass: strided sequential sums over T
// threads per entry, then a pairwise smem tree; passes combined in order).
// opsel(e): 0 sum, 1 max, 2 min.  All threads of the CTA must call; stash >= blockDim.x.
template <typename OpSel>
__device__ void reduce_parts(const double* src, int nparts, int stride, int nent, OpSel opsel,
                             double* buf, int bufn, double* stash, double* out)
{
    const int nth = (int)blockDim.x;
    int T = 1;
    while (T * 2 * nent <= nth) T *= 2;
    const int epr = nth / T;                         // entries per round
    const int per_pass = bufn / nent > 0 ? bufn / nent : 1;
    for (int p0 = 0; p0 < nparts; p0 += per_pass) {
        const int np = nparts - p0 < per_pass ? nparts - p0 : per_pass;
        const int tot = np * nent;
        // 8 independent loads in flight per thread (the L2 round trips of a
        // load-store loop would serialise: buf and src may alias for the compiler)
        for (int i0 = threadIdx.x; i0 < tot; i0 += 8 * nth) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * nth;
                if (i < tot) {
                    const int p = i / nent, e = i - p * nent;
                    v[u] = __ldcg(src + (size_t)(p0 + p) * stride + e);
                }
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * nth;
                if (i < tot) buf[i] = v[u];
            }
        }
        __syncthreads();
        for (int eb = 0; eb < nent; eb += epr) {
            const int e = eb + threadIdx.x / T, j = threadIdx.x % T;
            const int op = e < nent ? opsel(e) : 0;
            double s = op == 0 ? 0.0 : (op == 1 ? -INFINITY : INFINITY);
            if (e < nent) {
                for (int p = j; p < np; p += T) {
                    const double v = buf[p * nent + e];
                    s = op == 0 ? s + v : (op == 1 ? (v > s ? v : s) : (v < s ? v : s));
                }
            }
            stash[threadIdx.x] = s;
            __syncthreads();
            for (int h = T / 2; h > 0; h >>= 1) {
                if (e < nent && j < h) {
                    const double a = stash[threadIdx.x], b = stash[threadIdx.x + h];
                    stash[threadIdx.x] = op == 0 ? a + b : (op == 1 ? (b > a ? b : a) : (b < a ? b : a));
                }
                __syncthreads();
            }
            if (e < nent && j == 0) {
                const double v = stash[threadIdx.x];
                if (p0 == 0) out[e] = v;
                else {
                    const double a = out[e];
                    out[e] = op == 0 ? a + v : (op == 1 ? (v > a ? v : a) : (v < a ? v : a));
                }
            }
            __syncthreads();
        }
    }
}

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

// Entries of the per-CTA Gram partial.  When the entries are few (m_h small)
// R = 2..8 threads share an entry and each sums every R-th tile row (fixed
// assignment); otherwise a thread owns up to 3 entries (e = tid + k blockDim).
// finalize() combines the R partials of an entry in ascending j and writes
// the CTA's partial: deterministic either way.
struct GramEnt {
    int a[3], b[3];
    bool full[3];
    int R, j;
    __device__ void set_entry(int k, int e, int nb, int ne, int ntot, int nh)
    {
        a[k] = -1; b[k] = -1; full[k] = false;
        if (e < ne) {
            int aa = 0, rem = e;
            while (rem >= nb - aa) { rem -= nb - aa; ++aa; }
            a[k] = aa; b[k] = aa + rem;
        } else if (e < ntot) {
            a[k] = b[k] = nh + (e - ne); full[k] = true;
        }
    }
    __device__ void init(int nb, int ne, int ntot, int nh)
    {
        R = 1;
        while (R < 8 && R * 2 * ntot <= (int)blockDim.x) R *= 2;
        if (R > 1) {
            j = threadIdx.x % R;
            set_entry(0, threadIdx.x / R, nb, ne, ntot, nh);
            a[1] = a[2] = b[1] = b[2] = -1;
            full[1] = full[2] = false;
        } else {
            j = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k) set_entry(k, threadIdx.x + k * (int)blockDim.x, nb, ne, ntot, nh);
        }
    }
    // acc[k] += sum over this thread's tile rows (in row order) of mask * B_a * B_b
    __device__ void accumulate(const double* tile, const double* mk, int rows, int nb, double* acc) const
    {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (a[k] < 0) continue;
            const int aa = a[k], bb = b[k];
            double s = 0.0;
            // 8 rows per batch with every shared-memory load issued before the FMAs: the
            // conditional loads of a plain loop serialised ~3 dependent LDS per row
            // (k_bwd_wd, C4 shape: ~4.7 us per 256-row tile).  Same FMAs in the same order.
            int r = j;
            if (!full[k]) {
                for (; r + 7 * R < rows; r += 8 * R) {
                    double m8[8], a8[8], b8[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int rr = r + u * R;
                        m8[u] = mk[rr];
                        a8[u] = tile[rr * nb + aa];
                        b8[u] = tile[rr * nb + bb];
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        if (m8[u] != 0.0) s = fma(a8[u], b8[u], s);
                }
                for (; r < rows; r += R)
                    if (mk[r] != 0.0) s = fma(tile[r * nb + aa], tile[r * nb + bb], s);
            } else {
                for (; r + 7 * R < rows; r += 8 * R) {
                    double a8[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) a8[u] = tile[(r + u * R) * nb + aa];
#pragma unroll
                    for (int u = 0; u < 8; ++u) s = fma(a8[u], a8[u], s);
                }
                for (; r < rows; r += R) s = fma(tile[r * nb + aa], tile[r * nb + aa], s);
            }
            acc[k] += s;
        }
    }
    // write this CTA's partial entries out[0 .. ntot); sh: >= blockDim doubles (smem)
    __device__ void finalize(const double* acc, double* sh, double* out, int ntot) const
    {
        if (R == 1) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const int e = threadIdx.x + k * (int)blockDim.x;
                if (e < ntot) out[e] = acc[k];
            }
            return;
        }
        __syncthreads();
        sh[threadIdx.x] = a[0] >= 0 ? acc[0] : 0.0;
        __syncthreads();
        const int e = threadIdx.x / R;
        if (j == 0 && e < ntot) {
            double s = sh[threadIdx.x];
            for (int jj = 1; jj < R; ++jj) s += sh[threadIdx.x + jj];
            out[e] = s;
        }
        __syncthreads();
    }
};

// Reduced Gram (smem) -> convergence test (R15) and Alg. 3
// in vector-free form on the coefficient vector w of q = sum_b w_b B_b:
//   newest..oldest: rho_i = <s_i,y_i>_S, nu_i = ||y_i||^2_S (R3), ok_i = rho_i > eps nu_i,
//                   a_i = <s_i, q>_S / rho_i, q -= a_i y_i
//   q *= rho_{k-1}/nu_{k-1} if pair k-1 passes (R4)
//   oldest..newest: beta = <y_i, q>_S / rho_i, q += (a_i - beta) s_i
// d = -q on S (R5).  Single thread.
// tol and k are ctrl->tol and ctrl->k; the k_bwd tails pass the values they
// read at kernel entry (the tail's own loads would be dependent L2 round trips
// after the ticket's acquire invalidated L1).
__device__ __forceinline__ void recur_decide_tk(const Prob& P, Ctrl* C, const double* G, int nh, int op_mode,
                                                double tol, long long k)
{
    const int nb = 2 * nh + 1, ne = nb * (nb + 1) / 2;
    const int nfull = P.screen_full ? nh : 0;
    const double gm = G[ne + nfull], cnt = G[ne + nfull + 1];
    C->gfree = gm;
    C->nfree = (long long)cnt;
    if (!op_mode) {
        if (cnt == 0.0 || gm <= tol) { C->done = 1; C->status = S_CONVERGED; return; }
        if (k >= P.max_iters) { C->done = 1; C->status = S_MAX_ITERS; return; }
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

__device__ __forceinline__ void recur_decide(const Prob& P, Ctrl* C, const double* G, int nh, int op_mode)
{
    recur_decide_tk(P, C, G, nh, op_mode, C->tol, C->k);
}

// recur_decide_tk by one full warp (the kernel tails' last CTA): lane b holds
// the coefficient w_b (lane 0 also w_32 when nb = 33), every <B_a, q>_S is
// the lanes' products summed by a xor butterfly (commutative adds: the same
// bits in every lane), lane i keeps alpha_i, rho_i, nu_i.  One pass of the
// two loops costs ~10 shuffled dot products instead of ~10 x nb dependent
// local-memory round trips of the single-thread loops (7 us per iteration
// on B200 at m_hist = 5).  The dot products are summed in butterfly order,
// so the coefficients agree with recur_decide to rounding, not bitwise.
__device__ __forceinline__ void recur_decide_warp(const Prob& P, Ctrl* C, const double* G, int nh, int op_mode,
                                                  double tol, long long k)
{
    const int lane = threadIdx.x & 31;
    const int nb = 2 * nh + 1, ne = nb * (nb + 1) / 2;
    const int nfull = P.screen_full ? nh : 0;
    const double gm = G[ne + nfull], cnt = G[ne + nfull + 1];
    if (lane == 0) {
        C->gfree = gm;
        C->nfree = (long long)cnt;
    }
    if (!op_mode) {
        if (cnt == 0.0 || gm <= tol) {
            if (lane == 0) { C->done = 1; C->status = S_CONVERGED; }
            return;
        }
        if (k >= P.max_iters) {
            if (lane == 0) { C->done = 1; C->status = S_MAX_ITERS; }
            return;
        }
    }
    auto Gv = [&](int a, int b) { return a <= b ? G[tri(a, b, nb)] : G[tri(b, a, nb)]; };
    auto wsum = [](double v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    const int b0 = lane, b1 = lane + 32;
    double w0 = b0 == 2 * nh ? 1.0 : 0.0, w1 = b1 == 2 * nh ? 1.0 : 0.0;   // q = grad[S]
    double my_al = 0.0, my_rho = 1.0, my_nu = 1.0;
    bool my_ok = false;
    for (int i = nh - 1; i >= 0; --i) {
        const double rho = Gv(i, nh + i);
        const double nu = P.screen_full ? G[ne + i] : Gv(nh + i, nh + i);
        const bool ok = rho > P.eps * nu;
        double al = 0.0;
        if (ok) {
            double pr = b0 < nb ? w0 * Gv(i, b0) : 0.0;
            if (b1 < nb) pr = pr + w1 * Gv(i, b1);
            al = wsum(pr) / rho;                                  // <s_i, q>_S / rho_i
            if (b0 == nh + i) w0 = w0 - al;                       // q -= a_i y_i
        }
        if (lane == i) { my_al = al; my_rho = rho; my_nu = nu; my_ok = ok; }
    }
    if (nh > 0 && __shfl_sync(0xffffffffu, (int)my_ok, nh - 1)) {
        const double gam = __shfl_sync(0xffffffffu, my_rho, nh - 1) / __shfl_sync(0xffffffffu, my_nu, nh - 1);
        w0 = gam * w0;
        w1 = gam * w1;
    }
    for (int i = 0; i < nh; ++i) {
        if (!__shfl_sync(0xffffffffu, (int)my_ok, i)) continue;
        double pr = b0 < nb ? w0 * Gv(nh + i, b0) : 0.0;
        if (b1 < nb) pr = pr + w1 * Gv(nh + i, b1);
        const double beta = wsum(pr) / __shfl_sync(0xffffffffu, my_rho, i);   // <y_i, q>_S / rho_i
        const double ai = __shfl_sync(0xffffffffu, my_al, i);
        if (b0 == i) w0 = w0 + (ai - beta);                      // q += (a_i - beta) s_i
    }
    if (b0 < nb) C->coef[b0] = -w0;
    if (b1 < nb) C->coef[b1] = -w1;
}

// Alg. 2 line 3 decision (R9) and the line-search bound alpha_0 (R10).
__device__ __forceinline__ void dir_decide(const Prob& P, Ctrl* C, const double* res, int op_mode)
{
    const double eps = P.eps;
    const double Spg = res[0], Spp = res[1], Stg = res[2], amin_all = res[3];
    const int projected = (!P.no_projection && Spg <= -eps * Spp && Spp >= eps) ? 1 : 0;  // Alg. 2 line 3
    double amax = projected ? 1.0 : amin_all;
    if (amax < 0.0) amax = 0.0;
    const double gp = projected ? Spg : Stg;
    C->branch = projected;
    C->gp = gp;
    C->amax = amax;
    C->alpha0 = amax < 1.0 ? amax : 1.0;                        // R10
    C->ls_batch = 0;
    C->ls_tried = 0;
    C->cont = 0;
    if (op_mode) return;
    if (!(gp < 0.0)) {                                          // guard (R14)
        if (C->fallback) { C->done = 1; C->status = S_LS_FAIL; }
        else C->stall = ST_FALLBACK;
    }
}

// Trial objective from reduced sums (oracle order: 1/2 S + phi,
// phi = c^T x + delta/2 ||x||^2, then the AL terms of Eq. (3)).
__device__ __forceinline__ double trial_value(const Prob& P, const Ctrl* C, double quad, const double* sep,
                              double* ccoef, double* hval, double* fbase)
{
    const int ncons = P.n_eq + P.n_in;
    const double cx = sep ? sep[0] : 0.0, xx = sep ? sep[1] : 0.0;
    double phi = cx + 0.5 * P.delta * xx;
    if (fbase) *fbase = quad + phi;
    for (int k = 0; k < ncons; ++k) {
        const double hv = sep[2 + k] - C->rhs[k];
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
    return quad + phi;
}

// Quadratic part of the KT trial values of the current batch:
//   LSQ: 1/2 ||fma(alpha_t, q, r)||^2 = 1/2 S[t]          (R13, carried residual)
//   QP : 1/2 x^T w + alpha_t p^T w + 1/2 alpha_t^2 p^T q   (exact expansion of
//        1/2 (x + alpha p)^T Q~ (x + alpha p) with the carried w = Q~ x)
__device__ __forceinline__ void quad_values(const Prob& P, const Ctrl* C, const double* S, double* quad)
{
    if (P.diff) {                                               // R29: linear / quadratic coefficients
        quad[0] = P.qp ? C->qp_pw : S[0];
        quad[1] = P.qp ? C->qp_pq : S[1];
        return;
    }
    double a = C->alpha0;
    for (int t = 0; t < KT; ++t) {
        if (t > 0) a = a * P.shrink;
        quad[t] = P.qp ? 0.5 * C->qp_xw + a * C->qp_pw + 0.5 * a * a * C->qp_pq : 0.5 * S[t];
    }
}

// Armijo decision over one batch of KT trials (R10, R11, R13); single thread.
// S[t] = sum (r + alpha_t q)^2, sep[t*NSEP + s] the separable sums.
__device__ __forceinline__ void accept_step(const Prob& P, Ctrl* C, int t)
{
    C->n_fg += t + 1;
    C->n_bt += t;
    const int head = (C->head + 1) % P.mh;                      // store pair
    C->head = head;
    C->slot = head;
    C->nh = C->nh + 1 < P.mh ? C->nh + 1 : P.mh;
    C->k += 1;
    C->fallback = 0;
}

// Difference form of the Armijo test (reading R29): with L, Q the linear and
// quadratic coefficients of the smooth part along p (quad[0], quad[1]) and the
// separable sums sep = (c^T p, x^T p, E_k^T p | -, p^T p),
//   Delta(a) = a (L + c^T p + delta x^T p) + a^2/2 (Q + delta p^T p) + sum_k dphi_k(a),
// accepted when Delta(a) <= c1 a g^T p; all max_bt + 1 trials in one pass.
__device__ __forceinline__ void armijo_decide_diff(const Prob& P, Ctrl* C, const double* quad,
                                                   const double* sep)
{
    const int ncons = P.n_eq + P.n_in;
    const double cp = sep ? sep[0] : 0.0, xp = sep ? sep[1] : 0.0, pp = sep ? sep[NSEP + 1] : 0.0;
    const double lin = quad[0] + cp + P.delta * xp;
    const double qua = quad[1] + P.delta * pp;
    double a = C->alpha0;
    for (int t = 0; t <= P.max_bt; ++t) {
        if (t > 0) a = a * P.shrink;
        double dl = a * lin + 0.5 * a * a * qua;
        for (int k = 0; k < ncons; ++k) {
            const double ak = sep[2 + k];
            const double t0 = C->hval[k] + C->lam[k] / C->rho, t1 = t0 + a * ak;
            if (k < P.n_eq || (t0 > 0.0 && t1 > 0.0)) {
                dl += C->rho * a * ak * (t0 + 0.5 * a * ak);
            } else {
                const double p0 = t0 > 0.0 ? t0 : 0.0, p1 = t1 > 0.0 ? t1 : 0.0;
                dl += 0.5 * C->rho * (p1 * p1 - p0 * p0);
            }
        }
        if (dl <= P.c1 * a * C->gp) {
            C->alpha = a;
            C->f = C->f + dl;
            C->f_new = C->f;
            for (int k = 0; k < ncons; ++k) {
                const double hv = C->hval[k] + a * sep[2 + k];
                C->hval[k] = hv;
                if (k < P.n_eq) {
                    C->ccoef[k] = C->rho * hv + C->lam[k];
                } else {
                    double tt = hv + C->lam[k] / C->rho;
                    C->ccoef[k] = C->rho * (tt > 0.0 ? tt : 0.0);
                }
            }
            accept_step(P, C, t);
            return;
        }
    }
    C->n_fg += P.max_bt + 1;
    C->n_bt += P.max_bt + 1;
    if (C->fallback) { C->done = 1; C->status = S_LS_FAIL; }
    else C->stall = ST_FALLBACK;
}

__device__ __forceinline__ void armijo_decide(const Prob& P, Ctrl* C, const double* quad, const double* sep)
{
    if (P.diff) { armijo_decide_diff(P, C, quad, sep); return; }
    double cc[MAXC], hv[MAXC];
    const int ncons = P.n_eq + P.n_in;
    double a = C->alpha0;
    int tried = 0;
    const int tpp = P.tpp;                                     // trials decided per pass (<= KT)
    for (int t = 0; t < tpp; ++t) {
        if (t > 0) a = a * P.shrink;
        if (C->ls_batch * tpp + t > P.max_bt) break;
        ++tried;
        const double ft = trial_value(P, C, quad[t], sep ? sep + t * NSEP : nullptr, cc, hv, nullptr);
        if (ft <= C->f + P.c1 * a * C->gp) {                    // Armijo condition
            C->alpha = a;
            C->f_new = ft;
            C->f = ft;
            for (int k = 0; k < ncons; ++k) { C->ccoef[k] = cc[k]; C->hval[k] = hv[k]; }
            accept_step(P, C, t);
            return;
        }
    }
    C->n_fg += tried;
    C->n_bt += tried;
    if ((C->ls_batch + 1) * tpp > P.max_bt) {                   // trials exhausted
        if (C->fallback) { C->done = 1; C->status = S_LS_FAIL; }
        else C->stall = ST_FALLBACK;
    } else {
        C->alpha0 = a * P.shrink;
        C->ls_batch += 1;
        C->stall = ST_LS_CONT;
    }
}


}  // namespace lb
