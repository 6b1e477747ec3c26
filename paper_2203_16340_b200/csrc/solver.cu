// solver.cu -- host control of liblbfgsb: the C ABI of include/lbfgsb.h and
// include/lbfgsb_ops.h.  Every step of the method runs in the device kernels
// of kernels.cu; the host only sequences launches, replays a CUDA graph of
// check_every iterations and reads the ~400-byte control block between
// replays.  No CPU fallback exists: without a device every call returns
// LBFGSB_ERR_CUDA.
//
// Citations: PAPER.md:N (paper LaTeX line), R<k>.
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "impl.cuh"
#include "../../include/lbfgsb_ops.h"

#ifdef LBFGSB_WITH_NCCL
#include <nccl.h>
#endif

using namespace lb;

// ------------------------------------------------------------------ errors
static thread_local std::string g_err = "no error";

static lbfgsb_err fail(lbfgsb_err e, const char* fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return e;
}

#define CK(expr)                                                                        \
    do {                                                                                \
        cudaError_t e_ = (expr);                                                        \
        if (e_ != cudaSuccess)                                                          \
            return fail(e_ == cudaErrorMemoryAllocation ? LBFGSB_ERR_OOM : LBFGSB_ERR_CUDA, \
                        "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

#define TRY(expr)                                                                       \
    do {                                                                                \
        lbfgsb_err t_ = (expr);                                                         \
        if (t_ != LBFGSB_OK) return t_;                                                 \
    } while (0)

extern "C" const char* lbfgsb_last_error(void) { return g_err.c_str(); }

#ifdef LB_TRACE
namespace lb { void trace_set_bwd(void*, void*); void trace_set_kernels(void*, void*); }
// A/B variant builds only (tools/trace_phases.py): point the per-CTA phase
// trace of k_bwd_s / k_bwd_w / k_fwd / k_dir at device buffers (NULL: off).
extern "C" int lbfgsb_trace_set(void* recs, void* count)
{
    lb::trace_set_bwd(recs, count);
    lb::trace_set_kernels(recs, count);
    return (int)cudaDeviceSynchronize();
}
#endif

// ------------------------------------------------------------------ objects
struct lbfgsb_objective {
    int kind;                       // 0 LSQ (and QP), 1 callback, 2 transport
    int64_t tm = 0, tn = 0;         // transport: P is tm x tn
    int reg = 0;                    // transport: 0 entropy, 1 Gaussian
    double lam = 0.0;               // transport: regularisation weight
    const double* M;
    int64_t m, ncols, ld;
    const double* colscale;
    int split;
    const double* b;
    const double* c;
    double delta;
    lbfgsb_fg_cb fg;
    void* user;
    int qp;                         // 1: 1/2 x^T D M D x (+ c, delta); M n x n symmetric
};

namespace {
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { release(); }
    lbfgsb_err ensure(size_t need, bool zero = false)
    {
        if (need <= bytes && p) return LBFGSB_OK;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        if (need == 0) need = 16;
        cudaError_t e = cudaMalloc(&p, need);
        // always zeroed: recycled device memory must not leak a previous handle's state
        (void)zero;
        if (e == cudaSuccess) e = cudaMemset(p, 0, need);
        if (e != cudaSuccess) {
            if (p) cudaFree(p);
            p = nullptr;
            return fail(LBFGSB_ERR_OOM, "cudaMalloc(%zu): %s", need, cudaGetErrorString(e));
        }
        bytes = need;
        return LBFGSB_OK;
    }
    void release()
    {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    double* d() const { return static_cast<double*>(p); }
};
}  // namespace

struct lbfgsb_t {
    int64_t n = 0;
    int mh = 0;
    lbfgsb_opts o{};
    cudaStream_t st = nullptr;
    bool own_stream = false;
    // n-sized
    DevBuf l, u, x, g, d, pp, pt, S, Y, mask, xt, gt;
    DevBuf gram_part, gram_grp, dir_part, kkt_part, tickets, sep_part;
    // m-sized (grown on demand)
    DevBuf r0, r1, q, qpart, lsp, fout;
    // sharded packs
    DevBuf pk_loc, qs_all, dir_all, gram_all, kkt_all;
    // host-buffer solve staging
    DevBuf Mh, bh, xh;
    // transport objective
    DevBuf tlam, te, tap, trow, tcol, tsp, tspr, tspc, tticket, tvout;
    // Cauchy-point op and the original L-BFGS-B
    DevBuf cp_d, cp_t, cp_xcp, cp_part, cp_red, cp_heap, cp_scal, cp_ticket;
    DevBuf og_S, og_Y, og_s, og_y, og_rc, og_du, og_d, og_gn, og_r, og_q, og_M, og_part, og_red, og_z, og_out,
        og_ticket;
    Ctrl* ctrl = nullptr;           // device
    Ctrl* hc = nullptr;             // pinned host mirror
    // graph cache
    // two slots (the double-buffered host-batch solve alternates between two
    // operator copies; any other use hits slot 0 again and again)
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    std::vector<Prob> gkey[2];          // the Probs of every logical rank the graph launches
    int gchunk[2] = {0, 0};
    cudaStream_t gstream[2] = {nullptr, nullptr};
    int glast = 0;
    // host-batch double buffering (lbfgsb_solve_lsq_host_batch)
    DevBuf Mh2, bh2, xh2;
    cudaStream_t cst = nullptr;
    cudaEvent_t cev[4] = {nullptr, nullptr, nullptr, nullptr};   // [0,1] copied, [2,3] x* read back
    // profiling
    std::vector<cudaEvent_t> ev;    // 4 per iteration in a chunk: fwd0 fwd1 bwd0 bwd1
    double prof_ms[2] = {0, 0};
    int64_t prof_n[2] = {0, 0};
    int64_t launches = 0;
    int64_t nact_total = 0;
    // sharding
    int rank = 0, nranks = 1;
    int64_t n_global = 0;
    bool comm_owned = false;
    bool sharded = false;
    // P2P exchange (p2p.cu): own mailbox (cudaMalloc, IPC-exportable), the mapped
    // mailboxes of all ranks (own one at [rank]), consumed-count targets
    bool p2p = false;
    void* mb = nullptr;
    int64_t mb_mmax = 0;
    int mb_nranks = 0;
    size_t mb_bytes = 0;
    void* peer_mb[P2P_MAXR] = {};
    bool peer_ipc[P2P_MAXR] = {};
    DevBuf p2p_tgt;
#ifdef LBFGSB_WITH_NCCL
    ncclComm_t comm = nullptr;
#endif
};

// ------------------------------------------------------------------ defaults
extern "C" void lbfgsb_opts_default(lbfgsb_opts* o)
{
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->eps = 1e-9;             // R1
    o->c1 = 1e-4;              // R11
    o->shrink = 0.5;           // R11
    o->tol = 1e-6;             // R15
    o->max_backtracks = 50;    // R11
    o->screen_full_norm = 0;   // R3
    o->check_every = 8;
    o->use_graph = 1;
    o->profile = 0;
    o->max_iters = 10000;
}

extern "C" void al_opts_default(al_opts* o)
{
    if (!o) return;
    std::memset(o, 0, sizeof *o);
    o->feas_tol = 1e-6;
    o->rho0 = 1.0;
    o->rho_factor = 2.0;
    o->rho_cap = 1e12;
    o->max_outer = 100;
}

// ------------------------------------------------------------------ bounds
namespace {
__global__ void k_fill_bounds(double* l, double* u, const double* lin, const double* uin, int64_t n,
                              int* bad)
{
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double a = lin ? lin[j] : -INFINITY;
        const double b = uin ? uin[j] : INFINITY;
        l[j] = a;
        u[j] = b;
        if (!(a <= b)) atomicExch(bad, 1);      // l > u or NaN
    }
}

// l <= u and no NaN, without copying (the batched entry point reads the caller's bounds)
__global__ void k_check_bounds(const double* lin, const double* uin, int64_t n, int* bad)
{
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        const double a = lin ? lin[j] : -INFINITY;
        const double b = uin ? uin[j] : INFINITY;
        if (!(a <= b)) atomicExch(bad, 1);
    }
}
}  // namespace

// option values every entry point accepts (eps > 0, 0 < c1 < 1, 0 < shrink < 1,
// tol >= 0, max_backtracks >= 0, max_iters >= 0); NaN fails every test
static bool opts_valid(const lbfgsb_opts& o)
{
    return (o.eps > 0) && (o.c1 > 0 && o.c1 < 1) && (o.shrink > 0 && o.shrink < 1) && (o.tol >= 0) &&
           o.max_backtracks >= 0 && o.max_iters >= 0;
}

static int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
static int64_t clampi(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

// ------------------------------------------------------------------ create / destroy
static lbfgsb_err alloc_n(lbfgsb_t* h)
{
    const size_t nb = sizeof(double) * (size_t)h->n;
    TRY(h->l.ensure(nb)); TRY(h->u.ensure(nb)); TRY(h->x.ensure(nb)); TRY(h->g.ensure(nb));
    TRY(h->d.ensure(nb)); TRY(h->pp.ensure(nb)); TRY(h->pt.ensure(nb));
    TRY(h->S.ensure(nb * h->mh)); TRY(h->Y.ensure(nb * h->mh));
    TRY(h->mask.ensure((size_t)h->n));
    const int sms = sm_count();
    const int64_t parts = 64LL * sms;     // >= max(GB, G1) for any occupancy
    TRY(h->gram_part.ensure(sizeof(double) * parts * GRAM_STRIDE));
    TRY(h->gram_grp.ensure(sizeof(double) * cdiv(parts, GRP) * GRAM_STRIDE));
    TRY(h->dir_part.ensure(sizeof(double) * 4LL * sms * 4));
    TRY(h->kkt_part.ensure(sizeof(double) * 4LL * sms * 3));
    TRY(h->sep_part.ensure(sizeof(double) * (SEP_MAXG + 1) * KT * NSEP));
    TRY(h->tickets.ensure(sizeof(unsigned) * (NTICKETS + TICKETS_EXTRA), true));
    TRY(h->fout.ensure(sizeof(double) * KT));
    CK(cudaMalloc(&h->ctrl, sizeof(Ctrl)));
    CK(cudaMallocHost(&h->hc, sizeof(Ctrl)));
    std::memset(h->hc, 0, sizeof(Ctrl));
    return LBFGSB_OK;
}

static lbfgsb_err create_common(int64_t n, int32_t m_hist, const double* lower, const double* upper,
                                const lbfgsb_opts* opts, void* stream, lbfgsb_t** out)
{
    if (!out) return fail(LBFGSB_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (n <= 0) return fail(LBFGSB_ERR_DIM, "n = %lld must be positive", (long long)n);
    if (m_hist < 1 || m_hist > LBFGSB_MAX_HIST)
        return fail(LBFGSB_ERR_ARG, "m_hist = %d outside [1, %d]", m_hist, LBFGSB_MAX_HIST);
    lbfgsb_opts o;
    lbfgsb_opts_default(&o);
    if (opts) o = *opts;
    if (!opts_valid(o)) return fail(LBFGSB_ERR_ARG, "invalid option value");
    if (o.trials_per_pass < 0 || o.trials_per_pass > KT || o.refresh_every < 0)
        return fail(LBFGSB_ERR_ARG, "trials_per_pass outside [0, %d] or refresh_every < 0", KT);
    if (o.check_every < 1) o.check_every = 1;
    if (o.check_every > 64) o.check_every = 64;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(LBFGSB_ERR_CUDA, "no CUDA device available (the library has no CPU path)");
    init_kernels();
    lbfgsb_t* h = new lbfgsb_t();
    h->n = n;
    h->n_global = n;
    h->mh = m_hist;
    h->o = o;
    h->st = static_cast<cudaStream_t>(stream);
    if (!h->st) {
        // the legacy default stream cannot be graph-captured: use a private
        // BLOCKING stream, which the legacy stream implicitly orders with
        if (cudaStreamCreate(&h->st) != cudaSuccess) {
            delete h;
            return fail(LBFGSB_ERR_CUDA, "cudaStreamCreate failed");
        }
        h->own_stream = true;
    }
    lbfgsb_err e = alloc_n(h);
    if (e != LBFGSB_OK) { lbfgsb_destroy(h); return e; }
    int* bad = nullptr;
    cudaError_t ce = cudaMalloc(&bad, sizeof(int));
    if (ce == cudaSuccess) ce = cudaMemsetAsync(bad, 0, sizeof(int), h->st);
    if (ce == cudaSuccess) {
        k_fill_bounds<<<256, 256, 0, h->st>>>(h->l.d(), h->u.d(), lower, upper, n, bad);
        ce = cudaGetLastError();
    }
    int hbad = 0;
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, h->st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->st);
    if (bad) cudaFree(bad);
    if (ce != cudaSuccess) {
        lbfgsb_destroy(h);
        return fail(LBFGSB_ERR_CUDA, "bounds setup: %s", cudaGetErrorString(ce));
    }
    if (hbad) { lbfgsb_destroy(h); return fail(LBFGSB_ERR_BOUNDS, "l_i > u_i or NaN bound"); }
    *out = h;
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_create(int64_t n, int32_t m_hist, const double* lower,
                                    const double* upper, const lbfgsb_opts* opts,
                                    void* cuda_stream, lbfgsb_t** out)
{
    return create_common(n, m_hist, lower, upper, opts, cuda_stream, out);
}

extern "C" void lbfgsb_destroy(lbfgsb_t* h)
{
    if (!h) return;
    if (h->st) cudaStreamSynchronize(h->st);
    for (int k = 0; k < 2; ++k)
        if (h->gexec[k]) cudaGraphExecDestroy(h->gexec[k]);
    for (int k = 0; k < 4; ++k)
        if (h->cev[k]) cudaEventDestroy(h->cev[k]);
    if (h->cst) cudaStreamDestroy(h->cst);
    h->Mh2.release(); h->bh2.release(); h->xh2.release();
    for (auto e : h->ev) cudaEventDestroy(e);
    DevBuf* bufs[] = {&h->l, &h->u, &h->x, &h->g, &h->d, &h->pp, &h->pt, &h->S, &h->Y, &h->mask,
                      &h->xt, &h->gt, &h->gram_part, &h->gram_grp, &h->dir_part, &h->kkt_part,
                      &h->tickets, &h->sep_part, &h->r0, &h->r1, &h->q, &h->qpart, &h->lsp,
                      &h->fout, &h->Mh, &h->bh, &h->xh, &h->pk_loc, &h->qs_all, &h->dir_all,
                      &h->gram_all, &h->kkt_all, &h->tlam, &h->te, &h->tap, &h->trow,
                      &h->tcol, &h->tsp, &h->tspr, &h->tspc, &h->tticket, &h->tvout, &h->cp_d,
                      &h->cp_t, &h->cp_xcp, &h->cp_part, &h->cp_red, &h->cp_heap, &h->cp_scal,
                      &h->cp_ticket, &h->og_S, &h->og_Y, &h->og_s, &h->og_y, &h->og_rc, &h->og_du,
                      &h->og_d, &h->og_gn, &h->og_r, &h->og_q, &h->og_M, &h->og_part, &h->og_red,
                      &h->og_z, &h->og_out, &h->og_ticket};
    for (DevBuf* b : bufs) b->release();
    for (int r = 0; r < P2P_MAXR; ++r)
        if (h->peer_ipc[r] && h->peer_mb[r]) cudaIpcCloseMemHandle(h->peer_mb[r]);
    if (h->mb) cudaFree(h->mb);
    h->p2p_tgt.release();
    if (h->ctrl) cudaFree(h->ctrl);
    if (h->hc) cudaFreeHost(h->hc);
#ifdef LBFGSB_WITH_NCCL
    if (h->comm && h->comm_owned) ncclCommDestroy(h->comm);
#endif
    if (h->own_stream) cudaStreamDestroy(h->st);
    delete h;
}

// ------------------------------------------------------------------ objectives
extern "C" lbfgsb_err lbfgsb_objective_lsq(const double* M, int64_t m, int64_t ncols, int64_t ld,
                                           const double* colscale, int32_t split, const double* b,
                                           const double* c, double delta, lbfgsb_objective** out)
{
    if (!out) return fail(LBFGSB_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (!M) return fail(LBFGSB_ERR_ARG, "M is NULL");
    if (m <= 0 || ncols <= 0 || ld < m) return fail(LBFGSB_ERR_DIM, "bad shape m=%lld ncols=%lld ld=%lld",
                                                    (long long)m, (long long)ncols, (long long)ld);
    if (m > (int64_t)FWD_ROWS * 8192 || ncols > (1LL << 31) - 1)
        return fail(LBFGSB_ERR_DIM, "shape too large (m <= %d, ncols < 2^31)", FWD_ROWS * 8192);
    if (split && colscale) return fail(LBFGSB_ERR_ARG, "split and colscale are exclusive");
    if (!std::isfinite(delta)) return fail(LBFGSB_ERR_ARG, "delta not finite");
    auto* o = new lbfgsb_objective();
    o->kind = 0;
    o->M = M; o->m = m; o->ncols = ncols; o->ld = ld;
    o->colscale = colscale; o->split = split ? 1 : 0;
    o->b = b; o->c = c; o->delta = delta;
    *out = o;
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_objective_qp(const double* Q, int64_t n, int64_t ld, const double* colscale,
                                          const double* c, double delta, lbfgsb_objective** out)
{
    TRY(lbfgsb_objective_lsq(Q, n, n, ld, colscale, 0, nullptr, c, delta, out));
    (*out)->qp = 1;
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_objective_transport(const double* M, int64_t m, int64_t n, int32_t reg,
                                                 double lam, lbfgsb_objective** out)
{
    if (!out) return fail(LBFGSB_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (!M) return fail(LBFGSB_ERR_ARG, "M is NULL");
    if (m <= 0 || n <= 0 || m > (1LL << 40) / n) return fail(LBFGSB_ERR_DIM, "bad shape m=%lld n=%lld",
                                                             (long long)m, (long long)n);
    if (reg != 0 && reg != 1) return fail(LBFGSB_ERR_ARG, "reg must be 0 (entropy) or 1 (Gaussian)");
    if (!(lam > 0) || !std::isfinite(lam)) return fail(LBFGSB_ERR_ARG, "lam must be positive");
    auto* o = new lbfgsb_objective();
    o->kind = 2;
    o->M = M; o->m = m; o->ncols = n; o->ld = m;
    o->tm = m; o->tn = n; o->reg = reg; o->lam = lam;
    *out = o;
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_objective_callback(lbfgsb_fg_cb fg, void* user, lbfgsb_objective** out)
{
    if (!out) return fail(LBFGSB_ERR_ARG, "out is NULL");
    *out = nullptr;
    if (!fg) return fail(LBFGSB_ERR_ARG, "fg is NULL");
    auto* o = new lbfgsb_objective();
    o->kind = 1;
    o->fg = fg;
    o->user = user;
    *out = o;
    return LBFGSB_OK;
}

extern "C" void lbfgsb_objective_free(lbfgsb_objective* obj) { delete obj; }

// ------------------------------------------------------------------ geometry
// GEMV launch geometry for an m x ncols operator:
//  k_fwd: RB row blocks of 512 rows x CC column chunks, RB*CC <= resident CTAs
//  k_bwd: GB = min(ncols, resident CTAs) persistent CTAs, balanced columns
static void gemv_geometry(Prob& P)
{
    const int sms = sm_count();
    P.RB = (int)cdiv(P.m, FWD_ROWS);
    static const int waves = getenv("LBFGSB_FWD_WAVES") ? atoi(getenv("LBFGSB_FWD_WAVES")) : 1;
    const int64_t slots_f = (int64_t)sms * fwd_ctas_per_sm(P.m) * (waves > 0 ? waves : 1);
    int64_t cc = clampi(slots_f / P.RB, 1, clampi(cdiv(P.ncols, 16), 1, 1 << 20));
    // the two-level q tail of k_fwd (> FWD_GRPC chunks) has FWD_MAXCG group tickets per row block
    cc = clampi(cc, 1, (int64_t)FWD_GRPC * FWD_MAXCG);
    if (cc > FWD_GRPC && (int64_t)P.RB * FWD_MAXCG > 4096) cc = FWD_GRPC;
    P.chunk = cdiv(P.ncols, cc);
    P.CC = (int)cdiv(P.ncols, P.chunk);
    P.GB = (int)clampi((int64_t)sms * bwd_ctas_per_sm(), 1, P.ncols);
    P.GLS = (int)clampi(cdiv(P.m, NT * 4), 1, 2LL * sms);
}

// Fill the kernel argument block for (handle, objective) and make sure the
// m-sized workspace exists.  Constraint columns are attached by al_solve.
static lbfgsb_err make_prob(lbfgsb_t* h, const lbfgsb_objective* ob, Prob& P)
{
    std::memset(&P, 0, sizeof P);
    const int sms = sm_count();
    P.n = h->n;
    P.l = h->l.d(); P.u = h->u.d();
    P.eps = h->o.eps; P.c1 = h->o.c1; P.shrink = h->o.shrink;
    P.max_bt = h->o.max_backtracks; P.screen_full = h->o.screen_full_norm; P.mh = h->mh;
    P.tpp = h->o.trials_per_pass >= 1 && h->o.trials_per_pass <= KT ? h->o.trials_per_pass : KT;
    P.no_projection = h->o.no_projection ? 1 : 0;
    P.max_iters = h->o.max_iters;
    P.x = h->x.d(); P.g = h->g.d(); P.d = h->d.d(); P.pp = h->pp.d(); P.pt = h->pt.d();
    P.S = h->S.d(); P.Y = h->Y.d(); P.mask = static_cast<uint8_t*>(h->mask.p);
    P.gram_part = h->gram_part.d(); P.gram_grp = h->gram_grp.d();
    P.dir_part = h->dir_part.d(); P.kkt_part = h->kkt_part.d(); P.sep_part = h->sep_part.d();
    P.tickets = static_cast<unsigned*>(h->tickets.p);
    P.ctrl = h->ctrl;
    P.G1 = (int)clampi(cdiv(h->n, NT), 1, 4LL * sms);        // 4 CTAs / SM: latency hiding at large n
    P.nranks = h->nranks;
    P.sharded = h->sharded ? 1 : 0;
    if (ob && ob->kind == 0) {
        const int64_t nv = ob->split ? 2 * ob->ncols : ob->ncols;
        if (nv != h->n)
            return fail(LBFGSB_ERR_DIM, "objective has %lld variables, handle %lld", (long long)nv,
                        (long long)h->n);
        P.m = ob->m; P.ncols = ob->ncols; P.ld = ob->ld; P.M = ob->M;
        P.colscale = ob->colscale; P.split = ob->split; P.b = ob->b; P.c = ob->c; P.delta = ob->delta;
        P.qp = ob->qp;
        P.diff = h->o.armijo_diff ? 1 : 0;                  // R29 (LSQ / QP objectives only)
        if (P.qp && h->sharded) return fail(LBFGSB_ERR_UNSUPPORTED, "QP objectives are single-GPU");
        gemv_geometry(P);
        const size_t mb = sizeof(double) * (size_t)P.m;
        TRY(h->r0.ensure(mb)); TRY(h->r1.ensure(mb)); TRY(h->q.ensure(mb));
        TRY(h->qpart.ensure(mb * P.CC));
        TRY(h->lsp.ensure(sizeof(double) * (size_t)(P.RB > P.GLS ? P.RB : P.GLS) * KT));
        P.rbuf[0] = h->r0.d(); P.rbuf[1] = h->r1.d(); P.q = h->q.d(); P.qpart = h->qpart.d();
        P.lsp = h->lsp.d();
        if (h->sharded) {
            const int R = h->nranks;
            TRY(h->pk_loc.ensure(sizeof(double) * (size_t)pk_len(P), true));
            TRY(h->qs_all.ensure(sizeof(double) * (size_t)R * qs_len(P)));
            TRY(h->dir_all.ensure(sizeof(double) * (size_t)R * 4));
            TRY(h->gram_all.ensure(sizeof(double) * (size_t)R * GRAM_STRIDE));
            TRY(h->kkt_all.ensure(sizeof(double) * (size_t)R * 4));
            P.pk_loc = h->pk_loc.d(); P.qs_all = h->qs_all.d(); P.dir_all = h->dir_all.d();
            P.gram_all = h->gram_all.d(); P.kkt_all = h->kkt_all.d();
            if (h->p2p) {                                     // gathered sections live in the mailbox
                if (R != h->mb_nranks)
                    return fail(LBFGSB_ERR_ARG, "P2P mailbox made for %d ranks, group has %d", h->mb_nranks, R);
                if (P.m > h->mb_mmax)
                    return fail(LBFGSB_ERR_DIM, "P2P mailbox sized for m <= %lld, objective has m = %lld",
                                (long long)h->mb_mmax, (long long)P.m);
                for (int r = 0; r < R; ++r)
                    if (!h->peer_mb[r]) return fail(LBFGSB_ERR_ARG, "P2P exchange: rank %d not connected", r);
                P.p2p = 1;
                P.rank_id = h->rank;
                for (int r = 0; r < R; ++r) P.peer_mb[r] = static_cast<double*>(h->peer_mb[r]);
                double* mb = static_cast<double*>(h->mb);
                P.mb_hdr = static_cast<unsigned long long*>(h->mb);
                P.p2p_tgt = static_cast<unsigned long long*>(h->p2p_tgt.p);
                P.qs_all = mb + mb_off(P, XS_QS);
                P.dir_all = mb + mb_off(P, XS_DIR);
                P.gram_all = mb + mb_off(P, XS_GRAM);
                P.kkt_all = mb + mb_off(P, XS_KKT);
            }
        }
    }
    if (ob && ob->kind == 2) {                                 // transport
        if (ob->tm * ob->tn != h->n)
            return fail(LBFGSB_ERR_DIM, "transport objective has %lld variables, handle %lld",
                        (long long)(ob->tm * ob->tn), (long long)h->n);
        if (h->sharded) return fail(LBFGSB_ERR_UNSUPPORTED, "transport objectives are single-GPU");
        P.tp = 1;
        P.tm = ob->tm; P.tn = ob->tn;
        P.c = ob->M;
        if (ob->reg == 1) P.delta = ob->lam; else P.ent = ob->lam;
        P.diff = 1;                                            // R29 (always, see transport.cu)
        P.TRB = (int)cdiv(P.tm, NT);
        P.TCB = (int)cdiv(P.tn, TCOLS);
        const int64_t K = P.tm + P.tn;
        const size_t kb = sizeof(double) * (size_t)K;
        TRY(h->r0.ensure(kb)); TRY(h->r1.ensure(kb));
        TRY(h->tlam.ensure(kb)); TRY(h->te.ensure(kb)); TRY(h->tap.ensure(kb));
        TRY(h->trow.ensure(sizeof(double) * (size_t)P.TCB * P.tm));
        TRY(h->tcol.ensure(sizeof(double) * (size_t)P.TRB * P.tn));
        TRY(h->tsp.ensure(sizeof(double) * (size_t)P.TRB * P.TCB * TNS));
        TRY(h->tspr.ensure(sizeof(double) * (size_t)P.TRB * 2));
        TRY(h->tspc.ensure(sizeof(double) * (size_t)P.TCB * 2));
        TRY(h->tticket.ensure(sizeof(unsigned) * (size_t)(P.TRB + P.TCB + 2), true));
        TRY(h->tvout.ensure(sizeof(double)));
        P.rbuf[0] = h->r0.d(); P.rbuf[1] = h->r1.d();
        P.tlam = h->tlam.d(); P.te = h->te.d(); P.tap = h->tap.d();
        P.trow = h->trow.d(); P.tcol = h->tcol.d(); P.tsp = h->tsp.d();
        P.tspr = h->tspr.d(); P.tspc = h->tspc.d();
        P.tticket = static_cast<unsigned*>(h->tticket.p);
    }
    return LBFGSB_OK;
}

static void set_sep(Prob& P)
{
    const bool has_sep = P.c || P.delta != 0.0 || (P.n_eq + P.n_in) > 0;
    P.GS = has_sep ? (int)clampi(cdiv(P.n, 1024), 1, SEP_MAXG) : 0;
}

static lbfgsb_err ctrl_to_dev(lbfgsb_t* h, cudaStream_t st)
{
    CK(cudaMemcpyAsync(h->ctrl, h->hc, sizeof(Ctrl), cudaMemcpyHostToDevice, st));
    return LBFGSB_OK;
}
static lbfgsb_err ctrl_to_host(lbfgsb_t* h, cudaStream_t st)
{
    CK(cudaMemcpyAsync(h->hc, h->ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return LBFGSB_OK;
}

#define FOR_RANKS_P for (size_t i_ = 0; i_ < g.Ps.size(); ++i_)
// ------------------------------------------------------------------ groups
// A Group is the set of handles that take part in one solve: one handle (a
// single-GPU solve, or this rank of an NCCL-sharded solve), or nranks
// handles acting as logical ranks of a loopback-sharded solve on one device.
// All launches of a group go to one stream.
namespace {
enum Section { SEC_QS = 0, SEC_DIR, SEC_GRAM, SEC_KKT };
struct Group {
    std::vector<lbfgsb_t*> hs;
    std::vector<Prob> Ps;
    cudaStream_t st = nullptr;
    bool sharded = false;     // local packs + exchange + *_decide
    bool loopback = false;    // exchange by device copies between the handles
    lbfgsb_t* h0() const { return hs[0]; }
};
}  // namespace

static lbfgsb_err ctrl_to_dev(Group& g)
{
    for (auto* h : g.hs) TRY(ctrl_to_dev(h, g.st));
    return LBFGSB_OK;
}
static lbfgsb_err ctrl_to_host(Group& g)
{
    for (auto* h : g.hs) TRY(ctrl_to_host(h, g.st));
    return LBFGSB_OK;
}

// All-gather one pack section across the ranks (rank order).  P2P handles:
// the producing kernel already pushed its section (fused in its tail) unless
// `put`; only the waits are launched here.  `iter`: the producer returns at
// entry when the solve is halted, so the wait is skipped then too.  A fused
// k_fwd push signals once per row block (`per_rb`).
static lbfgsb_err xchg(Group& g, Section sec, bool iter = false, bool per_rb = false, bool put = false)
{
    const Prob& P0 = g.Ps[0];
    if (P0.p2p) {
        const int R = (int)P0.nranks;
        if (put) {
            FOR_RANKS_P launch_p2p_put(g.Ps[i_], g.st, (int)sec, 0, qs_len(P0));
        }
        // the consuming kernel waits in its prologue (k_dir_decide, k_ls, k_gram_decide, k_kkt_decide)
        (void)R; (void)iter; (void)per_rb;
        return LBFGSB_OK;
    }
    int64_t off = 0, cnt = 0;
    switch (sec) {
        case SEC_QS: off = 0; cnt = qs_len(P0); break;
        case SEC_DIR: off = off_dir(P0); cnt = 4; break;
        case SEC_GRAM: off = off_gram(P0); cnt = GRAM_STRIDE; break;
        case SEC_KKT: off = off_kkt(P0); cnt = 4; break;
    }
    auto recv_of = [&](const Prob& P) {
        return sec == SEC_QS ? P.qs_all : sec == SEC_DIR ? P.dir_all : sec == SEC_GRAM ? P.gram_all : P.kkt_all;
    };
    if (g.loopback) {
        const int R = (int)g.hs.size();
        for (int q = 0; q < R; ++q)
            for (int p = 0; p < R; ++p)
                CK(cudaMemcpyAsync(recv_of(g.Ps[q]) + (int64_t)p * cnt, g.Ps[p].pk_loc + off,
                                   sizeof(double) * (size_t)cnt, cudaMemcpyDeviceToDevice, g.st));
        return LBFGSB_OK;
    }
#ifdef LBFGSB_WITH_NCCL
    ncclResult_t r = ncclAllGather(P0.pk_loc + off, recv_of(P0), (size_t)cnt, ncclDouble, g.h0()->comm, g.st);
    if (r != ncclSuccess) return fail(LBFGSB_ERR_NCCL, "ncclAllGather: %s", ncclGetErrorString(r));
    return LBFGSB_OK;
#else
    return fail(LBFGSB_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

#define FOR_RANKS for (size_t i_ = 0; i_ < g.hs.size(); ++i_)
#define PR g.Ps[i_]

static void rec_event(Group& g, int idx)
{
    lbfgsb_t* h = g.h0();
    if (!h->o.profile || idx < 0) return;
    cudaEventRecordWithFlags(h->ev[idx], g.st, cudaEventRecordExternal);
}

static int per_iteration_launches(const Group& g)
{
    const int sep = g.Ps[0].GS > 0;
    if (g.Ps[0].tp) return g.Ps[0].ent != 0.0 ? 4 : 3;
    return g.sharded ? (int)g.hs.size() * (6 + sep) : 3 + sep;
}

// One LSQ iteration (Alg. 1 lines 3-10).  Single GPU: k_dir [k_sep] k_fwd
// k_bwd with fused decisions.  Sharded: each decision point becomes local
// pack -> all-gather -> *_decide.
static lbfgsb_err launch_iteration(Group& g, int ev_base)
{
    cudaStream_t st = g.st;
    if (g.Ps[0].tp) {                                          // transport: k_dir k_tsum k_qpu
        const Prob& P = g.Ps[0];
        launch_dir(P, st, 0);
        rec_event(g, ev_base >= 0 ? ev_base + 0 : -1);
        launch_tsum(P, st, TS_ITER);
        if (P.ent != 0.0) launch_tsum(P, st, TS_CONT);          // no-op unless trial 0 failed
        rec_event(g, ev_base >= 0 ? ev_base + 1 : -1);     // also the start of k_bwd (no +2 node)
        launch_bwd(P, st, BWD_ITER, nullptr, nullptr);
        rec_event(g, ev_base >= 0 ? ev_base + 3 : -1);
    } else if (!g.sharded) {
        const Prob& P = g.Ps[0];
        launch_dir(P, st, 0);
        launch_sep(P, st, SEP_ITER, nullptr);
        rec_event(g, ev_base >= 0 ? ev_base + 0 : -1);
        launch_fwd(P, st, FWD_ITER, nullptr, nullptr);
        rec_event(g, ev_base >= 0 ? ev_base + 1 : -1);     // also the start of k_bwd (no +2 node)
        launch_bwd(P, st, BWD_ITER, nullptr, nullptr);
        rec_event(g, ev_base >= 0 ? ev_base + 3 : -1);
    } else {
        FOR_RANKS launch_dir(PR, st, 0);
        TRY(xchg(g, SEC_DIR, true));
        FOR_RANKS launch_dir_decide(PR, st);
        FOR_RANKS launch_sep(PR, st, SEP_ITER, nullptr);
        rec_event(g, ev_base >= 0 ? ev_base + 0 : -1);
        FOR_RANKS launch_fwd(PR, st, FWD_ITER, nullptr, nullptr);
        rec_event(g, ev_base >= 0 ? ev_base + 1 : -1);
        TRY(xchg(g, SEC_QS, true, true));
        FOR_RANKS launch_ls(PR, st, LS_SH_ITER, nullptr, nullptr, nullptr, 0);
        rec_event(g, ev_base >= 0 ? ev_base + 2 : -1);
        FOR_RANKS launch_bwd(PR, st, BWD_ITER, nullptr, nullptr);
        rec_event(g, ev_base >= 0 ? ev_base + 3 : -1);
        TRY(xchg(g, SEC_GRAM, true));
        FOR_RANKS launch_gram_decide(PR, st, BWD_ITER);
    }
    g.h0()->launches += per_iteration_launches(g);
    return LBFGSB_OK;
}

// f(x), r = M~x - b, and the constraint values at x (setup / AL start).
static lbfgsb_err launch_fval(Group& g, bool clip)
{
    cudaStream_t st = g.st;
    if (g.Ps[0].tp) {
        if (clip) launch_clip(g.Ps[0], st);
        launch_tsum(g.Ps[0], st, TS_SETUP);
        return LBFGSB_OK;
    }
    FOR_RANKS {
        if (clip) launch_clip(PR, st);
        launch_sep(PR, st, SEP_SETUP, PR.x);
        launch_fwd(PR, st, FWD_SETUP, PR.x, nullptr);
    }
    if (g.sharded) {
        TRY(xchg(g, SEC_QS, false, true));
        FOR_RANKS launch_ls(PR, st, LS_SH_SETUP, nullptr, nullptr, nullptr, 0);
    }
    return LBFGSB_OK;
}

// Setup at x^0 (x = clip(x0); r = M~x - b; f; g; S^0; Gram;
// convergence test; coefficients of the first direction).
static lbfgsb_err launch_setup(Group& g)
{
    TRY(launch_fval(g, true));
    FOR_RANKS launch_bwd(PR, g.st, BWD_SETUP, nullptr, nullptr);
    if (g.sharded) {
        TRY(xchg(g, SEC_GRAM));
        FOR_RANKS launch_gram_decide(PR, g.st, BWD_SETUP);
    }
    g.h0()->launches += 4;
    return LBFGSB_OK;
}

// Final refresh (R13): r = M~x - b, f, g = grad f(x) and the KKT report.
static lbfgsb_err launch_refresh(Group& g)
{
    TRY(launch_fval(g, false));
    FOR_RANKS {
        launch_bwd(PR, g.st, BWD_REFRESH, nullptr, nullptr);
        launch_kkt(PR, g.st);
    }
    if (g.sharded) {
        TRY(xchg(g, SEC_KKT));
        FOR_RANKS launch_kkt_decide(PR, g.st);
    }
    g.h0()->launches += 4;
    return LBFGSB_OK;
}

// Stall continuation: next Armijo batch, then the gradient pass.
static lbfgsb_err launch_ls_cont(Group& g)
{
    if (g.Ps[0].tp) {
        launch_tsum(g.Ps[0], g.st, TS_NEXT);
        launch_bwd(g.Ps[0], g.st, BWD_ITER, nullptr, nullptr);
        g.h0()->launches += 2;
        return LBFGSB_OK;
    }
    FOR_RANKS launch_sep(PR, g.st, SEP_NEXT, nullptr);
    if (g.sharded && g.Ps[0].GS > 0) TRY(xchg(g, SEC_QS, false, false, true));
    FOR_RANKS launch_ls(PR, g.st, LS_NEXT, nullptr, nullptr, nullptr, 0);
    FOR_RANKS launch_bwd(PR, g.st, BWD_ITER, nullptr, nullptr);
    if (g.sharded) {
        TRY(xchg(g, SEC_GRAM, true));
        FOR_RANKS launch_gram_decide(PR, g.st, BWD_ITER);
    }
    g.h0()->launches += 3;
    return LBFGSB_OK;
}

static lbfgsb_err ensure_events(lbfgsb_t* h)
{
    const size_t need = (size_t)4 * h->o.check_every;
    while (h->ev.size() < need) {
        cudaEvent_t e;
        CK(cudaEventCreate(&e));
        h->ev.push_back(e);
    }
    return LBFGSB_OK;
}

static lbfgsb_err run_chunk(Group& g, int chunk)
{
    lbfgsb_t* h = g.h0();
    const bool graph = h->o.use_graph && !g.loopback;
    if (graph) {
        int sl = -1;
        for (int k = 0; k < 2 && sl < 0; ++k)
            if (h->gexec[k] && h->gkey[k].size() == g.Ps.size() &&
                std::memcmp(h->gkey[k].data(), g.Ps.data(), sizeof(Prob) * g.Ps.size()) == 0 &&
                h->gchunk[k] == chunk && h->gstream[k] == g.st)
                sl = k;
        if (sl < 0) {
            sl = h->gexec[0] == nullptr ? 0 : (h->gexec[1] == nullptr ? 1 : h->glast ^ 1);   // replace the LRU slot
            if (h->gexec[sl]) { cudaGraphExecDestroy(h->gexec[sl]); h->gexec[sl] = nullptr; }
            cudaGraph_t gr = nullptr;
            CK(cudaStreamBeginCapture(g.st, cudaStreamCaptureModeThreadLocal));
            const int64_t l0 = h->launches;
            lbfgsb_err e0 = LBFGSB_OK;
            for (int i = 0; i < chunk && e0 == LBFGSB_OK; ++i) e0 = launch_iteration(g, h->o.profile ? 4 * i : -1);
            h->launches = l0;
            cudaError_t e = cudaStreamEndCapture(g.st, &gr);
            if (e0 != LBFGSB_OK) { if (gr) cudaGraphDestroy(gr); return e0; }
            if (e != cudaSuccess) return fail(LBFGSB_ERR_CUDA, "graph capture: %s", cudaGetErrorString(e));
            e = cudaGraphInstantiate(&h->gexec[sl], gr, 0);
            cudaGraphDestroy(gr);
            if (e != cudaSuccess) return fail(LBFGSB_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(e));
            h->gkey[sl] = g.Ps;
            h->gchunk[sl] = chunk;
            h->gstream[sl] = g.st;
        }
        h->glast = sl;
        CK(cudaGraphLaunch(h->gexec[sl], g.st));
        h->launches += (int64_t)per_iteration_launches(g) * chunk;
    } else {
        for (int i = 0; i < chunk; ++i) TRY(launch_iteration(g, h->o.profile ? 4 * i : -1));
    }
    CK(cudaGetLastError());
    return LBFGSB_OK;
}

static void collect_profile(lbfgsb_t* h, int64_t iters_done)
{
    if (!h->o.profile) return;
    const int64_t c = iters_done < h->o.check_every ? iters_done : h->o.check_every;
    for (int64_t i = 0; i < c; ++i) {
        float a = 0.f, b = 0.f;
        if (cudaEventElapsedTime(&a, h->ev[4 * i + 0], h->ev[4 * i + 1]) == cudaSuccess) {
            h->prof_ms[0] += a; h->prof_n[0] += 1;
        }
        // single GPU: k_bwd follows k_fwd directly, so its start event is the fwd-end one
        const int bs = h->sharded ? 2 : 1;
        if (cudaEventElapsedTime(&b, h->ev[4 * i + bs], h->ev[4 * i + 3]) == cudaSuccess) {
            h->prof_ms[1] += b; h->prof_n[1] += 1;
        }
    }
    cudaGetLastError();
}

static void init_ctrl(lbfgsb_t* h, double tol)
{
    Ctrl* c = h->hc;
    double lam[MAXC], rhs[MAXC], rho = c->rho;
    std::memcpy(lam, c->lam, sizeof lam);
    std::memcpy(rhs, c->rhs, sizeof rhs);
    std::memset(c, 0, sizeof(Ctrl));
    c->head = h->mh - 1;          // first stored pair goes to slot 0
    c->tol = tol;
    c->rho = rho > 0 ? rho : 1.0;
    std::memcpy(c->lam, lam, sizeof lam);
    std::memcpy(c->rhs, rhs, sizeof rhs);
}

// Alg. 1 on an LSQ objective for a group; xs[p] (device) in/out.  AL params
// already in every handle's host mirror.
static lbfgsb_err solve_group(Group& g, double* const* xs, double tol, lbfgsb_result* res)
{
    auto t0 = std::chrono::steady_clock::now();
    lbfgsb_t* h = g.h0();
    FOR_RANKS {
        lbfgsb_t* hh = g.hs[i_];
        if (xs[i_] != PR.x)
            CK(cudaMemcpyAsync(PR.x, xs[i_], sizeof(double) * hh->n, cudaMemcpyDeviceToDevice, g.st));
        init_ctrl(hh, tol);
        hh->hc->n_fg = 1;
    }
    TRY(ctrl_to_dev(g));
    TRY(launch_setup(g));
    CK(cudaGetLastError());
    TRY(ctrl_to_host(g));
    if (h->hc->nonfinite) return fail(LBFGSB_ERR_NONFINITE, "f(x0) is not finite");
    if (h->o.profile) TRY(ensure_events(h));

    const int64_t guard = h->o.max_iters + 64;
    const int R = h->o.refresh_every > 0 ? h->o.refresh_every : 0;
    int64_t loops = 0;
    while (!h->hc->done) {
        const long long k0 = h->hc->k;
        // with a periodic refresh every chunk ends at the next multiple of R
        int chunk = h->o.check_every;
        if (R > 0 && R - (int)(k0 % R) < chunk) chunk = R - (int)(k0 % R);
        TRY(run_chunk(g, chunk));
        TRY(ctrl_to_host(g));
        collect_profile(h, h->hc->k - k0);
        if (++loops > guard) return fail(LBFGSB_ERR_CUDA, "solver loop did not terminate");
        // ---- stall handling (rare): finish the stalled iteration on the host's cue
        while (h->hc->stall && !h->hc->done) {
            const int s = h->hc->stall;
            for (auto* hh : g.hs) {
                Ctrl* c = hh->hc;
                c->stall = 0;
                if (s == ST_FALLBACK) {
                    // R14: clear the history, d[S] = -g[S], redo Alg. 2 + the search
                    c->fallback = 1;
                    c->nh = 0;
                    c->n_fallbacks += 1;
                    c->coef[0] = -1.0;
                }
            }
            TRY(ctrl_to_dev(g));
            // P2P: no rank may re-push DIR / QS while a peer still reads the previous pack
            if (g.Ps[0].p2p) launch_p2p_barrier(g.Ps.data(), (int)g.Ps.size(), g.st);
            if (s == ST_FALLBACK) TRY(launch_iteration(g, -1));
            else TRY(launch_ls_cont(g));
            CK(cudaGetLastError());
            TRY(ctrl_to_host(g));
        }
        // R13's optional refresh at the top of iteration k, k % R == 0: r = M~x - b, f, g, the
        // working set, the convergence test and Alg. 3 again from the exact values (the setup
        // sequence without the clip; the curvature pairs are kept)
        if (R > 0 && !h->hc->done && h->hc->k > 0 && h->hc->k % R == 0 && h->hc->k != k0 &&
            !g.Ps[0].tp && !h->hc->stall) {
            if (g.Ps[0].p2p) launch_p2p_barrier(g.Ps.data(), (int)g.Ps.size(), g.st);
            TRY(launch_fval(g, false));
            FOR_RANKS launch_bwd(PR, g.st, BWD_SETUP, nullptr, nullptr);
            if (g.sharded) {
                TRY(xchg(g, SEC_GRAM));
                FOR_RANKS launch_gram_decide(PR, g.st, BWD_SETUP);
            }
            h->launches += 4;
            CK(cudaGetLastError());
            TRY(ctrl_to_host(g));
        }
    }
    const Ctrl fin = *h->hc;
    for (auto* hh : g.hs) h->nact_total += hh->hc->nact;     // active columns read by every local k_fwd
    TRY(launch_refresh(g));
    CK(cudaGetLastError());
    TRY(ctrl_to_host(g));
    if (g.Ps[0].p2p) {
        unsigned long long to = 0;
        FOR_RANKS {
            unsigned long long v = 0;
            CK(cudaMemcpyAsync(&v, PR.mb_hdr + 4, sizeof v, cudaMemcpyDeviceToHost, g.st));
            CK(cudaStreamSynchronize(g.st));
            to |= v;
        }
        if (to) return fail(LBFGSB_ERR_NCCL, "P2P exchange timed out (a peer stopped signalling)");
    }
    FOR_RANKS {
        if (xs[i_] != PR.x)
            CK(cudaMemcpyAsync(xs[i_], PR.x, sizeof(double) * g.hs[i_]->n, cudaMemcpyDeviceToDevice, g.st));
    }
    CK(cudaStreamSynchronize(g.st));
    auto t1 = std::chrono::steady_clock::now();
    if (res) {
        std::memset(res, 0, sizeof *res);
        res->f = h->hc->f;
        res->pg_inf = h->hc->pg;
        res->gfree_inf = h->hc->gfree;
        res->n_free = h->hc->nfree;
        res->iters = fin.k;
        res->n_fg = fin.n_fg;
        res->n_backtracks = fin.n_bt;
        res->n_fallbacks = fin.n_fallbacks;
        res->status = fin.status;
        res->last_branch = fin.branch;
        res->seconds = std::chrono::duration<double>(t1 - t0).count();
    }
    return LBFGSB_OK;
}

static lbfgsb_err single_group(lbfgsb_t* h, const lbfgsb_objective* obj, Group& g)
{
    g.hs = {h};
    g.Ps.resize(1);
    TRY(make_prob(h, obj, g.Ps[0]));
    g.st = h->st;
    g.sharded = h->sharded;
    g.loopback = false;
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ callback objective
static lbfgsb_err solve_cb(lbfgsb_t* h, const lbfgsb_objective* ob, double* x_user, double tol,
                           lbfgsb_result* res)
{
    auto t0 = std::chrono::steady_clock::now();
    Prob P;
    TRY(make_prob(h, ob, P));
    const size_t nb = sizeof(double) * h->n;
    TRY(h->xt.ensure(nb));
    TRY(h->gt.ensure(nb));
    cudaStream_t st = h->st;
    CK(cudaMemcpyAsync(P.x, x_user, nb, cudaMemcpyDeviceToDevice, st));
    init_ctrl(h, tol);
    launch_clip(P, st);
    CK(cudaGetLastError());
    double f = 0.0;
    if (ob->fg(ob->user, P.x, P.g, &f, st) != 0) return fail(LBFGSB_ERR_CALLBACK, "callback failed at x0");
    if (!std::isfinite(f)) return fail(LBFGSB_ERR_NONFINITE, "f(x0) is not finite");
    Ctrl* c = h->hc;
    c->f = f;
    c->n_fg = 1;
    TRY(ctrl_to_dev(h, st));
    for (;;) {
        launch_gram_recur(P, st, 0);
        launch_dir(P, st, 0);
        h->launches += 2;
        CK(cudaGetLastError());
        TRY(ctrl_to_host(h, st));
        if (c->done) break;
        if (c->stall == ST_FALLBACK) {
            c->stall = 0; c->fallback = 1; c->nh = 0; c->n_fallbacks += 1;
            TRY(ctrl_to_dev(h, st));
            continue;
        }
        double a = c->alpha0, ft = 0.0;
        bool acc = false;
        for (int t = 0; t <= h->o.max_backtracks; ++t) {
            if (t > 0) a = a * h->o.shrink;
            launch_cb_trial(P, st, a, h->xt.d());
            h->launches += 1;
            if (ob->fg(ob->user, h->xt.d(), h->gt.d(), &ft, st) != 0)
                return fail(LBFGSB_ERR_CALLBACK, "callback failed");
            c->n_fg += 1;
            if (ft <= c->f + h->o.c1 * a * c->gp) { acc = true; break; }
            c->n_bt += 1;
        }
        if (!acc) {
            if (c->fallback) { c->done = 1; c->status = S_LS_FAIL; break; }
            c->fallback = 1; c->nh = 0; c->n_fallbacks += 1;
            TRY(ctrl_to_dev(h, st));
            continue;
        }
        const int head = (c->head + 1) % h->mh;
        launch_cb_commit(P, st, h->xt.d(), h->gt.d(), head);
        h->launches += 1;
        c->head = head; c->slot = head;
        c->nh = c->nh + 1 < h->mh ? c->nh + 1 : h->mh;
        c->k += 1; c->fallback = 0; c->f = ft; c->alpha = a;
        TRY(ctrl_to_dev(h, st));
    }
    const Ctrl fin = *c;
    launch_kkt(P, st);
    h->launches += 1;
    CK(cudaGetLastError());
    TRY(ctrl_to_host(h, st));
    CK(cudaMemcpyAsync(x_user, P.x, nb, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    auto t1 = std::chrono::steady_clock::now();
    if (res) {
        std::memset(res, 0, sizeof *res);
        res->f = fin.f;
        res->pg_inf = h->hc->pg;
        res->gfree_inf = h->hc->gfree;
        res->n_free = h->hc->nfree;
        res->iters = fin.k; res->n_fg = fin.n_fg; res->n_backtracks = fin.n_bt;
        res->n_fallbacks = fin.n_fallbacks; res->status = fin.status; res->last_branch = fin.branch;
        res->seconds = std::chrono::duration<double>(t1 - t0).count();
    }
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_solve(lbfgsb_t* h, const lbfgsb_objective* obj, double* x, double tol,
                                   lbfgsb_result* res)
{
    if (!h || !obj || !x) return fail(LBFGSB_ERR_ARG, "NULL handle, objective or x");
    const double t = tol > 0 ? tol : h->o.tol;
    if (obj->kind == 1) {
        if (h->sharded) return fail(LBFGSB_ERR_UNSUPPORTED, "callback objectives are single-GPU");
        return solve_cb(h, obj, x, t, res);
    }
    if (obj->kind == 2)
        return fail(LBFGSB_ERR_UNSUPPORTED, "transport objectives are solved with al_solve_transport");
    Group g;
    TRY(single_group(h, obj, g));
    set_sep(g.Ps[0]);
    h->hc->rho = 1.0;
    std::memset(h->hc->lam, 0, sizeof h->hc->lam);
    std::memset(h->hc->rhs, 0, sizeof h->hc->rhs);
    double* xs[1] = {x};
    return solve_group(g, xs, t, res);
}

extern "C" lbfgsb_err lbfgsb_solve_loopback(lbfgsb_t* const* hs, const lbfgsb_objective* const* objs,
                                            double* const* xs, int32_t nranks, double tol, lbfgsb_result* res)
{
    if (!hs || !objs || !xs || nranks < 1) return fail(LBFGSB_ERR_ARG, "bad arguments");
    Group g;
    g.st = hs[0]->st;
    g.sharded = nranks > 1;
    g.loopback = nranks > 1;
    g.Ps.resize(nranks);
    int64_t nglob = 0;
    for (int p = 0; p < nranks; ++p) {
        if (!hs[p] || !objs[p] || !xs[p] || objs[p]->kind != 0) return fail(LBFGSB_ERR_ARG, "bad rank %d", p);
        if (hs[p]->comm_owned) return fail(LBFGSB_ERR_ARG, "NCCL handle in loopback");
        nglob += hs[p]->n;
    }
    for (int p = 0; p < nranks; ++p) {
        hs[p]->nranks = nranks;
        hs[p]->sharded = nranks > 1;
        hs[p]->rank = p;
        hs[p]->n_global = nglob;
        g.hs.push_back(hs[p]);
        lbfgsb_err e = make_prob(hs[p], objs[p], g.Ps[p]);
        if (e == LBFGSB_OK && objs[p]->m != objs[0]->m) e = fail(LBFGSB_ERR_DIM, "ranks disagree on m");
        if (e != LBFGSB_OK) {
            for (int q = 0; q < nranks; ++q) { hs[q]->nranks = 1; hs[q]->sharded = false; }
            return e;
        }
        set_sep(g.Ps[p]);
        hs[p]->hc->rho = 1.0;
        std::memset(hs[p]->hc->lam, 0, sizeof hs[p]->hc->lam);
        std::memset(hs[p]->hc->rhs, 0, sizeof hs[p]->hc->rhs);
    }
    // separable-part geometry must agree across ranks (it is part of the pack layout)
    const double t = tol > 0 ? tol : hs[0]->o.tol;
    lbfgsb_err e = solve_group(g, xs, t, res);
    for (int p = 0; p < nranks; ++p) {
        hs[p]->nranks = 1; hs[p]->sharded = false; hs[p]->rank = 0; hs[p]->n_global = hs[p]->n;
    }
    return e;
}

// SURVEY 8(e) bitwise P-invariance: a process hosts n_local LOGICAL ranks of a
// P2P-sharded solve over C = nranks fixed column chunks (each handle made by
// lbfgsb_create_sharded_p2p with its logical rank, mailboxes wired with
// lbfgsb_p2p_open_group).  Every logical rank runs its kernels with the
// geometry of its own chunk and every decision reduces the C packs in
// logical-rank order, so the iterates do not depend on how the C chunks are
// spread over processes / GPUs.  All launches go to hs[0]'s stream; the
// iteration is captured as one CUDA graph over all local logical ranks.
extern "C" lbfgsb_err lbfgsb_solve_group(lbfgsb_t* const* hs, const lbfgsb_objective* const* objs,
                                         double* const* xs, int32_t n_local, double tol, lbfgsb_result* res)
{
    if (!hs || !objs || !xs || n_local < 1) return fail(LBFGSB_ERR_ARG, "bad arguments");
    Group g;
    g.st = hs[0]->st;
    g.sharded = true;
    g.loopback = false;
    g.Ps.resize(n_local);
    for (int p = 0; p < n_local; ++p) {
        if (!hs[p] || !objs[p] || !xs[p] || objs[p]->kind != 0) return fail(LBFGSB_ERR_ARG, "bad local rank %d", p);
        if (!hs[p]->p2p || !hs[p]->sharded || hs[p]->nranks != hs[0]->nranks)
            return fail(LBFGSB_ERR_ARG, "local rank %d: not a P2P-sharded handle of the same group", p);
        for (int r = 0; r < hs[p]->nranks; ++r)
            if (!hs[p]->peer_mb[r]) return fail(LBFGSB_ERR_ARG, "P2P exchange: rank %d not connected", r);
        g.hs.push_back(hs[p]);
        TRY(make_prob(hs[p], objs[p], g.Ps[p]));
        if (objs[p]->m != objs[0]->m) return fail(LBFGSB_ERR_DIM, "ranks disagree on m");
        set_sep(g.Ps[p]);
        hs[p]->hc->rho = 1.0;
        std::memset(hs[p]->hc->lam, 0, sizeof hs[p]->hc->lam);
        std::memset(hs[p]->hc->rhs, 0, sizeof hs[p]->hc->rhs);
    }
    const double t = tol > 0 ? tol : hs[0]->o.tol;
    return solve_group(g, xs, t, res);
}

extern "C" lbfgsb_err lbfgsb_solve_lsq_host(lbfgsb_t* h, const double* M_host, int64_t m, int64_t ncols,
                                            const double* b_host, double* x_host, double tol,
                                            lbfgsb_result* res)
{
    if (!h || !M_host || !x_host) return fail(LBFGSB_ERR_ARG, "NULL handle, M or x");
    if (m <= 0 || ncols != h->n) return fail(LBFGSB_ERR_DIM, "shape mismatch");
    const size_t mb = sizeof(double) * (size_t)m * (size_t)ncols;
    TRY(h->Mh.ensure(mb));
    TRY(h->bh.ensure(sizeof(double) * (size_t)m));
    TRY(h->xh.ensure(sizeof(double) * (size_t)ncols));
    CK(cudaMemcpyAsync(h->Mh.p, M_host, mb, cudaMemcpyHostToDevice, h->st));
    if (b_host) CK(cudaMemcpyAsync(h->bh.p, b_host, sizeof(double) * m, cudaMemcpyHostToDevice, h->st));
    CK(cudaMemcpyAsync(h->xh.p, x_host, sizeof(double) * ncols, cudaMemcpyHostToDevice, h->st));
    lbfgsb_objective ob{};
    ob.kind = 0; ob.M = h->Mh.d(); ob.m = m; ob.ncols = ncols; ob.ld = m;
    ob.b = b_host ? h->bh.d() : nullptr;
    TRY(lbfgsb_solve(h, &ob, h->xh.d(), tol, res));
    CK(cudaMemcpyAsync(x_host, h->xh.p, sizeof(double) * ncols, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return LBFGSB_OK;
}

// Many problems from host memory, double-buffered: the H2D copy of problem k+1
// (copy stream) overlaps the solve of problem k; every problem's H2D of M, b,
// x0 and D2H of x* happen inside the call.
extern "C" lbfgsb_err lbfgsb_solve_lsq_host_batch(lbfgsb_t* h, int32_t count, const double* const* M_hosts,
                                                  int64_t m, int64_t ncols, const double* const* b_hosts,
                                                  double* const* x_hosts, double tol, lbfgsb_result* res)
{
    if (!h || count < 0 || (count > 0 && (!M_hosts || !x_hosts || !res))) return fail(LBFGSB_ERR_ARG, "bad arguments");
    if (m <= 0 || ncols != h->n) return fail(LBFGSB_ERR_DIM, "shape mismatch");
    if (h->sharded) return fail(LBFGSB_ERR_UNSUPPORTED, "single-GPU handles only");
    if (count == 0) return LBFGSB_OK;
    for (int k = 0; k < count; ++k)
        if (!M_hosts[k] || !x_hosts[k]) return fail(LBFGSB_ERR_ARG, "NULL M or x of problem %d", k);
    const size_t mb = sizeof(double) * (size_t)m * (size_t)ncols;
    DevBuf* Mb[2] = {&h->Mh, &h->Mh2};
    DevBuf* bb[2] = {&h->bh, &h->bh2};
    DevBuf* xb[2] = {&h->xh, &h->xh2};
    for (int k = 0; k < 2 && k < count; ++k) {
        TRY(Mb[k]->ensure(mb));
        TRY(bb[k]->ensure(sizeof(double) * (size_t)m));
        TRY(xb[k]->ensure(sizeof(double) * (size_t)ncols));
    }
    if (!h->cst) CK(cudaStreamCreateWithFlags(&h->cst, cudaStreamNonBlocking));
    for (int k = 0; k < 4; ++k)
        if (!h->cev[k]) CK(cudaEventCreateWithFlags(&h->cev[k], cudaEventDisableTiming));
    CK(cudaStreamSynchronize(h->st));                       // buffers free
    auto issue = [&](int k) -> lbfgsb_err {
        const int s2 = k & 1;
        if (k >= 2) CK(cudaStreamWaitEvent(h->cst, h->cev[2 + s2], 0));   // x* of problem k-2 is read back
        CK(cudaMemcpyAsync(Mb[s2]->p, M_hosts[k], mb, cudaMemcpyHostToDevice, h->cst));
        if (b_hosts && b_hosts[k])
            CK(cudaMemcpyAsync(bb[s2]->p, b_hosts[k], sizeof(double) * m, cudaMemcpyHostToDevice, h->cst));
        CK(cudaMemcpyAsync(xb[s2]->p, x_hosts[k], sizeof(double) * ncols, cudaMemcpyHostToDevice, h->cst));
        CK(cudaEventRecord(h->cev[s2], h->cst));
        return LBFGSB_OK;
    };
    TRY(issue(0));
    for (int k = 0; k < count; ++k) {
        const int s2 = k & 1;
        // buffer (k+1)&1 was last read by solve k-1, which has returned (lbfgsb_solve is host-synchronous)
        if (k + 1 < count) TRY(issue(k + 1));
        CK(cudaStreamWaitEvent(h->st, h->cev[s2], 0));
        lbfgsb_objective ob{};
        ob.kind = 0; ob.M = Mb[s2]->d(); ob.m = m; ob.ncols = ncols; ob.ld = m;
        ob.b = (b_hosts && b_hosts[k]) ? bb[s2]->d() : nullptr;
        TRY(lbfgsb_solve(h, &ob, xb[s2]->d(), tol, &res[k]));
        CK(cudaMemcpyAsync(x_hosts[k], xb[s2]->p, sizeof(double) * ncols, cudaMemcpyDeviceToHost, h->st));
        CK(cudaEventRecord(h->cev[2 + s2], h->st));
    }
    CK(cudaStreamSynchronize(h->st));
    CK(cudaStreamSynchronize(h->cst));
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ Alg. 4
static lbfgsb_err al_solve_general(lbfgsb_t* h, const lbfgsb_objective* obj, const al_constraints* cons,
                                   const al_opts& ao, double* x, double* lambda, double* mu, al_result* res);

extern "C" lbfgsb_err al_solve(lbfgsb_t* h, const lbfgsb_objective* obj, const al_constraints* cons,
                               const al_opts* opts, double* x, double* lambda, double* mu,
                               al_result* res)
{
    if (!h || !obj || !x) return fail(LBFGSB_ERR_ARG, "NULL handle, objective or x");
    al_opts ao;
    al_opts_default(&ao);
    if (opts) ao = *opts;
    if (!(ao.rho0 > 0) || !(ao.rho_factor > 1) || ao.max_outer < 1 || !(ao.rho_cap > 0))
        return fail(LBFGSB_ERR_ARG, "invalid al_opts");
    const int64_t neq64 = cons ? cons->m_eq : 0, nin64 = cons ? cons->p_in : 0;
    const int64_t mnl = cons ? cons->m_nl : 0, pnl = cons ? cons->p_nl : 0;
    if (neq64 < 0 || nin64 < 0 || mnl < 0 || pnl < 0) return fail(LBFGSB_ERR_DIM, "negative constraint count");
    if ((neq64 && (!cons->E || !cons->e)) || (nin64 && (!cons->G || !cons->hv)))
        return fail(LBFGSB_ERR_ARG, "constraint data missing");
    if ((mnl || pnl) && (!cons->hg || !cons->jtv)) return fail(LBFGSB_ERR_ARG, "nonlinear callbacks missing");
    if (ao.warm_start && ((neq64 + mnl > 0 && !lambda) || (nin64 + pnl > 0 && !mu)))
        return fail(LBFGSB_ERR_ARG, "warm start needs lambda / mu");
    if (h->sharded) return fail(LBFGSB_ERR_UNSUPPORTED, "al_solve is single-GPU");
    const bool fused = obj->kind == 0 && neq64 + nin64 <= MAXC && mnl + pnl == 0;
    if (!fused) {
        if (obj->kind == 2 || (obj->kind == 0 && obj->qp))
            return fail(LBFGSB_ERR_UNSUPPORTED, "general al_solve takes an LSQ or callback objective");
        return al_solve_general(h, obj, cons, ao, x, lambda, mu, res);
    }
    const int neq = (int)neq64, nin = (int)nin64;
    Group g;
    TRY(single_group(h, obj, g));
    Prob& P = g.Ps[0];
    P.n_eq = neq; P.n_in = nin;
    for (int k = 0; k < neq; ++k) P.Ecol[k] = cons->E + (int64_t)k * h->n;
    for (int k = 0; k < nin; ++k) P.Ecol[neq + k] = cons->G + (int64_t)k * h->n;
    set_sep(P);
    const double tol = h->o.tol;
    // x^0 = clip(0) (R19), lambda = 0, mu = 0, rho = rho0; warm start: as given
    if (!ao.warm_start) CK(cudaMemsetAsync(x, 0, sizeof(double) * h->n, h->st));
    double lam[MAXC] = {0}, rhs[MAXC] = {0};
    if (ao.warm_start) {
        for (int k = 0; k < neq; ++k) lam[k] = lambda[k];
        for (int k = 0; k < nin; ++k) lam[neq + k] = mu[k];
    }
    for (int k = 0; k < neq; ++k) rhs[k] = cons->e[k];
    for (int k = 0; k < nin; ++k) rhs[neq + k] = cons->hv[k];
    double rho = ao.rho0;
    auto set_al = [&]() {
        h->hc->rho = rho;
        std::memcpy(h->hc->lam, lam, sizeof lam);
        std::memcpy(h->hc->rhs, rhs, sizeof rhs);
    };
    auto viol = [&](const double* hv) {     // R21 (Birgin-Martinez measure)
        double v = 0.0;
        for (int k = 0; k < neq; ++k) v = std::fabs(hv[k]) > v ? std::fabs(hv[k]) : v;
        for (int k = 0; k < nin; ++k) {
            double t = -hv[neq + k];
            const double mr = lam[neq + k] / rho;
            if (mr < t) t = mr;
            v = std::fabs(t) > v ? std::fabs(t) : v;
        }
        return v;
    };
    // constraint values at x^0 (one f-evaluation pass)
    set_al();
    CK(cudaMemcpyAsync(P.x, x, sizeof(double) * h->n, cudaMemcpyDeviceToDevice, h->st));
    init_ctrl(h, tol);
    TRY(ctrl_to_dev(g));
    TRY(launch_fval(g, true));
    CK(cudaGetLastError());
    TRY(ctrl_to_host(g));
    CK(cudaMemcpyAsync(x, P.x, sizeof(double) * h->n, cudaMemcpyDeviceToDevice, h->st));
    double hv[MAXC];
    std::memcpy(hv, h->hc->hval, sizeof hv);
    double vprev = viol(hv);
    al_result R{};
    R.status = AL_MAX_OUTER;
    lbfgsb_result ir{};
    double* xs[1] = {x};
    for (int it = 0; it < ao.max_outer; ++it) {
        const double tin = 0.1 * vprev > tol ? 0.1 * vprev : tol;      // R22
        set_al();
        TRY(solve_group(g, xs, tin, &ir));                            // Alg. 4 line 5
        R.inner_iters_total += ir.iters;
        R.outer_iters = it + 1;
        R.pg_inf = ir.pg_inf;
        if (ir.status == LBFGSB_LINESEARCH_FAILURE) { R.status = AL_INNER_FAILURE; break; }
        std::memcpy(hv, h->hc->hval, sizeof hv);                       // h(x), g(x) at x*
        for (int k = 0; k < neq; ++k) lam[k] = lam[k] + rho * hv[k];   // line 6
        for (int k = 0; k < nin; ++k) {                                // line 7
            const double t = lam[neq + k] + rho * hv[neq + k];
            lam[neq + k] = t > 0.0 ? t : 0.0;
        }
        const double v = viol(hv);
        if (v > 0.5 * vprev) {                                         // line 8 (R20)
            rho = rho * ao.rho_factor;
            if (rho > ao.rho_cap) rho = ao.rho_cap;
        }
        vprev = v;
        if (ir.status == LBFGSB_CONVERGED && v <= ao.feas_tol && tin == tol) {
            R.status = LBFGSB_CONVERGED;
            break;
        }
    }
    R.f = h->hc->f_base;
    R.violation_inf = viol(hv);
    R.rho = rho;
    if (lambda) for (int k = 0; k < neq; ++k) lambda[k] = lam[k];
    if (mu) for (int k = 0; k < nin; ++k) mu[k] = lam[neq + k];
    if (res) *res = R;
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ Alg. 4, general constraints
// The general problem class through Eq. (3) as a callback
// objective of the inner Alg. 1 (solve_cb): L(x) = f(x) + penalty terms with
// f an LSQ objective (r = M~x - b by k_fwd, M~^T r by k_bwd) or the caller's
// callback, the linear blocks E^T x / G^T x by k_bwd and E w / G w by k_fwd
// (E as an n x K operator), the nonlinear blocks through hg / jtv, the
// stacked-vector parts in al.cu.  Every trial value is evaluated.
namespace {
struct GOp {                                // one operator for plain GEMV / GEMV^T passes
    Prob P{};
    DevBuf qpart, tick;
    lbfgsb_err init(const double* M, int64_t m, int64_t ncols, int64_t ld, const double* colscale, int split)
    {
        std::memset(&P, 0, sizeof P);
        P.m = m; P.ncols = ncols; P.ld = ld; P.M = M;
        P.colscale = colscale; P.split = split;
        P.n = split ? 2 * ncols : ncols;
        gemv_geometry(P);
        TRY(qpart.ensure(sizeof(double) * (size_t)P.m * (size_t)P.CC));
        TRY(tick.ensure(sizeof(unsigned) * (NTICKETS + TICKETS_EXTRA), true));
        P.qpart = qpart.d();
        P.tickets = static_cast<unsigned*>(tick.p);
        return LBFGSB_OK;
    }
    void fwd(const double* p, double* q, cudaStream_t st) { launch_fwd(P, st, FWD_P, p, q); }   // q = M~ p
    void bwd(const double* r, double* g, cudaStream_t st)                                       // g = M~^T r
    {
        P.rbuf[0] = const_cast<double*>(r);
        P.rbuf[1] = const_cast<double*>(r);
        launch_bwd(P, st, BWD_PLAIN, r, g);
    }
};

struct ALGen {
    lbfgsb_t* h = nullptr;
    const lbfgsb_objective* base = nullptr;
    const al_constraints* cons = nullptr;
    cudaStream_t st = nullptr;
    int64_t n = 0, m_eq = 0, p_in = 0, m_nl = 0, p_nl = 0, neq = 0, nin = 0;
    GOp opM, opE, opG;
    DevBuf r, lam, mu, hv, gv, weq, win, tmp, scal, erhs, hrhs;
    double* sh = nullptr;                   // pinned host scalars [base f, penalty, violation]
    double rho = 1.0;
    bool cb_fail = false;

    // stacked constraint values at x: hv = [E^T x - e; h_nl(x)], gv = [G^T x - hv; g_nl(x)]
    int values(const double* x)
    {
        if (m_eq) { opE.bwd(x, hv.d(), st); launch_sub(m_eq, hv.d(), erhs.d(), st); }
        if (p_in) { opG.bwd(x, gv.d(), st); launch_sub(p_in, gv.d(), hrhs.d(), st); }
        if (m_nl + p_nl) return cons->hg(cons->user, x, hv.d() + m_eq, gv.d() + p_in, st);
        return 0;
    }
    // base objective value (into sh[0] after a sync, or *fcb for a callback) and gradient g
    int base_fg(const double* x, double* g, double* fcb)
    {
        if (base->kind == 1) return base->fg(base->user, x, g, fcb, st);
        opM.fwd(x, r.d(), st);                                       // r = M~ x
        if (base->b) launch_sub(base->m, r.d(), base->b, st);       // - b
        opM.bwd(r.d(), g, st);                                       // g = M~^T r
        launch_lsq_value(base->m, r.d(), n, x, base->c, base->delta, g, scal.d(), st);
        return 0;
    }
};

// callback of the inner solve: f = L(x), g = grad L(x)
int32_t al_gen_fg(void* user, const double* x, double* g, double* f_host, void* /*stream*/)
{
    ALGen& A = *static_cast<ALGen*>(user);
    double fcb = 0.0;
    if (A.base_fg(x, g, &fcb) != 0 || A.values(x) != 0) { A.cb_fail = true; return 1; }
    launch_al_terms(A.neq, A.hv.d(), A.lam.d(), A.nin, A.gv.d(), A.mu.d(), A.rho, A.weq.d(), A.win.d(),
                    A.scal.d() + 1, A.st);
    if (A.m_eq) { A.opE.fwd(A.weq.d(), A.tmp.d(), A.st); launch_axpy(A.n, A.tmp.d(), g, A.st); }
    if (A.p_in) { A.opG.fwd(A.win.d(), A.tmp.d(), A.st); launch_axpy(A.n, A.tmp.d(), g, A.st); }
    if (A.m_nl + A.p_nl) {
        if (A.cons->jtv(A.cons->user, x, A.weq.d() + A.m_eq, A.win.d() + A.p_in, A.tmp.d(), A.st) != 0) {
            A.cb_fail = true;
            return 1;
        }
        launch_axpy(A.n, A.tmp.d(), g, A.st);
    }
    if (cudaMemcpyAsync(A.sh, A.scal.d(), sizeof(double) * 2, cudaMemcpyDeviceToHost, A.st) != cudaSuccess ||
        cudaStreamSynchronize(A.st) != cudaSuccess)
        return 1;
    *f_host = (A.base->kind == 1 ? fcb : A.sh[0]) + A.sh[1];
    return 0;
}
}  // namespace

static lbfgsb_err al_solve_general(lbfgsb_t* h, const lbfgsb_objective* obj, const al_constraints* cons,
                                   const al_opts& ao, double* x, double* lambda, double* mu, al_result* res)
{
    ALGen A;
    A.h = h; A.base = obj; A.cons = cons; A.st = h->st; A.n = h->n;
    A.m_eq = cons ? cons->m_eq : 0; A.p_in = cons ? cons->p_in : 0;
    A.m_nl = cons ? cons->m_nl : 0; A.p_nl = cons ? cons->p_nl : 0;
    A.neq = A.m_eq + A.m_nl; A.nin = A.p_in + A.p_nl;
    const int64_t n = h->n;
    cudaStream_t st = h->st;
    if (obj->kind == 0) {
        if ((obj->split ? 2 * obj->ncols : obj->ncols) != n) return fail(LBFGSB_ERR_DIM, "objective size != n");
        TRY(A.opM.init(obj->M, obj->m, obj->ncols, obj->ld, obj->colscale, obj->split));
        TRY(A.r.ensure(sizeof(double) * (size_t)obj->m));
    }
    if (A.m_eq) TRY(A.opE.init(cons->E, n, A.m_eq, n, nullptr, 0));
    if (A.p_in) TRY(A.opG.init(cons->G, n, A.p_in, n, nullptr, 0));
    const size_t be = sizeof(double) * (size_t)(A.neq > 0 ? A.neq : 1);
    const size_t bi = sizeof(double) * (size_t)(A.nin > 0 ? A.nin : 1);
    TRY(A.lam.ensure(be, true)); TRY(A.hv.ensure(be, true)); TRY(A.weq.ensure(be, true));
    TRY(A.mu.ensure(bi, true)); TRY(A.gv.ensure(bi, true)); TRY(A.win.ensure(bi, true));
    TRY(A.tmp.ensure(sizeof(double) * (size_t)n));
    TRY(A.scal.ensure(sizeof(double) * 4, true));
    if (A.m_eq) {
        TRY(A.erhs.ensure(sizeof(double) * (size_t)A.m_eq));
        CK(cudaMemcpyAsync(A.erhs.p, cons->e, sizeof(double) * A.m_eq, cudaMemcpyHostToDevice, st));
    }
    if (A.p_in) {
        TRY(A.hrhs.ensure(sizeof(double) * (size_t)A.p_in));
        CK(cudaMemcpyAsync(A.hrhs.p, cons->hv, sizeof(double) * A.p_in, cudaMemcpyHostToDevice, st));
    }
    CK(cudaMallocHost(&A.sh, sizeof(double) * 4));
    struct PinFree { double* p; ~PinFree() { if (p) cudaFreeHost(p); } } pin_guard{A.sh};
    // x^0 = clip(0), lambda = mu = 0 (R19); warm start: the given x (clipped), lambda, mu
    if (!ao.warm_start) {
        CK(cudaMemsetAsync(x, 0, sizeof(double) * n, st));
    } else {
        if (A.neq) CK(cudaMemcpyAsync(A.lam.p, lambda, be, cudaMemcpyHostToDevice, st));
        if (A.nin) CK(cudaMemcpyAsync(A.mu.p, mu, bi, cudaMemcpyHostToDevice, st));
    }
    lbfgsb_objective cbo{};
    cbo.kind = 1;
    cbo.fg = al_gen_fg;
    cbo.user = &A;
    {
        Prob P;
        TRY(make_prob(h, &cbo, P));
        CK(cudaMemcpyAsync(P.x, x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        launch_clip(P, st);
        CK(cudaMemcpyAsync(x, P.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    }
    double rho = ao.rho0;
    auto violation = [&](double* v) -> lbfgsb_err {
        launch_al_violation(A.neq, A.hv.d(), A.nin, A.gv.d(), A.mu.d(), rho, A.scal.d() + 2, st);
        CK(cudaMemcpyAsync(A.sh + 2, A.scal.d() + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        *v = A.sh[2];
        return LBFGSB_OK;
    };
    if (A.values(x) != 0) return fail(LBFGSB_ERR_CALLBACK, "constraint callback failed at x0");
    double vprev = 0.0;
    TRY(violation(&vprev));
    const double tol = h->o.tol;
    al_result R{};
    R.status = AL_MAX_OUTER;
    for (int it = 0; it < ao.max_outer; ++it) {
        const double tin = 0.1 * vprev > tol ? 0.1 * vprev : tol;          // R22
        A.rho = rho;
        lbfgsb_result ir{};
        lbfgsb_err e = solve_cb(h, &cbo, x, tin, &ir);                     // Alg. 4 line 5
        if (e != LBFGSB_OK) return A.cb_fail ? fail(LBFGSB_ERR_CALLBACK, "objective / constraint callback failed") : e;
        R.inner_iters_total += ir.iters;
        R.outer_iters = it + 1;
        R.pg_inf = ir.pg_inf;
        if (ir.status == LBFGSB_LINESEARCH_FAILURE) { R.status = AL_INNER_FAILURE; break; }
        if (A.values(x) != 0) return fail(LBFGSB_ERR_CALLBACK, "constraint callback failed");
        launch_al_update(A.neq, A.hv.d(), A.lam.d(), A.nin, A.gv.d(), A.mu.d(), rho, A.scal.d() + 2, st);  // lines 6-7
        CK(cudaMemcpyAsync(A.sh + 2, A.scal.d() + 2, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        const double v = A.sh[2];
        if (v > 0.5 * vprev) {                                             // line 8 (R20)
            rho = rho * ao.rho_factor;
            if (rho > ao.rho_cap) rho = ao.rho_cap;
        }
        vprev = v;
        if (ir.status == LBFGSB_CONVERGED && v <= ao.feas_tol && tin == tol) {
            R.status = LBFGSB_CONVERGED;
            break;
        }
    }
    // the original objective f(x) (no AL terms) and the final violation
    {
        double fcb = 0.0;
        if (A.base_fg(x, A.tmp.d(), &fcb) != 0) return fail(LBFGSB_ERR_CALLBACK, "objective callback failed");
        CK(cudaMemcpyAsync(A.sh, A.scal.d(), sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        R.f = obj->kind == 1 ? fcb : A.sh[0];
        if (A.values(x) != 0) return fail(LBFGSB_ERR_CALLBACK, "constraint callback failed");
        TRY(violation(&R.violation_inf));
    }
    R.rho = rho;
    if (lambda && A.neq) CK(cudaMemcpyAsync(lambda, A.lam.p, sizeof(double) * A.neq, cudaMemcpyDeviceToHost, st));
    if (mu && A.nin) CK(cudaMemcpyAsync(mu, A.mu.p, sizeof(double) * A.nin, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (res) *res = R;
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ Alg. 4, marginal constraints
static const bool g_al_trace = std::getenv("LBFGSB_AL_TRACE") != nullptr;   // per-outer stderr line

// Joint probability / regularised OT: the m + n
// equalities h(P) = [P 1 - u; P^T 1 - v] with device multipliers; otherwise
// the rules of al_solve (R19-R22; the violation of equalities is ||h||_inf).
extern "C" lbfgsb_err al_solve_transport(lbfgsb_t* h, const lbfgsb_objective* obj, const double* u,
                                         const double* v, const al_opts* opts, double* x,
                                         double* lambda, al_result* res)
{
    if (!h || !obj || !x || !u || !v) return fail(LBFGSB_ERR_ARG, "NULL handle, objective, u, v or x");
    if (obj->kind != 2) return fail(LBFGSB_ERR_ARG, "al_solve_transport needs a transport objective");
    al_opts ao;
    al_opts_default(&ao);
    if (opts) ao = *opts;
    if (!(ao.rho0 > 0) || !(ao.rho_factor > 1) || ao.max_outer < 1)
        return fail(LBFGSB_ERR_ARG, "invalid al_opts");
    Group g;
    TRY(single_group(h, obj, g));
    Prob& P = g.Ps[0];
    cudaStream_t st = h->st;
    const int64_t K = P.tm + P.tn;
    CK(cudaMemcpyAsync(h->te.d(), u, sizeof(double) * P.tm, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(h->te.d() + P.tm, v, sizeof(double) * P.tn, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemsetAsync(P.tlam, 0, sizeof(double) * K, st));            // lambda^0 = 0
    CK(cudaMemsetAsync(x, 0, sizeof(double) * h->n, st));              // x^0 = clip(0) (R19)
    const double tol = h->o.tol;
    double rho = ao.rho0;
    double* vout = h->tvout.d();
    auto violation = [&](int update, double& out) -> lbfgsb_err {
        launch_tviol(P, st, rho, update, vout);
        CK(cudaGetLastError());
        CK(cudaMemcpyAsync(&out, vout, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return LBFGSB_OK;
    };
    h->hc->rho = rho;
    CK(cudaMemcpyAsync(P.x, x, sizeof(double) * h->n, cudaMemcpyDeviceToDevice, st));
    init_ctrl(h, tol);
    TRY(ctrl_to_dev(g));
    TRY(launch_fval(g, true));
    CK(cudaGetLastError());
    TRY(ctrl_to_host(g));
    CK(cudaMemcpyAsync(x, P.x, sizeof(double) * h->n, cudaMemcpyDeviceToDevice, st));
    double vprev = 0.0;
    TRY(violation(0, vprev));
    al_result R{};
    R.status = AL_MAX_OUTER;
    lbfgsb_result ir{};
    double* xs[1] = {x};
    double vlast = vprev;
    for (int it = 0; it < ao.max_outer; ++it) {
        const double tin = 0.1 * vprev > tol ? 0.1 * vprev : tol;      // R22
        h->hc->rho = rho;
        TRY(solve_group(g, xs, tin, &ir));                            // Alg. 4 line 5
        R.inner_iters_total += ir.iters;
        R.outer_iters = it + 1;
        R.pg_inf = ir.pg_inf;
        R.f = h->hc->f_base;
        if (ir.status == LBFGSB_LINESEARCH_FAILURE) { R.status = AL_INNER_FAILURE; break; }
        double vv = 0.0;
        TRY(violation(1, vv));                                         // line 6: lam += rho h
        vlast = vv;
        if (g_al_trace)
            std::fprintf(stderr, "[al_transport] outer %d rho %.3e tol_in %.3e inner %lld status %d "
                         "pg %.3e viol %.3e f %.15g n_fg %lld n_bt %lld fallbacks %lld %.3fs\n", it, rho,
                         tin, (long long)ir.iters, ir.status, ir.pg_inf, vv, h->hc->f_base,
                         (long long)ir.n_fg, (long long)ir.n_backtracks, (long long)ir.n_fallbacks,
                         ir.seconds);
        if (vv > 0.5 * vprev) {                                        // line 8 (R20)
            rho = rho * ao.rho_factor;
            if (rho > ao.rho_cap) rho = ao.rho_cap;
        }
        vprev = vv;
        if (ir.status == LBFGSB_CONVERGED && vv <= ao.feas_tol && tin == tol) {
            R.status = LBFGSB_CONVERGED;
            break;
        }
    }
    R.violation_inf = vlast;
    R.rho = rho;
    if (lambda) CK(cudaMemcpyAsync(lambda, P.tlam, sizeof(double) * K, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    if (res) *res = R;
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ N3: Cauchy point op
extern "C" lbfgsb_err lbfgsb_op_cauchy_point(lbfgsb_t* h, const double* x, const double* g, int32_t nh,
                                             const double* S, const double* Y, double theta, double* xcp,
                                             double* c, int64_t* passed, double* scan_ms)
{
    if (!h || !x || !g || !xcp) return fail(LBFGSB_ERR_ARG, "NULL handle, x, g or xcp");
    if (nh < 0 || nh > 8 || (nh > 0 && (!S || !Y))) return fail(LBFGSB_ERR_ARG, "0 <= nh <= 8 pairs required");
    if (h->sharded) return fail(LBFGSB_ERR_UNSUPPORTED, "single-GPU op");
    const int64_t n = h->n;
    const size_t nb = sizeof(double) * (size_t)n;
    TRY(h->cp_d.ensure(nb)); TRY(h->cp_t.ensure(nb)); TRY(h->cp_heap.ensure(2 * nb));
    TRY(h->cp_part.ensure(sizeof(double) * (size_t)(2 * sm_count()) * cauchy_nr()));
    TRY(h->cp_red.ensure(sizeof(double) * (size_t)cauchy_nr()));
    TRY(h->cp_scal.ensure(sizeof(double) * 32));
    TRY(h->cp_ticket.ensure(sizeof(unsigned) * 4, true));
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (scan_ms) { CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1)); }
    if (launch_cauchy(n, x, g, h->l.d(), h->u.d(), nh, S, Y, theta, h->cp_d.d(), h->cp_t.d(), xcp,
                      h->cp_part.d(), h->cp_red.d(), static_cast<unsigned*>(h->cp_ticket.p), h->cp_heap.d(),
                      h->cp_scal.d(), h->st, e0, e1))
        return fail(LBFGSB_ERR_ARG, "bad history length");
    CK(cudaGetLastError());
    double sc[32];
    CK(cudaMemcpyAsync(sc, h->cp_scal.d(), sizeof sc, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    if (passed) *passed = (int64_t)sc[1];
    if (c) for (int j = 0; j < 2 * nh; ++j) c[j] = sc[2 + j];
    if (scan_ms) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        *scan_ms = ms;
        cudaEventDestroy(e0); cudaEventDestroy(e1);
    }
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ N4: batched small problems
extern "C" lbfgsb_err lbfgsb_solve_batched_lsq(int32_t batch, int64_t m, int64_t n, const double* M,
                                               const double* b, const double* lower, const double* upper,
                                               double* x, int32_t m_hist, const lbfgsb_opts* opts,
                                               double tol, void* cuda_stream, lbfgsb_result* res)
{
    if (batch < 0 || m <= 0 || n <= 0) return fail(LBFGSB_ERR_DIM, "bad batch shape");
    if (batch == 0) return LBFGSB_OK;
    if (!M || !b || !x || !res) return fail(LBFGSB_ERR_ARG, "NULL M, b, x or res");
    if (m_hist < 1 || m_hist > LBFGSB_MAX_HIST) return fail(LBFGSB_ERR_ARG, "bad m_hist");
    lbfgsb_opts o;
    lbfgsb_opts_default(&o);
    if (opts) o = *opts;
    if (!opts_valid(o) || !(tol >= 0)) return fail(LBFGSB_ERR_ARG, "invalid option value");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        return fail(LBFGSB_ERR_CUDA, "no CUDA device available (the library has no CPU path)");
    init_kernels();
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    if (lower || upper) {                                   // l <= u, no NaN
        int* bad = nullptr;
        CK(cudaMallocAsync(reinterpret_cast<void**>(&bad), sizeof(int), st));
        CK(cudaMemsetAsync(bad, 0, sizeof(int), st));
        k_check_bounds<<<256, 256, 0, st>>>(lower, upper, (int64_t)batch * n, bad);
        CK(cudaGetLastError());
        int hbad = 0;
        CK(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaFreeAsync(bad, st));
        CK(cudaStreamSynchronize(st));
        if (hbad) return fail(LBFGSB_ERR_BOUNDS, "l_i > u_i or NaN bound");
    }
    lbfgsb_result* dres = nullptr;
    CK(cudaMallocAsync(reinterpret_cast<void**>(&dres), sizeof(lbfgsb_result) * (size_t)batch, st));
    auto t0 = std::chrono::steady_clock::now();
    const int rc = launch_batch(batch, m, n, M, b, lower, upper, x, m_hist, o, tol > 0 ? tol : o.tol, dres, st);
    if (rc) { cudaFreeAsync(dres, st); return fail(LBFGSB_ERR_DIM, "problem too large for one CTA's shared memory"); }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(res, dres, sizeof(lbfgsb_result) * (size_t)batch, cudaMemcpyDeviceToHost, st));
    CK(cudaFreeAsync(dres, st));
    CK(cudaStreamSynchronize(st));
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (int32_t i = 0; i < batch; ++i) res[i].seconds = secs;
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ N3: the original L-BFGS-B
// Host-driven loop (one synchronisation per step, as the baseline ran):
// projected-gradient test; generalized Cauchy point (cauchy.cu: parallel
// breakpoints, ONE-thread breakpoint loop); direct primal subspace
// minimisation and backtrack (original.cu); Armijo along d = xbar - x with
// the same trial machinery as lbfgsb_op_trials; pair kept iff s^T y > eps
// y^T y; theta = y^T y / s^T y.  Mirrors orc_lbfgsb_original.
extern "C" lbfgsb_err lbfgsb_solve_original(lbfgsb_t* h, const lbfgsb_objective* obj, double* x_user, double tol,
                                            lbfgsb_result* res, double* cp_ms)
{
    if (!h || !obj || !x_user) return fail(LBFGSB_ERR_ARG, "NULL handle, objective or x");
    if (obj->kind != 0 || obj->qp || obj->c || obj->delta != 0.0)
        return fail(LBFGSB_ERR_UNSUPPORTED, "the original L-BFGS-B runs plain least squares (no c, delta)");
    if (h->sharded) return fail(LBFGSB_ERR_UNSUPPORTED, "single-GPU");
    if (h->mh > 8) return fail(LBFGSB_ERR_UNSUPPORTED, "m_hist <= 8");
    auto t0 = std::chrono::steady_clock::now();
    const double tl = tol > 0 ? tol : h->o.tol;
    Prob P;
    TRY(make_prob(h, obj, P));
    set_sep(P);
    cudaStream_t st = h->st;
    const int64_t n = h->n, m = P.m, mh = h->mh;
    const size_t nb = sizeof(double) * (size_t)n, mb = sizeof(double) * (size_t)m;
    TRY(h->og_S.ensure(nb * mh)); TRY(h->og_Y.ensure(nb * mh)); TRY(h->og_s.ensure(nb)); TRY(h->og_y.ensure(nb));
    TRY(h->og_rc.ensure(nb)); TRY(h->og_du.ensure(nb)); TRY(h->og_d.ensure(nb)); TRY(h->og_gn.ensure(nb));
    TRY(h->og_r.ensure(mb)); TRY(h->og_q.ensure(mb));
    TRY(h->og_M.ensure(sizeof(double) * 300)); TRY(h->og_z.ensure(sizeof(double) * 32));
    TRY(h->og_out.ensure(sizeof(double) * 8));
    TRY(h->og_part.ensure(sizeof(double) * (size_t)(2 * sm_count()) * (orig_nr() > 4 ? orig_nr() : 4)));
    TRY(h->og_red.ensure(sizeof(double) * (size_t)orig_nr()));
    TRY(h->og_ticket.ensure(sizeof(unsigned) * 8, true));
    TRY(h->cp_d.ensure(nb)); TRY(h->cp_t.ensure(nb)); TRY(h->cp_xcp.ensure(nb)); TRY(h->cp_heap.ensure(2 * nb));
    TRY(h->cp_part.ensure(sizeof(double) * (size_t)(2 * sm_count()) * cauchy_nr()));
    TRY(h->cp_red.ensure(sizeof(double) * (size_t)cauchy_nr()));
    TRY(h->cp_scal.ensure(sizeof(double) * 32));
    TRY(h->cp_ticket.ensure(sizeof(unsigned) * 4, true));
    double* x = P.x;
    double* g = P.g;
    double* gn = h->og_gn.d();
    double* r = h->og_r.d();
    double* q = h->og_q.d();
    CK(cudaMemcpyAsync(x, x_user, nb, cudaMemcpyDeviceToDevice, st));
    launch_clip(P, st);
    OrigArgs A{};
    A.n = n; A.m = m; A.l = P.l; A.u = P.u; A.xc = h->cp_xcp.d();
    A.S = h->og_S.d(); A.Y = h->og_Y.d(); A.Mm = h->og_M.d();
    A.rc = h->og_rc.d(); A.du = h->og_du.d(); A.d = h->og_d.d();
    A.part = h->og_part.d(); A.red = h->og_red.d(); A.ticket = static_cast<unsigned*>(h->og_ticket.p);
    A.z = h->og_z.d(); A.out = h->og_out.d();
    double out[8];
    auto read_out = [&]() -> lbfgsb_err {
        CK(cudaMemcpyAsync(out, A.out, sizeof out, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        return LBFGSB_OK;
    };
    // f, r = M~x - b, g
    auto eval = [&](double* gout, double& f) -> lbfgsb_err {
        launch_fwd(P, st, FWD_P, x, r);
        A.x = x;
        launch_orig_residual(A, r, P.b, st);
        launch_bwd(P, st, BWD_PLAIN, r, gout);
        CK(cudaGetLastError());
        TRY(read_out());
        f = 0.5 * out[5];
        return LBFGSB_OK;
    };
    double f = 0.0;
    TRY(eval(g, f));
    int hp = 0;
    double theta = 1.0, tcp = 0.0;
    long long k = 0, nfg = 1, nbt = 0, nfb = 0;
    int status = S_MAX_ITERS;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    for (;;) {
        A.x = x; A.g = g; A.h = hp; A.theta = theta;
        launch_orig_pg(A, st);
        TRY(read_out());
        if (out[2] <= tl) { status = S_CONVERGED; break; }
        if (k >= h->o.max_iters) { status = S_MAX_ITERS; break; }
        // generalized Cauchy point (the single-thread loop is bracketed by e0 / e1)
        if (launch_cauchy(n, x, g, P.l, P.u, hp, A.S, A.Y, theta, h->cp_d.d(), h->cp_t.d(), h->cp_xcp.d(),
                          h->cp_part.d(), h->cp_red.d(), static_cast<unsigned*>(h->cp_ticket.p), h->cp_heap.d(),
                          h->cp_scal.d(), st, e0, e1, h->og_M.d()))
            return fail(LBFGSB_ERR_ARG, "history too long");
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        tcp += ms;
        // subspace minimisation, backtrack, direction, g^T d
        launch_orig_subspace(A, st);
        CK(cudaGetLastError());
        TRY(read_out());
        const double gd = out[1];
        if (!(gd < 0.0)) {
            if (hp == 0) { status = S_LS_FAIL; break; }
            hp = 0; theta = 1.0; ++nfb;
            continue;
        }
        // Armijo on the carried residual along d (alpha = 1, shrink, ...)
        launch_fwd(P, st, FWD_P, A.d, q);
        double alpha = 1.0, fnew = f;
        bool acc = false;
        for (int t0b = 0; t0b <= h->o.max_backtracks && !acc; t0b += KT) {
            init_ctrl(h, tl);
            h->hc->alpha0 = alpha;
            h->hc->rho = 1.0;
            TRY(ctrl_to_dev(h, st));
            Prob PT = P;
            PT.x = x;
            launch_sep(PT, st, SEP_OP, A.d);
            launch_ls(PT, st, LS_OP, r, q, h->fout.d(), KT);
            double ft[KT];
            CK(cudaMemcpyAsync(ft, h->fout.p, sizeof ft, cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            double a = alpha;
            for (int t = 0; t < KT && t0b + t <= h->o.max_backtracks; ++t) {
                if (t > 0) a = a * h->o.shrink;
                ++nfg;
                if (ft[t] <= f + h->o.c1 * a * gd) { acc = true; alpha = a; fnew = ft[t]; break; }
                ++nbt;
            }
            if (!acc) alpha = a * h->o.shrink;
        }
        if (!acc) {
            if (hp == 0) { status = S_LS_FAIL; break; }
            hp = 0; theta = 1.0; ++nfb;
            continue;
        }
        launch_orig_step(A, x, A.d, r, q, alpha, h->og_s.d(), st);
        launch_bwd(P, st, BWD_PLAIN, r, gn);
        launch_orig_pair(A, gn, g, h->og_s.d(), h->og_y.d(), st);
        CK(cudaGetLastError());
        TRY(read_out());
        const double sy = out[3], yy = out[4];
        if (sy > h->o.eps * yy) {
            if (hp == mh) {                                      // drop the oldest pair
                for (int i = 1; i < mh; ++i) {
                    CK(cudaMemcpyAsync(h->og_S.d() + (int64_t)(i - 1) * n, h->og_S.d() + (int64_t)i * n, nb,
                                       cudaMemcpyDeviceToDevice, st));
                    CK(cudaMemcpyAsync(h->og_Y.d() + (int64_t)(i - 1) * n, h->og_Y.d() + (int64_t)i * n, nb,
                                       cudaMemcpyDeviceToDevice, st));
                }
                hp = mh - 1;
            }
            CK(cudaMemcpyAsync(h->og_S.d() + (int64_t)hp * n, h->og_s.d(), nb, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(h->og_Y.d() + (int64_t)hp * n, h->og_y.d(), nb, cudaMemcpyDeviceToDevice, st));
            ++hp;
            theta = yy / sy;
        }
        CK(cudaMemcpyAsync(g, gn, nb, cudaMemcpyDeviceToDevice, st));
        f = fnew;
        ++k;
    }
    // final refresh: r = M~x - b, f, g, pg
    double ff = 0.0;
    TRY(eval(g, ff));
    A.x = x; A.g = g;
    launch_orig_pg(A, st);
    TRY(read_out());
    CK(cudaMemcpyAsync(x_user, x, nb, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    cudaEventDestroy(e0); cudaEventDestroy(e1);
    if (res) {
        std::memset(res, 0, sizeof *res);
        res->f = ff;                                             // 1/2 ||r||^2 (plain LSQ)
        res->pg_inf = out[2];
        res->iters = k;
        res->n_fg = nfg;
        res->n_backtracks = nbt;
        res->n_fallbacks = nfb;
        res->status = status;
        res->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (cp_ms) *cp_ms = tcp;
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ sharded (NCCL)
extern "C" lbfgsb_err lbfgsb_nccl_unique_id(void* out)
{
    if (!out) return fail(LBFGSB_ERR_ARG, "out is NULL");
#ifdef LBFGSB_WITH_NCCL
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId id;
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return fail(LBFGSB_ERR_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof id);
    return LBFGSB_OK;
#else
    return fail(LBFGSB_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

extern "C" lbfgsb_err lbfgsb_create_sharded(int64_t n_local, int64_t n_global, int32_t m_hist,
                                            const double* lower_local, const double* upper_local,
                                            const lbfgsb_opts* opts, void* cuda_stream,
                                            const void* nccl_unique_id, int32_t rank, int32_t nranks,
                                            lbfgsb_t** out)
{
    if (!out || !nccl_unique_id) return fail(LBFGSB_ERR_ARG, "NULL out or unique id");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(LBFGSB_ERR_ARG, "bad rank/nranks");
    if (n_global < n_local) return fail(LBFGSB_ERR_DIM, "n_global < n_local");
#ifdef LBFGSB_WITH_NCCL
    lbfgsb_t* h = nullptr;
    TRY(create_common(n_local, m_hist, lower_local, upper_local, opts, cuda_stream, &h));
    ncclUniqueId id;
    std::memcpy(&id, nccl_unique_id, sizeof id);
    ncclResult_t r = ncclCommInitRank(&h->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        lbfgsb_destroy(h);
        return fail(LBFGSB_ERR_NCCL, "ncclCommInitRank: %s", ncclGetErrorString(r));
    }
    h->comm_owned = true;
    h->sharded = true;          // sharded protocol even for a 1-rank communicator
    h->nranks = nranks;
    h->rank = rank;
    h->n_global = n_global;
    *out = h;
    return LBFGSB_OK;
#else
    (void)n_local; (void)m_hist; (void)lower_local; (void)upper_local; (void)opts; (void)cuda_stream;
    return fail(LBFGSB_ERR_UNSUPPORTED, "built without NCCL");
#endif
}

// ------------------------------------------------------------------ sharded (P2P exchange)
// Mailbox of one rank: header + the four gathered sections for m <= m_max
// (layout in impl.cuh mb_off).  cudaMalloc (not the
// stream-ordered allocator) so that it can be exported with CUDA IPC.
static lbfgsb_err alloc_mailbox(lbfgsb_t* h, int nranks, int64_t m_max)
{
    if (nranks < 1 || nranks > P2P_MAXR) return fail(LBFGSB_ERR_ARG, "P2P exchange: 1 <= nranks <= %d", P2P_MAXR);
    if (m_max < 1) return fail(LBFGSB_ERR_DIM, "m_max < 1");
    const size_t per = (size_t)(m_max + (int64_t)KT * NSEP + 4 + GRAM_STRIDE + 4);
    const size_t bytes = sizeof(double) * (MB_HDR + (size_t)nranks * per);
    if (h->mb) { cudaFree(h->mb); h->mb = nullptr; }
    cudaError_t e = cudaMalloc(&h->mb, bytes);
    if (e == cudaSuccess) e = cudaMemset(h->mb, 0, bytes);
    if (e != cudaSuccess) {
        if (h->mb) cudaFree(h->mb);
        h->mb = nullptr;
        return fail(LBFGSB_ERR_OOM, "mailbox cudaMalloc(%zu): %s", bytes, cudaGetErrorString(e));
    }
    TRY(h->p2p_tgt.ensure(sizeof(unsigned long long) * MB_HDR, true));
    CK(cudaMemset(h->p2p_tgt.p, 0, sizeof(unsigned long long) * MB_HDR));
    h->mb_mmax = m_max;
    h->mb_nranks = nranks;
    h->mb_bytes = bytes;
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_create_sharded_p2p(int64_t n_local, int64_t n_global, int32_t m_hist,
                                                const double* lower_local, const double* upper_local,
                                                const lbfgsb_opts* opts, void* cuda_stream, int32_t rank,
                                                int32_t nranks, int64_t m_max, lbfgsb_t** out)
{
    if (!out) return fail(LBFGSB_ERR_ARG, "NULL out");
    *out = nullptr;
    if (nranks < 1 || nranks > P2P_MAXR || rank < 0 || rank >= nranks)
        return fail(LBFGSB_ERR_ARG, "bad rank/nranks (P2P exchange: nranks <= %d)", P2P_MAXR);
    if (n_global < n_local) return fail(LBFGSB_ERR_DIM, "n_global < n_local");
    lbfgsb_t* h = nullptr;
    TRY(create_common(n_local, m_hist, lower_local, upper_local, opts, cuda_stream, &h));
    lbfgsb_err e = alloc_mailbox(h, nranks, m_max);
    if (e != LBFGSB_OK) { lbfgsb_destroy(h); return e; }
    h->p2p = true;
    h->sharded = true;
    h->nranks = nranks;
    h->rank = rank;
    h->n_global = n_global;
    h->peer_mb[rank] = h->mb;
    *out = h;
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_p2p_ipc_handle(lbfgsb_t* h, void* out)
{
    if (!h || !out || !h->p2p || !h->mb) return fail(LBFGSB_ERR_ARG, "not a P2P handle");
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "cudaIpcMemHandle_t size");
    cudaIpcMemHandle_t ih;
    CK(cudaIpcGetMemHandle(&ih, h->mb));
    std::memcpy(out, &ih, sizeof ih);
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_p2p_open(lbfgsb_t* h, const void* handles)
{
    if (!h || !handles || !h->p2p) return fail(LBFGSB_ERR_ARG, "not a P2P handle");
    for (int r = 0; r < h->nranks; ++r) {
        if (r == h->rank) { h->peer_mb[r] = h->mb; continue; }
        if (h->peer_ipc[r] && h->peer_mb[r]) { cudaIpcCloseMemHandle(h->peer_mb[r]); h->peer_ipc[r] = false; }
        cudaIpcMemHandle_t ih;
        std::memcpy(&ih, static_cast<const char*>(handles) + 64 * (size_t)r, sizeof ih);
        void* p = nullptr;
        cudaError_t e = cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) return fail(LBFGSB_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", r,
                                          cudaGetErrorString(e));
        h->peer_mb[r] = p;
        h->peer_ipc[r] = true;
    }
    return LBFGSB_OK;
}

// Wire the n_local handles a process hosts (logical ranks of one P2P group,
// any subset of 0..nranks-1) to every mailbox: the local ones directly, the
// others through CUDA IPC, each remote mailbox mapped ONCE per process (the
// mapping is owned, and closed, by hs[0]; destroy the group's handles together).
extern "C" lbfgsb_err lbfgsb_p2p_open_group(lbfgsb_t* const* hs, int32_t n_local, const void* handles)
{
    if (!hs || n_local < 1 || !handles) return fail(LBFGSB_ERR_ARG, "bad arguments");
    const int R = hs[0]->nranks;
    void* local[P2P_MAXR] = {};
    for (int p = 0; p < n_local; ++p) {
        if (!hs[p] || !hs[p]->p2p || !hs[p]->mb || hs[p]->nranks != R)
            return fail(LBFGSB_ERR_ARG, "local rank %d: not a P2P handle of the group", p);
        if (local[hs[p]->rank]) return fail(LBFGSB_ERR_ARG, "logical rank %d hosted twice", hs[p]->rank);
        local[hs[p]->rank] = hs[p]->mb;
    }
    for (int p = 0; p < n_local; ++p)
        for (int r = 0; r < R; ++r)
            if (hs[p]->peer_ipc[r] && hs[p]->peer_mb[r]) {
                cudaIpcCloseMemHandle(hs[p]->peer_mb[r]);
                hs[p]->peer_ipc[r] = false;
                hs[p]->peer_mb[r] = nullptr;
            }
    for (int r = 0; r < R; ++r) {
        void* ptr = local[r];
        bool ipc = false;
        if (!ptr) {
            cudaIpcMemHandle_t ih;
            std::memcpy(&ih, static_cast<const char*>(handles) + 64 * (size_t)r, sizeof ih);
            cudaError_t e = cudaIpcOpenMemHandle(&ptr, ih, cudaIpcMemLazyEnablePeerAccess);
            if (e != cudaSuccess) return fail(LBFGSB_ERR_CUDA, "cudaIpcOpenMemHandle(rank %d): %s", r,
                                              cudaGetErrorString(e));
            ipc = true;
        }
        for (int p = 0; p < n_local; ++p) {
            hs[p]->peer_mb[r] = ptr;
            hs[p]->peer_ipc[r] = ipc && p == 0;
        }
    }
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_p2p_connect_local(lbfgsb_t* const* hs, int32_t nranks, int64_t m_max)
{
    if (!hs || nranks < 1 || nranks > P2P_MAXR) return fail(LBFGSB_ERR_ARG, "bad arguments");
    for (int p = 0; p < nranks; ++p) {
        if (!hs[p] || hs[p]->comm_owned || (hs[p]->p2p && hs[p]->peer_ipc[0]))
            return fail(LBFGSB_ERR_ARG, "rank %d: not a plain single-GPU handle", p);
        TRY(alloc_mailbox(hs[p], nranks, m_max));
    }
    for (int p = 0; p < nranks; ++p) {
        hs[p]->p2p = true;
        for (int r = 0; r < nranks; ++r) { hs[p]->peer_mb[r] = hs[r]->mb; hs[p]->peer_ipc[r] = false; }
    }
    return LBFGSB_OK;
}

// ------------------------------------------------------------------ ops
extern "C" lbfgsb_err lbfgsb_op_gemv(const lbfgsb_objective* obj, const double* p, double* q,
                                     void* cuda_stream)
{
    if (!obj || obj->kind != 0 || !p || !q) return fail(LBFGSB_ERR_ARG, "bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(LBFGSB_ERR_CUDA, "no device");
    init_kernels();
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    Prob P;
    std::memset(&P, 0, sizeof P);
    P.m = obj->m; P.ncols = obj->ncols; P.ld = obj->ld; P.M = obj->M;
    P.colscale = obj->colscale; P.split = obj->split; P.qp = obj->qp;
    P.n = obj->split ? 2 * obj->ncols : obj->ncols;
    gemv_geometry(P);
    double* qpart = nullptr;
    unsigned* tick = nullptr;
    CK(cudaMallocAsync(&qpart, sizeof(double) * (size_t)P.m * P.CC, st));
    CK(cudaMallocAsync(&tick, sizeof(unsigned) * (NTICKETS + TICKETS_EXTRA), st));
    CK(cudaMemsetAsync(tick, 0, sizeof(unsigned) * (NTICKETS + TICKETS_EXTRA), st));
    P.qpart = qpart;
    P.tickets = tick;
    launch_fwd(P, st, FWD_P, p, q);
    cudaError_t e = cudaGetLastError();
    cudaFreeAsync(qpart, st);
    cudaFreeAsync(tick, st);
    if (e != cudaSuccess) return fail(LBFGSB_ERR_CUDA, "gemv: %s", cudaGetErrorString(e));
    CK(cudaStreamSynchronize(st));
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_op_gaussian_kernel(const double* X, int64_t N, int64_t d, double gamma,
                                                double* K, int64_t ldk, void* cuda_stream)
{
    if (!X || !K || N <= 0 || d <= 0 || ldk < N || !(gamma > 0)) return fail(LBFGSB_ERR_ARG, "bad arguments");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(LBFGSB_ERR_CUDA, "no device");
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    launch_gauss(X, N, d, gamma, K, ldk, st);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_op_gemvt(const lbfgsb_objective* obj, const double* r, double* g,
                                      void* cuda_stream)
{
    if (!obj || obj->kind != 0 || !r || !g) return fail(LBFGSB_ERR_ARG, "bad arguments");
    if (obj->qp) return lbfgsb_op_gemv(obj, r, g, cuda_stream);   // Q~ is symmetric
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return fail(LBFGSB_ERR_CUDA, "no device");
    init_kernels();
    cudaStream_t st = static_cast<cudaStream_t>(cuda_stream);
    Prob P;
    std::memset(&P, 0, sizeof P);
    P.m = obj->m; P.ncols = obj->ncols; P.ld = obj->ld; P.M = obj->M;
    P.colscale = obj->colscale; P.split = obj->split;
    P.n = obj->split ? 2 * obj->ncols : obj->ncols;
    gemv_geometry(P);
    P.rbuf[0] = const_cast<double*>(r);
    P.rbuf[1] = const_cast<double*>(r);
    launch_bwd(P, st, BWD_PLAIN, r, g);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_op_direction(lbfgsb_t* h, const double* x, const double* g, int32_t nh,
                                          const double* S, const double* Y, uint8_t* free_out,
                                          double* d_out, double* p_out, int32_t* projected, double* gp,
                                          double* amax)
{
    if (!h || !x || !g) return fail(LBFGSB_ERR_ARG, "NULL handle, x or g");
    if (nh < 0 || nh > h->mh || (nh > 0 && (!S || !Y))) return fail(LBFGSB_ERR_DIM, "bad history");
    Prob P;
    TRY(make_prob(h, nullptr, P));
    cudaStream_t st = h->st;
    const size_t nb = sizeof(double) * h->n;
    CK(cudaMemcpyAsync(P.x, x, nb, cudaMemcpyDeviceToDevice, st));
    CK(cudaMemcpyAsync(P.g, g, nb, cudaMemcpyDeviceToDevice, st));
    launch_ring_load(P, st, nh, S, Y);
    init_ctrl(h, h->o.tol);
    h->hc->nh = nh;
    h->hc->head = nh > 0 ? nh - 1 : h->mh - 1;
    TRY(ctrl_to_dev(h, h->st));
    launch_gram_recur(P, st, 1);
    launch_dir(P, st, 1);
    CK(cudaGetLastError());
    TRY(ctrl_to_host(h, h->st));
    const int br = h->hc->branch;
    if (free_out) CK(cudaMemcpyAsync(free_out, P.mask, (size_t)h->n, cudaMemcpyDeviceToDevice, st));
    if (d_out) CK(cudaMemcpyAsync(d_out, P.d, nb, cudaMemcpyDeviceToDevice, st));
    if (p_out) CK(cudaMemcpyAsync(p_out, br ? P.pp : P.pt, nb, cudaMemcpyDeviceToDevice, st));
    CK(cudaStreamSynchronize(st));
    if (projected) *projected = br;
    if (gp) *gp = h->hc->gp;
    if (amax) *amax = h->hc->amax;
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_op_trials(lbfgsb_t* h, const lbfgsb_objective* obj, const double* r,
                                       const double* q, const double* x, const double* p, double alpha0,
                                       int32_t ntrials, double* f_out)
{
    if (!h || !obj || obj->kind != 0 || !r || !q || !x || !p || !f_out)
        return fail(LBFGSB_ERR_ARG, "bad arguments");
    if (ntrials < 1 || ntrials > KT) return fail(LBFGSB_ERR_ARG, "ntrials in [1, %d]", KT);
    if (obj->qp) return fail(LBFGSB_ERR_UNSUPPORTED, "op_trials is for LSQ objectives");
    Prob P;
    TRY(make_prob(h, obj, P));
    set_sep(P);
    P.x = const_cast<double*>(x);
    init_ctrl(h, h->o.tol);
    h->hc->alpha0 = alpha0;
    h->hc->rho = 1.0;
    TRY(ctrl_to_dev(h, h->st));
    launch_sep(P, h->st, SEP_OP, p);
    launch_ls(P, h->st, LS_OP, r, q, h->fout.d(), ntrials);
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(f_out, h->fout.p, sizeof(double) * ntrials, cudaMemcpyDeviceToHost, h->st));
    CK(cudaStreamSynchronize(h->st));
    return LBFGSB_OK;
}

extern "C" lbfgsb_err lbfgsb_profile_get(lbfgsb_t* h, int32_t cap, const char** names, double* ms,
                                         int64_t* launches, int32_t* count, int32_t reset)
{
    if (!h || !count) return fail(LBFGSB_ERR_ARG, "NULL handle or count");
    static const char* kn[4] = {"gemv_active (k_fwd)", "gemvT_epi (k_bwd)", "all_kernel_launches",
                                "fwd_active_columns"};
    const double vals[4] = {h->prof_ms[0], h->prof_ms[1], 0.0, 0.0};
    const int64_t cnts[4] = {h->prof_n[0], h->prof_n[1], h->launches, h->nact_total};
    int c = 0;
    for (int i = 0; i < 4 && i < cap; ++i, ++c) {
        if (names) names[i] = kn[i];
        if (ms) ms[i] = vals[i];
        if (launches) launches[i] = cnts[i];
    }
    *count = c;
    if (reset) {
        h->prof_ms[0] = h->prof_ms[1] = 0;
        h->prof_n[0] = h->prof_n[1] = 0;
        h->launches = 0;
        h->nact_total = 0;
    }
    return LBFGSB_OK;
}
