// cauchy.cu -- SURVEY.md 8(f) N3: the generalized Cauchy point of the ORIGINAL
// L-BFGS-B (Byrd, Lu, Nocedal, Zhu 1995, Algorithm CP) on the GPU, as the
// paper's baseline runs it ("an inherently
// sequential Cauchy point computation ... all but one core ... idle").
//
//   k_cp_prep   (parallel) breakpoints t_i, d = -g on {t_i > 0}, x_cp = x, and
//               the reductions f' = -d^T d, p = W^T d, S^T S, S^T Y (fixed-order
//               per-CTA partials, last-CTA tail);
//   k_cp_scan   (ONE thread) the middle matrix M = [[-D, L^T], [L, theta S^T S]]^{-1},
//               a binary heap of the breakpoints keyed (t_i, i) (shared memory when
//               it fits, else global), and the breakpoint loop of Algorithm CP
//               (O(h^2) scalar work per breakpoint passed);
//   k_cp_final  (parallel) x_cp = x + t d on the variables still moving.
//
// The parallel parts are as parallel as B200 allows; the scan is the part the
// paper shows cannot be: its time is what the N3 measurement reports.
#include "impl.cuh"
#include "common.cuh"

namespace lb {

constexpr int CP_MAXH = 8;                   // pairs supported by the op
constexpr int CP_NR = 1 + 2 * CP_MAXH + 2 * CP_MAXH * CP_MAXH;

struct CpArgs {
    int64_t n;
    const double* x; const double* g; const double* l; const double* u;
    int h;
    const double* S; const double* Y;        // h x n, pair i at + i n (oldest first)
    double theta;
    double* d;                               // n
    double* tk;                              // n breakpoints (+inf: never; 0: fixed)
    double* xcp;                             // n
    double* part;                            // [G][CP_NR]
    double* red;                             // [CP_NR] reduced: f', p (2h), S^T S (h*h), S^T Y (h*h)
    unsigned* ticket;
    double* heap_g;                          // global heap (2 doubles per entry) when smem is short
    int64_t heap_cap_smem;                   // entries that fit in dynamic smem
    double* scal;                            // out: [0] t_old, [1] passed, [2..2+2h) c
    double* Mout;                            // out (may be NULL): M (2h x 2h row-major), then M c (2h)
};

__global__ void __launch_bounds__(NT) k_cp_prep(CpArgs A)
{
    const int h = A.h, nr = 1 + 2 * h + 2 * h * h;
    __shared__ double red[NT / 32];
    __shared__ double buf[4096];
    __shared__ double stash[NT];
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += stride) {
        const double gi = A.g[i], xi = A.x[i];
        double ti = INFINITY;
        if (gi < 0.0 && A.u) ti = (xi - A.u[i]) / gi;
        else if (gi > 0.0 && A.l) ti = (xi - A.l[i]) / gi;
        A.d[i] = (ti == 0.0) ? 0.0 : -gi;
        A.tk[i] = ti;
        A.xcp[i] = xi;
    }
    // per-CTA partials of the nr reduced values (one block reduction each)
    for (int r = 0; r < nr; ++r) {
        double s = 0.0;
        for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += stride) {
            const double gi = A.g[i], xi = A.x[i];
            double ti = INFINITY;
            if (gi < 0.0 && A.u) ti = (xi - A.u[i]) / gi;
            else if (gi > 0.0 && A.l) ti = (xi - A.l[i]) / gi;
            const double di = (ti == 0.0) ? 0.0 : -gi;
            if (r == 0) {
                s -= di * di;                                   // f' = -d^T d
            } else if (r <= 2 * h) {
                const int a = r - 1;                            // p = W^T d, W = [Y, theta S]
                s += a < h ? A.Y[(int64_t)a * A.n + i] * di : A.theta * A.S[(int64_t)(a - h) * A.n + i] * di;
            } else {
                const int e = r - 1 - 2 * h;                    // S^T S then S^T Y, row-major h x h
                const int which = e / (h * h), ij = e % (h * h), ii = ij / h, jj = ij % h;
                const double si = A.S[(int64_t)ii * A.n + i];
                s += si * (which == 0 ? A.S[(int64_t)jj * A.n + i] : A.Y[(int64_t)jj * A.n + i]);
            }
        }
        const double b = block_reduce<0>(s, red);
        if (threadIdx.x == 0) A.part[(int64_t)blockIdx.x * CP_NR + r] = b;
    }
    if (!last_cta(A.ticket, gridDim.x)) return;
    reduce_parts(A.part, gridDim.x, CP_NR, nr, [](int) { return 0; }, buf, 4096, stash, A.red);
}

// ---- single-thread helpers
struct CpHeap {
    double* t; int64_t* i; int64_t size;
    __device__ bool less(int64_t a, int64_t b) const { return t[a] < t[b] || (t[a] == t[b] && i[a] < i[b]); }
    __device__ void swap(int64_t a, int64_t b)
    {
        const double tt = t[a]; t[a] = t[b]; t[b] = tt;
        const int64_t ii = i[a]; i[a] = i[b]; i[b] = ii;
    }
    __device__ void down(int64_t k)
    {
        for (;;) {
            const int64_t l = 2 * k + 1, r = l + 1;
            int64_t m = k;
            if (l < size && less(l, m)) m = l;
            if (r < size && less(r, m)) m = r;
            if (m == k) return;
            swap(k, m);
            k = m;
        }
    }
    __device__ void pop()
    {
        --size;
        if (size > 0) { t[0] = t[size]; i[0] = i[size]; down(0); }
    }
};

__device__ void cp_matvec(int k, const double* M, const double* v, double* out)
{
    for (int a = 0; a < k; ++a) {
        double s = 0.0;
        for (int b = 0; b < k; ++b) s += M[a * k + b] * v[b];
        out[a] = s;
    }
}

__global__ void k_cp_scan(CpArgs A)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    extern __shared__ __align__(16) double hs[];
    const int h = A.h, k = 2 * h;
    const double theta = A.theta;
    double M[4 * CP_MAXH * CP_MAXH], T[2 * CP_MAXH * 4 * CP_MAXH];
    // middle matrix: [[-D, L^T], [L, theta S^T S]]^{-1} (Gauss-Jordan, partial pivoting)
    const double* SS = A.red + 1 + 2 * h;
    const double* SY = SS + h * h;
    for (int a = 0; a < h; ++a)
        for (int b = 0; b < h; ++b) {
            const double sy = SY[a * h + b];
            M[a * k + b] = a == b ? -sy : 0.0;
            M[(h + a) * k + b] = a > b ? sy : 0.0;
            M[b * k + h + a] = a > b ? sy : 0.0;
            M[(h + a) * k + h + b] = theta * SS[a * h + b];
        }
    for (int a = 0; a < k; ++a) {
        for (int b = 0; b < k; ++b) T[a * 2 * k + b] = M[a * k + b];
        for (int b = 0; b < k; ++b) T[a * 2 * k + k + b] = a == b ? 1.0 : 0.0;
    }
    for (int c = 0; c < k; ++c) {
        int piv = c;
        for (int r = c + 1; r < k; ++r) if (fabs(T[r * 2 * k + c]) > fabs(T[piv * 2 * k + c])) piv = r;
        if (piv != c)
            for (int j = 0; j < 2 * k; ++j) { const double t = T[c * 2 * k + j]; T[c * 2 * k + j] = T[piv * 2 * k + j]; T[piv * 2 * k + j] = t; }
        const double dv = T[c * 2 * k + c];
        for (int j = 0; j < 2 * k; ++j) T[c * 2 * k + j] /= dv;
        for (int r = 0; r < k; ++r) {
            if (r == c) continue;
            const double f = T[r * 2 * k + c];
            if (f == 0.0) continue;
            for (int j = 0; j < 2 * k; ++j) T[r * 2 * k + j] -= f * T[c * 2 * k + j];
        }
    }
    for (int a = 0; a < k; ++a) for (int b = 0; b < k; ++b) M[a * k + b] = T[a * 2 * k + k + b];

    double p[2 * CP_MAXH], c[2 * CP_MAXH], Mv[2 * CP_MAXH], wb[2 * CP_MAXH];
    for (int j = 0; j < k; ++j) { p[j] = A.red[1 + j]; c[j] = 0.0; }
    double fp = A.red[0];
    if (fp == 0.0) {                                            // d = 0: x is the Cauchy point
        A.scal[0] = 0.0; A.scal[1] = 0.0;
        for (int j = 0; j < k; ++j) A.scal[2 + j] = 0.0;
        if (A.Mout) {
            for (int j = 0; j < k * k; ++j) A.Mout[j] = M[j];
            for (int j = 0; j < k; ++j) A.Mout[k * k + j] = 0.0;
        }
        return;
    }
    // heap of the breakpoints {t_i > 0}, keyed (t_i, i)
    CpHeap H;
    const bool in_smem = A.n <= A.heap_cap_smem;
    H.t = in_smem ? hs : A.heap_g;
    H.i = reinterpret_cast<int64_t*>(in_smem ? hs + A.n : A.heap_g + A.n);
    H.size = 0;
    for (int64_t i = 0; i < A.n; ++i) {
        const double ti = A.tk[i];
        if (ti > 0.0) { H.t[H.size] = ti; H.i[H.size] = i; ++H.size; }
    }
    for (int64_t q = H.size / 2 - 1; q >= 0; --q) H.down(q);
    cp_matvec(k, M, p, Mv);
    double pMp = 0.0;
    for (int j = 0; j < k; ++j) pMp += p[j] * Mv[j];
    double fpp = -theta * fp - pMp;
    double dtmin = -fp / fpp, told = 0.0;
    long long passed = 0;
    double t = H.size > 0 ? H.t[0] : INFINITY;
    double dt = t - told;
    while (H.size > 0 && dtmin >= dt) {
        const int64_t b = H.i[0];
        H.pop();
        ++passed;
        const double gb = A.g[b];
        const double db = A.d[b];
        const double xb = db > 0.0 ? A.u[b] : A.l[b];
        A.xcp[b] = xb;
        const double zb = xb - A.x[b];
        for (int j = 0; j < k; ++j) c[j] += dt * p[j];
        for (int a = 0; a < h; ++a) { wb[a] = A.Y[(int64_t)a * A.n + b]; wb[h + a] = theta * A.S[(int64_t)a * A.n + b]; }
        double wMc = 0.0, wMp = 0.0, wMw = 0.0;
        cp_matvec(k, M, c, Mv);
        for (int j = 0; j < k; ++j) wMc += wb[j] * Mv[j];
        cp_matvec(k, M, p, Mv);
        for (int j = 0; j < k; ++j) wMp += wb[j] * Mv[j];
        cp_matvec(k, M, wb, Mv);
        for (int j = 0; j < k; ++j) wMw += wb[j] * Mv[j];
        fp = fp + dt * fpp + gb * gb + theta * gb * zb - gb * wMc;
        fpp = fpp - theta * gb * gb - 2.0 * gb * wMp - gb * gb * wMw;
        for (int j = 0; j < k; ++j) p[j] += gb * wb[j];
        A.d[b] = 0.0;
        dtmin = -fp / fpp;
        told = t;
        t = H.size > 0 ? H.t[0] : INFINITY;
        dt = t - told;
    }
    if (dtmin < 0.0) dtmin = 0.0;
    told = told + dtmin;
    for (int j = 0; j < k; ++j) c[j] += dtmin * p[j];
    A.scal[0] = told;
    A.scal[1] = (double)passed;
    for (int j = 0; j < k; ++j) A.scal[2 + j] = c[j];
    if (A.Mout) {                                               // for the subspace minimisation
        for (int j = 0; j < k * k; ++j) A.Mout[j] = M[j];
        cp_matvec(k, M, c, Mv);
        for (int j = 0; j < k; ++j) A.Mout[k * k + j] = Mv[j];
    }
}

__global__ void __launch_bounds__(NT) k_cp_final(CpArgs A)
{
    const double told = A.scal[0];
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * NT) {
        const double di = A.d[i];
        if (di != 0.0) A.xcp[i] = A.x[i] + told * di;
    }
}

// Launch the three kernels; ev (4 events, may be NULL) brackets the scan.
int launch_cauchy(int64_t n, const double* x, const double* g, const double* l, const double* u, int h,
                  const double* S, const double* Y, double theta, double* d, double* tk, double* xcp,
                  double* part, double* red, unsigned* ticket, double* heap_g, double* scal,
                  cudaStream_t st, cudaEvent_t e0, cudaEvent_t e1, double* Mout)
{
    if (h < 0 || h > CP_MAXH) return 1;
    CpArgs A;
    A.Mout = Mout;
    A.n = n; A.x = x; A.g = g; A.l = l; A.u = u; A.h = h; A.S = S; A.Y = Y; A.theta = theta;
    A.d = d; A.tk = tk; A.xcp = xcp; A.part = part; A.red = red; A.ticket = ticket;
    A.heap_g = heap_g; A.scal = scal;
    const size_t smem_max = 200 * 1024;
    A.heap_cap_smem = (int64_t)(smem_max / 16);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_cp_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max);
        attr = true;
    }
    int G = (int)((n + NT - 1) / NT);
    if (G > 2 * sm_count()) G = 2 * sm_count();
    if (G < 1) G = 1;
    k_cp_prep<<<G, NT, 0, st>>>(A);
    if (e0) cudaEventRecord(e0, st);
    const size_t smem = n <= A.heap_cap_smem ? (size_t)n * 16 : 0;
    k_cp_scan<<<1, 32, smem, st>>>(A);
    if (e1) cudaEventRecord(e1, st);
    k_cp_final<<<G, NT, 0, st>>>(A);
    return 0;
}

int cauchy_nr() { return CP_NR; }

}  // namespace lb
