// original.cu -- SURVEY.md 8(f) N3: the steps of the ORIGINAL L-BFGS-B
// (Byrd, Lu, Nocedal, Zhu 1995) around its generalized Cauchy point
// (cauchy.cu), so that lbfgsb_solve_original runs the paper's baseline
// ("L-BFGS-B GPU") end to end on B200:
//   k_og_pg     ||P(x - g) - x||_inf (the original's stopping test);
//   k_og_red    direct primal subspace minimisation, part 1 (BLNZ section
//               5.1): free set F = {l < x^c < u}, reduced gradient
//               r^c = g + theta (x^c - x) - W M c on F, v = W^T Z r^c and
//               K = W^T Z Z^T W (fixed-order per-CTA partials, last-CTA tail);
//   k_og_solve  (one thread) z = N^{-1} M v, N = I - (1/theta) M K;
//   k_og_dir    d^u = -(1/theta) r^c - (1/theta^2) W z on F and the largest
//               alpha* <= 1 that keeps x^c + alpha* d^u in the box (min);
//   k_og_apply  xbar = x^c + alpha* d^u, d = xbar - x, g^T d;
//   k_og_step   x' = clip(x + alpha d), s = x' - x, r' = r + alpha q;
//   k_og_pair   y = g' - g, s^T y, y^T y.
// All reductions: fixed thread -> data map, block trees, last CTA reduces
// the per-CTA partials in block order.
#include "impl.cuh"
#include "common.cuh"

namespace lb {

constexpr int OG_MAXH = 8;
constexpr int OG_NR = 2 * OG_MAXH + 4 * OG_MAXH * OG_MAXH;     // v (2h) + K (2h x 2h)

__device__ __forceinline__ bool og_free(const OrigArgs& A, int64_t i)
{
    const double xc = A.xc[i];
    return (!A.l || xc > A.l[i]) && (!A.u || xc < A.u[i]);
}

// w_i (2h) = (Y[:, i], theta S[:, i])
__device__ __forceinline__ double og_w(const OrigArgs& A, int a, int64_t i)
{
    return a < A.h ? A.Y[(int64_t)a * A.n + i] : A.theta * A.S[(int64_t)(a - A.h) * A.n + i];
}

__global__ void __launch_bounds__(NT) k_og_pg(OrigArgs A)
{
    __shared__ double red[NT / 32];
    __shared__ double buf[1024];
    __shared__ double stash[NT];
    double pg = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * NT) {
        const double v = fabs(clipd(A.x[i] - A.g[i], A.l[i], A.u[i]) - A.x[i]);
        pg = v > pg ? v : pg;
    }
    const double b = block_reduce<1>(pg, red);
    if (threadIdx.x == 0) A.part[blockIdx.x] = b;
    if (!last_cta(A.ticket + 0, gridDim.x)) return;
    reduce_parts(A.part, gridDim.x, 1, 1, [](int) { return 1; }, buf, 1024, stash, A.out + 2);
}

__global__ void __launch_bounds__(NT) k_og_red(OrigArgs A)
{
    __shared__ double red[NT / 32];
    __shared__ double buf[4096];
    __shared__ double stash[NT];
    const int k = 2 * A.h, nr = k + k * k;
    const double* Mc = A.Mm + k * k;
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += stride) {
        double rc = 0.0;
        if (og_free(A, i)) {
            double wMc = 0.0;
            for (int a = 0; a < k; ++a) wMc += og_w(A, a, i) * Mc[a];
            rc = A.g[i] + A.theta * (A.xc[i] - A.x[i]) - wMc;
        }
        A.rc[i] = rc;
    }
    for (int r = 0; r < nr; ++r) {
        double s = 0.0;
        for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += stride) {
            if (!og_free(A, i)) continue;
            if (r < k) {
                double wMc = 0.0;
                for (int a = 0; a < k; ++a) wMc += og_w(A, a, i) * Mc[a];
                const double rc = A.g[i] + A.theta * (A.xc[i] - A.x[i]) - wMc;
                s += og_w(A, r, i) * rc;                        // v = W^T Z r^c
            } else {
                const int e = r - k, a = e / k, b = e % k;
                s += og_w(A, a, i) * og_w(A, b, i);             // K = W^T Z Z^T W
            }
        }
        const double b = block_reduce<0>(s, red);
        if (threadIdx.x == 0) A.part[(int64_t)blockIdx.x * OG_NR + r] = b;
    }
    if (nr == 0) return;                                        // no pairs: r^c only
    if (!last_cta(A.ticket + 1, gridDim.x)) return;
    reduce_parts(A.part, gridDim.x, OG_NR, nr, [](int) { return 0; }, buf, 4096, stash, A.red);
}

__global__ void k_og_solve(OrigArgs A)
{
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const int k = 2 * A.h;
    const double* M = A.Mm;
    const double* v = A.red;
    const double* K = A.red + k;
    double Mv[2 * OG_MAXH], T[2 * OG_MAXH * 4 * OG_MAXH];
    for (int a = 0; a < k; ++a) {
        double s = 0.0;
        for (int b = 0; b < k; ++b) s += M[a * k + b] * v[b];
        Mv[a] = s;
    }
    for (int a = 0; a < k; ++a) {                                // [N | I], N = I - (1/theta) M K
        for (int b = 0; b < k; ++b) {
            double s = 0.0;
            for (int e = 0; e < k; ++e) s += M[a * k + e] * K[e * k + b];
            T[a * 2 * k + b] = (a == b ? 1.0 : 0.0) - s / A.theta;
        }
        for (int b = 0; b < k; ++b) T[a * 2 * k + k + b] = a == b ? 1.0 : 0.0;
    }
    for (int c = 0; c < k; ++c) {                                // Gauss-Jordan, partial pivoting
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
    for (int a = 0; a < k; ++a) {
        double s = 0.0;
        for (int b = 0; b < k; ++b) s += T[a * 2 * k + k + b] * Mv[b];
        A.z[a] = s;
    }
}

__global__ void __launch_bounds__(NT) k_og_dir(OrigArgs A)
{
    __shared__ double red[NT / 32];
    __shared__ double buf[1024];
    __shared__ double stash[NT];
    const int k = 2 * A.h;
    double amin = 1.0;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * NT) {
        double du = 0.0;
        if (og_free(A, i)) {
            double wz = 0.0;
            for (int a = 0; a < k; ++a) wz += og_w(A, a, i) * A.z[a];
            du = -A.rc[i] / A.theta - wz / (A.theta * A.theta);
            if (du > 0.0) { const double t = (A.u[i] - A.xc[i]) / du; amin = t < amin ? t : amin; }
            if (du < 0.0) { const double t = (A.l[i] - A.xc[i]) / du; amin = t < amin ? t : amin; }
        }
        A.du[i] = du;
    }
    const double b = block_reduce<2>(amin, red);
    if (threadIdx.x == 0) A.part[blockIdx.x] = b;
    if (!last_cta(A.ticket + 2, gridDim.x)) return;
    reduce_parts(A.part, gridDim.x, 1, 1, [](int) { return 2; }, buf, 1024, stash, A.out + 0);
    if (threadIdx.x == 0 && A.out[0] < 0.0) A.out[0] = 0.0;
}

__global__ void __launch_bounds__(NT) k_og_apply(OrigArgs A)
{
    __shared__ double red[NT / 32];
    __shared__ double buf[1024];
    __shared__ double stash[NT];
    const double as = A.out[0];
    double gd = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * NT) {
        const double xb = A.xc[i] + as * A.du[i];
        const double di = xb - A.x[i];
        A.d[i] = di;
        gd += A.g[i] * di;
    }
    const double b = block_reduce<0>(gd, red);
    if (threadIdx.x == 0) A.part[blockIdx.x] = b;
    if (!last_cta(A.ticket + 3, gridDim.x)) return;
    reduce_parts(A.part, gridDim.x, 1, 1, [](int) { return 0; }, buf, 1024, stash, A.out + 1);
}

__global__ void __launch_bounds__(NT) k_og_step(OrigArgs A, double* x, const double* dvec, double* r,
                                                const double* q, double alpha, double* s_out)
{
    const int64_t stride = (int64_t)gridDim.x * NT;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += stride) {
        const double xo = x[i];
        const double xn = clipd(fma(alpha, dvec[i], xo), A.l[i], A.u[i]);
        x[i] = xn;
        s_out[i] = xn - xo;
    }
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.m; i += stride) r[i] = fma(alpha, q[i], r[i]);
}

__global__ void __launch_bounds__(NT) k_og_pair(OrigArgs A, const double* gnew, const double* gold,
                                                const double* s, double* y_out)
{
    __shared__ double msh[NT / 32 * 2];
    __shared__ double buf[1024];
    __shared__ double stash[NT];
    __shared__ double o2[2];
    double acc[2] = {0.0, 0.0};
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.n; i += (int64_t)gridDim.x * NT) {
        const double y = gnew[i] - gold[i];
        y_out[i] = y;
        acc[0] += s[i] * y;
        acc[1] += y * y;
    }
    block_sum_multi<2>(acc, msh, o2);
    if (threadIdx.x < 2) A.part[(int64_t)blockIdx.x * 2 + threadIdx.x] = o2[threadIdx.x];
    if (!last_cta(A.ticket + 4, gridDim.x)) return;
    reduce_parts(A.part, gridDim.x, 2, 2, [](int) { return 0; }, buf, 1024, stash, A.out + 3);
}

__global__ void __launch_bounds__(NT) k_og_residual(OrigArgs A, double* r, const double* b)
{
    __shared__ double red[NT / 32];
    __shared__ double buf[1024];
    __shared__ double stash[NT];
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)NT + threadIdx.x; i < A.m; i += (int64_t)gridDim.x * NT) {
        const double ri = b ? r[i] - b[i] : r[i];
        r[i] = ri;
        s += ri * ri;
    }
    const double t = block_reduce<0>(s, red);
    if (threadIdx.x == 0) A.part[blockIdx.x] = t;
    if (!last_cta(A.ticket + 5, gridDim.x)) return;
    reduce_parts(A.part, gridDim.x, 1, 1, [](int) { return 0; }, buf, 1024, stash, A.out + 5);
}

static int og_blocks(int64_t n)
{
    int64_t g = (n + NT - 1) / NT;
    const int64_t cap = 2LL * sm_count();
    return (int)(g < 1 ? 1 : (g > cap ? cap : g));
}

void launch_orig_pg(const OrigArgs& A, cudaStream_t st) { k_og_pg<<<og_blocks(A.n), NT, 0, st>>>(A); }

void launch_orig_subspace(const OrigArgs& A, cudaStream_t st)
{
    const int G = og_blocks(A.n);
    if (A.h > 0) {
        k_og_red<<<G, NT, 0, st>>>(A);
        k_og_solve<<<1, 32, 0, st>>>(A);
    } else {
        k_og_red<<<G, NT, 0, st>>>(A);                           // r^c only (no pairs: z unused)
    }
    k_og_dir<<<G, NT, 0, st>>>(A);
    k_og_apply<<<G, NT, 0, st>>>(A);
}

void launch_orig_step(const OrigArgs& A, double* x, const double* dvec, double* r, const double* q, double alpha,
                      double* s_out, cudaStream_t st)
{
    k_og_step<<<og_blocks(A.n > A.m ? A.n : A.m), NT, 0, st>>>(A, x, dvec, r, q, alpha, s_out);
}

void launch_orig_pair(const OrigArgs& A, const double* gnew, const double* gold, const double* s, double* y_out,
                      cudaStream_t st)
{
    k_og_pair<<<og_blocks(A.n), NT, 0, st>>>(A, gnew, gold, s, y_out);
}

void launch_orig_residual(const OrigArgs& A, double* r, const double* b, cudaStream_t st)
{
    k_og_residual<<<og_blocks(A.m), NT, 0, st>>>(A, r, b);
}

int orig_nr() { return OG_NR; }

}  // namespace lb
