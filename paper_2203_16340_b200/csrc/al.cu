// al.cu -- a8 of SURVEY.md 8(a) for the GENERAL problem class of the paper
// (min f(x) s.t. h(x) = 0, g(x) <= 0, l <= x <= u, with h
// and g arbitrary differentiable maps): the pieces of Eq. (3)
// and of Alg. 4 lines 6-8 that act on the stacked
// constraint vectors, on the device:
//   k_al_terms   -- w_eq = rho h + lambda, w_in = (rho g + mu)_+ and the
//                   penalty value rho/2 ||h + lambda/rho||^2 + rho/2 ||(g + mu/rho)_+||^2;
//   k_al_update  -- lambda += rho h, mu = (mu + rho g)_+ and the violation
//                   max(||h||_inf, ||min(-g, mu/rho)||_inf) (readings R20/R21);
//   k_lsq_value  -- the LSQ base objective's value and the separable part of
//                   its gradient from r = M~x - b: 1/2||r||^2 + c^T x + delta/2||x||^2,
//                   g += c + delta x;
//   k_sub / k_axpy -- r -= b, y += x.
// The linear constraint blocks E^T x (K dots of length n) and E w (a sum of K
// columns) run on the GEMV kernels themselves (k_bwd / k_fwd, with E as the
// operator: n rows, K columns), so a constraint pass costs one read of E.
// One CTA per reduction (deterministic order: thread-strided sums, then a
// fixed shuffle / shared-memory tree); K and n here are at most a few 1e5.
#include "common.cuh"

namespace lb {

constexpr int AT = 1024;

__global__ void __launch_bounds__(AT) k_al_terms(int64_t neq, const double* h, const double* lam, int64_t nin,
                                                 const double* g, const double* mu, double rho, double* weq,
                                                 double* win, double* out)
{
    __shared__ double sh[AT / 32];
    double s = 0.0;
    for (int64_t k = threadIdx.x; k < neq; k += AT) {
        const double t = h[k] + lam[k] / rho;                // Eq. (3): h + lambda / rho
        s += 0.5 * rho * t * t;
        weq[k] = rho * h[k] + lam[k];                        // grad: J_h^T (rho h + lambda)
    }
    for (int64_t k = threadIdx.x; k < nin; k += AT) {
        double t = g[k] + mu[k] / rho;
        if (t < 0.0) t = 0.0;                                // (.)_+
        s += 0.5 * rho * t * t;
        win[k] = rho * t;                                    // grad: J_g^T (rho g + mu)_+
    }
    const double v = block_reduce<0>(s, sh);
    if (threadIdx.x == 0) out[0] = v;
}

__global__ void __launch_bounds__(AT) k_al_update(int64_t neq, const double* h, double* lam, int64_t nin,
                                                  const double* g, double* mu, double rho, double* vout)
{
    __shared__ double sh[AT / 32];
    double v = 0.0;
    for (int64_t k = threadIdx.x; k < neq; k += AT) {
        lam[k] = lam[k] + rho * h[k];                        // Alg. 4 line 6
        const double a = fabs(h[k]);
        v = a > v ? a : v;
    }
    for (int64_t k = threadIdx.x; k < nin; k += AT) {
        const double t = mu[k] + rho * g[k];                 // Alg. 4 line 7
        const double m1 = t > 0.0 ? t : 0.0;
        mu[k] = m1;
        double c = -g[k];                                    // R21: min(-g, mu/rho)
        const double mr = m1 / rho;
        if (mr < c) c = mr;
        const double a = fabs(c);
        v = a > v ? a : v;
    }
    const double r = block_reduce<1>(v, sh);
    if (threadIdx.x == 0) vout[0] = r;
}

// violation only (at the start: v(x^0) with the initial multipliers)
__global__ void __launch_bounds__(AT) k_al_violation(int64_t neq, const double* h, int64_t nin, const double* g,
                                                     const double* mu, double rho, double* vout)
{
    __shared__ double sh[AT / 32];
    double v = 0.0;
    for (int64_t k = threadIdx.x; k < neq; k += AT) {
        const double a = fabs(h[k]);
        v = a > v ? a : v;
    }
    for (int64_t k = threadIdx.x; k < nin; k += AT) {
        double c = -g[k];
        const double mr = mu[k] / rho;
        if (mr < c) c = mr;
        const double a = fabs(c);
        v = a > v ? a : v;
    }
    const double r = block_reduce<1>(v, sh);
    if (threadIdx.x == 0) vout[0] = r;
}

// LSQ base objective at x from r = M~x - b: out[0] = 1/2||r||^2 + c^T x + delta/2||x||^2,
// g += c + delta x (g holds M~^T r on entry)
__global__ void __launch_bounds__(AT) k_lsq_value(int64_t m, const double* r, int64_t n, const double* x,
                                                  const double* c, double delta, double* g, double* out)
{
    __shared__ double sh[AT / 32];
    double rr = 0.0, cx = 0.0, xx = 0.0;
    for (int64_t i = threadIdx.x; i < m; i += AT) rr += r[i] * r[i];
    for (int64_t j = threadIdx.x; j < n; j += AT) {
        const double xj = x[j];
        double gj = g[j];
        if (c) { cx += c[j] * xj; gj = gj + c[j]; }
        xx += xj * xj;
        gj = gj + delta * xj;
        g[j] = gj;
    }
    const double a = block_reduce<0>(rr, sh);
    __syncthreads();
    const double b = block_reduce<0>(cx, sh);
    __syncthreads();
    const double d = block_reduce<0>(xx, sh);
    if (threadIdx.x == 0) out[0] = 0.5 * a + b + 0.5 * delta * d;
}

__global__ void k_sub(int64_t n, double* r, const double* b)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        r[i] = r[i] - b[i];
}

__global__ void k_axpy(int64_t n, const double* x, double* y)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = y[i] + x[i];
}

void launch_al_terms(int64_t neq, const double* h, const double* lam, int64_t nin, const double* g,
                     const double* mu, double rho, double* weq, double* win, double* out, cudaStream_t st)
{
    k_al_terms<<<1, AT, 0, st>>>(neq, h, lam, nin, g, mu, rho, weq, win, out);
}

void launch_al_update(int64_t neq, const double* h, double* lam, int64_t nin, const double* g, double* mu,
                      double rho, double* vout, cudaStream_t st)
{
    k_al_update<<<1, AT, 0, st>>>(neq, h, lam, nin, g, mu, rho, vout);
}

void launch_al_violation(int64_t neq, const double* h, int64_t nin, const double* g, const double* mu, double rho,
                         double* vout, cudaStream_t st)
{
    k_al_violation<<<1, AT, 0, st>>>(neq, h, nin, g, mu, rho, vout);
}

void launch_lsq_value(int64_t m, const double* r, int64_t n, const double* x, const double* c, double delta,
                      double* g, double* out, cudaStream_t st)
{
    k_lsq_value<<<1, AT, 0, st>>>(m, r, n, x, c, delta, g, out);
}

void launch_sub(int64_t n, double* r, const double* b, cudaStream_t st)
{
    const int64_t g = (n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184;
    if (n > 0) k_sub<<<(int)g, 256, 0, st>>>(n, r, b);
}

void launch_axpy(int64_t n, const double* x, double* y, cudaStream_t st)
{
    const int64_t g = (n + 255) / 256 < 1184 ? (n + 255) / 256 : 1184;
    if (n > 0) k_axpy<<<(int)g, 256, 0, st>>>(n, x, y);
}

}  // namespace lb
