// gen.cu -- device side of synth/philox.py: fills a column-major m x n matrix
// with A_ij = (u_ij - 1/2) * scale, u from Philox4x32-10 at counter
// (i >> 1, j0 + j, mat, 0), key (seed lo, seed hi).  Input synthesis only
// (test / bench infrastructure); bit-identical to the numpy implementation.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void philox(uint32_t c[4], uint32_t k0, uint32_t k1)
{
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) { k0 += W0; k1 += W1; }
        const uint64_t p0 = (uint64_t)M0 * c[0], p1 = (uint64_t)M1 * c[2];
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        const uint32_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
        c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    }
}

__global__ void k_fill_centered(double* A, int64_t m, int64_t ncols, int64_t ld, int64_t j0,
                                uint64_t seed, uint32_t mat, double scale)
{
    const int64_t pairs = (m + 1) / 2;
    const int64_t total = pairs * ncols;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t j = t / pairs, p = t - j * pairs;
        uint32_t c[4] = {(uint32_t)p, (uint32_t)(j0 + j), mat, 0u};
        philox(c, (uint32_t)seed, (uint32_t)(seed >> 32));
        const uint64_t e = ((uint64_t)c[1] << 32) | c[0];
        const uint64_t o = ((uint64_t)c[3] << 32) | c[2];
        const double ue = (double)(e >> 11) * 0x1.0p-53, uo = (double)(o >> 11) * 0x1.0p-53;
        double* col = A + j * ld;
        const int64_t i = 2 * p;
        col[i] = __dmul_rn(ue - 0.5, scale);
        if (i + 1 < m) col[i + 1] = __dmul_rn(uo - 0.5, scale);
    }
}

extern "C" int synth_fill_centered(double* A, int64_t m, int64_t ncols, int64_t ld, int64_t j0,
                                   uint64_t seed, uint32_t mat, double scale, void* stream)
{
    k_fill_centered<<<148 * 16, 256, 0, static_cast<cudaStream_t>(stream)>>>(A, m, ncols, ld, j0, seed,
                                                                              mat, scale);
    return (int)cudaGetLastError();
}
