// bw_probe.cu -- achievable HBM READ bandwidth on this B200 (the ceiling the
// GEMV kernels stream against).  Variants:
//   ldg<U>  : grid-stride LDG.128 sum, 148*k CTAs, U loads in flight per thread
//   bulk    : 1 CTA/SM, cp.async.bulk (TMA 1-D) ring of S stages x B bytes
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bw_probe tools/bw_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void ldg_sum(const double2* __restrict__ a, size_t n2, double* out)
{
    double s = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
    }
    for (; i < n2; i += stride) { double2 v = a[i]; s += v.x + v.y; }
    if (s == 123.456) out[0] = s;
}

// the same with 256-bit loads (LDG.E.ENL2.256, sm_100a): half the load instructions per byte
__device__ __forceinline__ void ld256cs(const double* p, double& a, double& b, double& c, double& d)
{
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
template <int U>
__global__ void ldg256_sum(const double* __restrict__ a, size_t n4, double* out)
{
    double s = 0.0;
    const size_t stride = (size_t)gridDim.x * blockDim.x;
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    for (; i + (U - 1) * stride < n4; i += U * stride) {
        double v[U][4];
#pragma unroll
        for (int u = 0; u < U; ++u) ld256cs(a + 4 * (i + u * stride), v[u][0], v[u][1], v[u][2], v[u][3]);
#pragma unroll
        for (int u = 0; u < U; ++u) s += (v[u][0] + v[u][1]) + (v[u][2] + v[u][3]);
    }
    if (s == 123.456) out[0] = s;
}

// contiguous chunk per CTA (like a persistent column range)
template <int U>
__global__ void ldg_chunk(const double2* __restrict__ a, size_t n2, double* out)
{
    const size_t per = (n2 + gridDim.x - 1) / gridDim.x;
    const size_t b0 = blockIdx.x * per, b1 = b0 + per < n2 ? b0 + per : n2;
    double s = 0.0;
    size_t i = b0 + threadIdx.x;
    const size_t stride = blockDim.x;
    for (; i + (U - 1) * stride < b1; i += U * stride) {
        double2 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldcs(a + i + u * stride);
#pragma unroll
        for (int u = 0; u < U; ++u) s += v[u].x + v[u].y;
    }
    for (; i < b1; i += stride) { double2 v = a[i]; s += v.x + v.y; }
    if (s == 123.456) out[0] = s;
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(bytes));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase)
{
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"((unsigned)__cvta_generic_to_shared(bar)), "r"(phase));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(dst)), "l"(src), "r"(bytes),
                    "r"((unsigned)__cvta_generic_to_shared(bar)) : "memory");
}

template <int STAGES, int BYTES>
__global__ void bulk_sum(const double* __restrict__ a, size_t n, double* out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const size_t per = (n + gridDim.x - 1) / gridDim.x;
    const size_t b0 = blockIdx.x * per, b1 = b0 + per < n ? b0 + per : n;
    const size_t elems = BYTES / 8;
    const size_t nchunks = (b1 - b0 + elems - 1) / elems;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](size_t c) {
        const int s = c % STAGES;
        const size_t e0 = b0 + c * elems;
        const size_t cnt = e0 + elems < b1 ? elems : b1 - e0;
        mbar_expect_tx(&full[s], (unsigned)(cnt * 8));
        bulk_g2s(sm + (size_t)s * BYTES, a + e0, (unsigned)(cnt * 8), &full[s]);
    };
    if (threadIdx.x == 0)
        for (size_t c = 0; c < (size_t)STAGES && c < nchunks; ++c) issue(c);
    double acc = 0.0;
    for (size_t c = 0; c < nchunks; ++c) {
        const int s = c % STAGES;
        mbar_wait(&full[s], (unsigned)((c / STAGES) & 1));
        const size_t e0 = b0 + c * elems;
        const size_t cnt = e0 + elems < b1 ? elems : b1 - e0;
        const double* buf = reinterpret_cast<const double*>(sm + (size_t)s * BYTES);
        for (size_t k = threadIdx.x; k < cnt; k += blockDim.x) acc += buf[k];
        __syncthreads();
        if (threadIdx.x == 0 && c + STAGES < nchunks) issue(c + STAGES);
    }
    if (acc == 123.456) out[0] = acc;
}


template <int STAGES, int BYTES>
__global__ void __cluster_dims__(2, 1, 1) bulk_sum_cl(const double* __restrict__ a, size_t n, double* out)
{
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const size_t per = (n + gridDim.x - 1) / gridDim.x;
    const size_t b0 = blockIdx.x * per, b1 = b0 + per < n ? b0 + per : n;
    const size_t elems = BYTES / 8;
    const size_t nchunks = (b1 - b0 + elems - 1) / elems;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](size_t c) {
        const int s = c % STAGES;
        const size_t e0 = b0 + c * elems;
        const size_t cnt = e0 + elems < b1 ? elems : b1 - e0;
        mbar_expect_tx(&full[s], (unsigned)(cnt * 8));
        bulk_g2s(sm + (size_t)s * BYTES, a + e0, (unsigned)(cnt * 8), &full[s]);
    };
    if (threadIdx.x == 0)
        for (size_t c = 0; c < (size_t)STAGES && c < nchunks; ++c) issue(c);
    double acc = 0.0;
    for (size_t c = 0; c < nchunks; ++c) {
        const int s = c % STAGES;
        mbar_wait(&full[s], (unsigned)((c / STAGES) & 1));
        const size_t e0 = b0 + c * elems;
        const size_t cnt = e0 + elems < b1 ? elems : b1 - e0;
        const double* buf = reinterpret_cast<const double*>(sm + (size_t)s * BYTES);
        for (size_t k = threadIdx.x; k < cnt; k += blockDim.x) acc += buf[k];
        __syncthreads();
        if (threadIdx.x == 0 && c + STAGES < nchunks) issue(c + STAGES);
    }
    if (acc == 123.456) out[0] = acc;
}


// GEMV^T-shaped stream (C2: m = 20000 rows x 10000 columns, per-CTA balanced column ranges,
// 4096-row segments per column (the last one 3616 rows), 4 x 32 KB TMA ring, thread 0 refills
// after a CTA barrier).  FMA = 0: sum the segment (as bulk_sum); 1: FMA against r' held in
// registers (thread t owns rows 512 k + 2 t), one accumulator per column.
template <int FMA>
__global__ void __launch_bounds__(256, 1) seg_stream(const double* __restrict__ a, int64_t m, int64_t ncols, double* out)
{
    constexpr int S = 4, R = 4096, NSC = 5;
    extern __shared__ __align__(128) unsigned char sm[];
    double* ring = reinterpret_cast<double*>(sm);
    __shared__ __align__(8) uint64_t full[S];
    const int G = gridDim.x, cta = blockIdx.x, tid = threadIdx.x;
    const int64_t j0 = (int64_t)cta * ncols / G, j1 = (int64_t)(cta + 1) * ncols / G;
    const int64_t total = (j1 - j0) * NSC;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    auto issue = [&](int64_t e) {
        const int64_t c = e / NSC, r0 = (e - c * NSC) * (int64_t)R;
        const int sl = (int)(e % S);
        const unsigned bytes = 8u * (unsigned)(m - r0 < R ? m - r0 : R);
        mbar_expect_tx(&full[sl], bytes);
        bulk_g2s(ring + (size_t)sl * R, a + (j0 + c) * m + r0, bytes, &full[sl]);
    };
    if (tid == 0) for (int64_t e = 0; e < S && e < total; ++e) issue(e);
    double2 rr[NSC * 8];
#pragma unroll
    for (int k = 0; k < NSC * 8; ++k) {
        if (FMA >= 2) {                                  // r' from global memory, as the kernels do
            const int64_t i = (int64_t)k * 512 + 2 * tid;
            rr[k] = i < m ? *reinterpret_cast<const double2*>(a + i) : make_double2(0.0, 0.0);
        } else {
            rr[k] = make_double2(1.0 + 1e-3 * k, 1.0 - 1e-3 * k);
        }
    }
    double acc = 0.0, tot = 0.0;
    int64_t it = 0;
    if (FMA == 3) {                                      // 8-column groups, 8 accumulators (k_bwd_t's body)
        for (int64_t jg = 0; jg < j1 - j0; jg += 8) {
            const int nc = (int)(j1 - j0 - jg < 8 ? j1 - j0 - jg : 8);
            double acc8[8];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                acc8[c] = 0.0;
                if (c < nc) {
#pragma unroll
                    for (int s = 0; s < NSC; ++s, ++it) {
                        const int sl = (int)(it % S);
                        mbar_wait(&full[sl], (unsigned)((it / S) & 1));
                        const double2* src = reinterpret_cast<const double2*>(ring + (size_t)sl * R) + tid;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk)
                            if ((int64_t)s * R + kk * 512 + 2 * tid < m) {
                                const double2 v = src[kk * 256];
                                acc8[c] = fma(v.x, rr[s * 8 + kk].x, acc8[c]);
                                acc8[c] = fma(v.y, rr[s * 8 + kk].y, acc8[c]);
                            }
                        __syncthreads();
                        if (tid == 0 && it + S < total) issue(it + S);
                    }
                }
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) tot += acc8[c];
        }
        if (tot == 123.456) out[0] = tot;
        return;
    }
    for (int64_t c = 0; c < j1 - j0; ++c) {
#pragma unroll
        for (int s = 0; s < NSC; ++s, ++it) {
            const int sl = (int)(it % S);
            mbar_wait(&full[sl], (unsigned)((it / S) & 1));
            const double2* src = reinterpret_cast<const double2*>(ring + (size_t)sl * R) + tid;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                if ((int64_t)s * R + kk * 512 + 2 * tid < m) {
                    const double2 v = src[kk * 256];
                    if (FMA) { acc = fma(v.x, rr[s * 8 + kk].x, acc); acc = fma(v.y, rr[s * 8 + kk].y, acc); }
                    else acc += v.x + v.y;
                }
            }
            __syncthreads();
            if (tid == 0 && it + S < total) issue(it + S);
        }
        tot += acc; acc = 0.0;
    }
    if (tot == 123.456) out[0] = tot;
}

template <typename F>
float timeit(F f, int reps)
{
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

__global__ void fill_random(double* a, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned long long z = (i + 1) * 0x9E3779B97F4A7C15ull;        // splitmix64
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        a[i] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
}

int main(int argc, char** argv)
{
    const size_t bytes = 1600000000ull;     // the C2 matrix
    const size_t n = bytes / 8;
    double* a; double* out;
    cudaMalloc(&a, bytes); cudaMalloc(&out, 8);
    cudaMemset(a, 0, bytes);
    const bool rnd = argc > 1 && argv[1][0] == 'r';   // "r": fill with pseudo-random doubles (no zero pages)
    if (rnd) { fill_random<<<1184, 256>>>(a, n); cudaDeviceSynchronize(); }
    printf("# data: %s\n", rnd ? "pseudo-random doubles in [-1, 1)" : "zeros (cudaMemset)");
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const double2* a2 = reinterpret_cast<const double2*>(a);
    auto rep = [&](const char* name, float ms) { printf("%-36s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
    {
        const size_t smem = 4 * 32768;
        cudaFuncSetAttribute(seg_stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(seg_stream<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        auto rep0 = [&](const char* name, float ms) { printf("%-36s %8.1f us  %7.1f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9); };
        rep0("seg_stream sum 4x32KB (C2 columns)", timeit([&] { seg_stream<0><<<sms, 256, smem>>>(a, 20000, 10000, out); }, 10));
        rep0("seg_stream fma 4x32KB (C2 columns)", timeit([&] { seg_stream<1><<<sms, 256, smem>>>(a, 20000, 10000, out); }, 10));
        cudaFuncSetAttribute(seg_stream<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(seg_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        rep0("seg_stream fma, r' from global", timeit([&] { seg_stream<2><<<sms, 256, smem>>>(a, 20000, 10000, out); }, 10));
        rep0("seg_stream fma, r' global, 8 acc", timeit([&] { seg_stream<3><<<sms, 256, smem>>>(a, 20000, 10000, out); }, 10));
    }
    for (int k : {1, 2, 4, 8}) {
        char nm[64];
        snprintf(nm, 64, "ldg_sum<4> grid=%dx%d tpb=256", sms, k);
        rep(nm, timeit([&] { ldg_sum<4><<<sms * k, 256>>>(a2, n / 2, out); }, 10));
        snprintf(nm, 64, "ldg_sum<8> grid=%dx%d tpb=256", sms, k);
        rep(nm, timeit([&] { ldg_sum<8><<<sms * k, 256>>>(a2, n / 2, out); }, 10));
        snprintf(nm, 64, "ldg_chunk<8> grid=%dx%d tpb=256", sms, k);
        rep(nm, timeit([&] { ldg_chunk<8><<<sms * k, 256>>>(a2, n / 2, out); }, 10));
    }
    for (int k : {1, 2, 4}) {
        char nm[64];
        snprintf(nm, 64, "ldg256_sum<2> grid=%dx%d tpb=256", sms, k);
        rep(nm, timeit([&] { ldg256_sum<2><<<sms * k, 256>>>(a, n / 4, out); }, 10));
        snprintf(nm, 64, "ldg256_sum<4> grid=%dx%d tpb=256", sms, k);
        rep(nm, timeit([&] { ldg256_sum<4><<<sms * k, 256>>>(a, n / 4, out); }, 10));
        snprintf(nm, 64, "ldg256_sum<8> grid=%dx%d tpb=256", sms, k);
        rep(nm, timeit([&] { ldg256_sum<8><<<sms * k, 256>>>(a, n / 4, out); }, 10));
    }
    rep("ldg_chunk<8> grid=148 tpb=512", timeit([&] { ldg_chunk<8><<<sms, 512>>>(a2, n / 2, out); }, 10));
    rep("ldg_chunk<16> grid=148 tpb=512", timeit([&] { ldg_chunk<16><<<sms, 512>>>(a2, n / 2, out); }, 10));
    rep("ldg_chunk<8> grid=148 tpb=1024", timeit([&] { ldg_chunk<8><<<sms, 1024>>>(a2, n / 2, out); }, 10));
    {
        constexpr int S = 4, B = 32768;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 4x32KB 1CTA/SM tpb=256", timeit([&] { bulk_sum<S, B><<<sms, 256, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 6, B = 32768;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 6x32KB 1CTA/SM tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 4, B = 16384;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 4x16KB 2CTA/SM tpb=256", timeit([&] { bulk_sum<S, B><<<sms * 2, 256, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 3, B = 16384;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 3x16KB 1CTA/SM tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
        rep("bulk 3x16KB 1CTA/SM tpb=256", timeit([&] { bulk_sum<S, B><<<sms, 256, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 4, B = 12288;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 4x12KB 1CTA/SM tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 2, B = 24576;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 2x24KB 1CTA/SM tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 8, B = 8192;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 8x8KB 1CTA/SM tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
        rep("bulk 8x8KB 1CTA/SM tpb=256", timeit([&] { bulk_sum<S, B><<<sms, 256, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 6, B = 8192;
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, S * B);
        rep("bulk 6x8KB 1CTA/SM tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
    }
    {
        constexpr int S = 4, B = 32768;
        cudaFuncSetAttribute(bulk_sum_cl<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        rep("bulk 4x32KB cluster2 smem128K tpb=512", timeit([&] { bulk_sum_cl<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
        rep("bulk 4x32KB cluster2 smem200K tpb=512", timeit([&] { bulk_sum_cl<S, B><<<sms, 512, 200 * 1024>>>(a, n, out); }, 10));
        cudaFuncSetAttribute(bulk_sum<S, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        rep("bulk 4x32KB nocluster smem200K tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, 200 * 1024>>>(a, n, out); }, 10));
        rep("bulk 4x32KB nocluster smem128K tpb=512", timeit([&] { bulk_sum<S, B><<<sms, 512, S * B>>>(a, n, out); }, 10));
    }
    // copy reference (cudaMemcpy D2D, read+write counted)
    double* b; cudaMalloc(&b, bytes / 2);
    float ms = timeit([&] { cudaMemcpyAsync(b, a, bytes / 2, cudaMemcpyDeviceToDevice); }, 10);
    printf("%-36s %8.1f us  %7.1f GB/s (read+write)\n", "memcpy D2D 0.8GB", ms * 1e3, bytes / (ms * 1e-3) / 1e9);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
