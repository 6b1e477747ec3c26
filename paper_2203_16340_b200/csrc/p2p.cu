// p2p.cu -- a9 of SURVEY.md 8(a)/8(e): the cross-GPU exchange of the
// column-sharded solve over peer memory, without NCCL.
//
// Every rank owns a mailbox (one cudaMalloc, exported with CUDA IPC and
// mapped by every peer): a header of section counters
// and the four gathered sections [R][qs_len] | [R][4] | [R][GRAM_STRIDE] |
// [R][4] in pack order.  The PRODUCING kernels' tails store their pack
// straight into slot [rank] of every mailbox and bump the section counter
// of every mailbox (p2p_push / the k_fwd row-block tail, common.cuh and
// kernels.cu): the m-length q partial of a1 leaves each row block's CTA the
// moment its rows are final, so the transfer overlaps the rest of the GEMV.
// The consumer side is k_p2p_wait: one thread spins (acquire, system scope)
// until the local counter reaches the count this exchange adds, then the
// *_decide kernel behind it reduces the gathered packs in rank order exactly
// as after the NCCL all-gather -- the bytes and their order are the same, so
// the P2P and NCCL exchanges give bit-identical solves.
#include "common.cuh"

namespace lb {

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

// Wait until `inc` more signals of section `sec` have arrived.  iter: skip
// when the solve is halted (every rank skips the producer identically).  A
// peer that never signals (it died, or the protocol diverged) trips the
// timeout flag in the header after 60 s instead of hanging the GPU.
__global__ void k_p2p_wait(Prob P, int sec, int inc, int iter)
{
    if (iter && halted(P.ctrl)) return;
    if (threadIdx.x != 0) return;
    const unsigned long long tgt = P.p2p_tgt[sec] + (unsigned long long)inc;
    const unsigned long long t0 = globaltimer_ns();
    while (ld_acquire_sys(P.mb_hdr + sec) < tgt) {
        __nanosleep(100);
        if (globaltimer_ns() - t0 > 60000000000ULL) { atomicExch(P.mb_hdr + 4, 1ULL); break; }
    }
    P.p2p_tgt[sec] = tgt;
    __threadfence();
}

// Stand-alone put of one section (the rare host-driven paths: the Armijo
// continuation's separable sums).  One CTA.
__global__ void __launch_bounds__(NT) k_p2p_put(Prob P, int sec, int64_t off, int64_t cnt)
{
    p2p_push(P, sec, off, cnt);
}

void launch_p2p_wait(const Prob& P, cudaStream_t st, int sec, int inc, int iter)
{
    k_p2p_wait<<<1, 32, 0, st>>>(P, sec, inc, iter);
}

void launch_p2p_put(const Prob& P, cudaStream_t st, int sec, int64_t off, int64_t cnt)
{
    k_p2p_put<<<1, NT, 0, st>>>(P, sec, off, cnt);
}

}  // namespace lb
