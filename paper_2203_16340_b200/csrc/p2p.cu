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
// The consumer side is the prologue of the consuming kernel (k_dir_decide,
// k_ls, k_gram_decide, k_kkt_decide; p2p_wait_take in common.cuh): one thread
// spins (acquire, system scope) until the local counter reaches the count
// this exchange adds, then the kernel reduces the gathered packs in rank
// order exactly as after the NCCL all-gather -- the bytes and their order
// are the same, so the P2P and NCCL exchanges give bit-identical solves.
#include "common.cuh"

namespace lb {

// Stand-alone put of one section (the rare host-driven paths: the Armijo
// continuation's separable sums).  One CTA.
__global__ void __launch_bounds__(NT) k_p2p_put(Prob P, int sec, int64_t off, int64_t cnt)
{
    p2p_push(P, sec, off, cnt);
}

void launch_p2p_put(const Prob& P, cudaStream_t st, int sec, int64_t off, int64_t cnt)
{
    k_p2p_put<<<1, NT, 0, st>>>(P, sec, off, cnt);
}

// Quiescence barrier of the host-driven stall paths (R14 fallback relaunch,
// Armijo continuation).  Inside a replayed iteration a rank cannot push a
// section again before every peer has read it (the next push follows a
// consumption of a later section the peer sends only after reading), but a
// relaunch decided on the host would re-push DIR / QS at once.  So before it
// every rank first ACKs (its stream has finished every consumer kernel
// launched so far) into every mailbox's barrier counter, then waits until
// all ranks have ACKed: after the wait no rank still reads a slot the
// relaunch overwrites.  Two kernels so that a loopback group on one stream
// (all ranks' ACKs enqueued before any wait) cannot deadlock.
__global__ void k_p2p_ack(Prob P)
{
    __threadfence_system();
    p2p_signal(P, MB_BARRIER);
}

__global__ void k_p2p_wait_ack(Prob P)
{
    p2p_wait_take(P, MB_BARRIER, (unsigned long long)P.nranks);
}

void launch_p2p_barrier(const Prob* Ps, int n, cudaStream_t st)
{
    for (int i = 0; i < n; ++i) k_p2p_ack<<<1, 1, 0, st>>>(Ps[i]);
    for (int i = 0; i < n; ++i) k_p2p_wait_ack<<<1, 1, 0, st>>>(Ps[i]);
}

}  // namespace lb
