// pfb_peer.cu -- the cross-GPU exchange of the exact accumulator over NVLink
// peer memory, replacing the NCCL all-reduce of 72 int64.
//
// Every rank owns a mailbox in its HBM, exported to the other processes with
// a CUDA IPC handle (exchanged once through torch.distributed).  One call:
// a single-CTA kernel stores this rank's 72 limbs into slot [parity][rank] of
// every peer's mailbox (NVLink P2P stores), fences at system scope, raises
// flag [parity][rank] = seq in every mailbox (release), waits until all
// flags of its own mailbox carry seq (acquire), and sums the world slots in
// rank order -- integer limbs, so the result is the single-GPU accumulator
// bit for bit on every rank.  Parity alternates per call, so a fast rank's
// next call never overwrites a slot a slow rank is still reading.  The wait
// is bounded: a missing peer turns into PFB_E_PEER_TIMEOUT, never a hung GPU.
#include <cstring>

#include "pfb_internal.cuh"

namespace pfb {

// the mailbox layout and the release / acquire helpers are in pfb_internal.cuh
// (shared with the fused exchange in the NLL kernels' epilogue)
struct PeerArgs {
    long long* mbox[kMaxPeers];  // every rank's mailbox (mbox[rank] is local)
    int world, rank;
    unsigned long long seq;
    long long timeout_cycles;
};

__global__ void __launch_bounds__(128) peer_allreduce_kernel(const __grid_constant__ PeerArgs P, long long* acc,
                                                             unsigned long long* status) {
    const int tid = threadIdx.x;
    const int par = (int)(P.seq & 1ull);
    __shared__ int s_timeout;
    if (tid == 0) s_timeout = 0;
    // 1. this rank's limbs into slot [par][rank] of every mailbox
    if (tid < PFB_ACC_WORDS) {
        const long long v = acc[tid];
        for (int q = 0; q < P.world; ++q) peer_slot(P.mbox[q], par, P.rank)[tid] = v;
    }
    __threadfence_system();
    __syncthreads();
    // 2. announce
    if (tid < P.world) st_release_sys(peer_flag(P.mbox[tid], par, P.rank), P.seq);
    // 3. wait for every rank's announcement in the local mailbox (bounded)
    if (tid < P.world) {
        const unsigned long long* f = peer_flag(P.mbox[P.rank], par, tid);
        const long long t0 = clock64();
        while (ld_acquire_sys(f) != P.seq) {
            if (clock64() - t0 > P.timeout_cycles) {
                atomicExch(&s_timeout, 1);
                break;
            }
            __nanosleep(100);
        }
    }
    __syncthreads();
    if (s_timeout) {
        if (tid == 0) *status = 1ull;
        return;
    }
    // 4. the sum over ranks, in rank order (integer: exact)
    if (tid < PFB_ACC_WORDS) {
        long long s = 0;
        for (int q = 0; q < P.world; ++q) s += peer_slot(P.mbox[P.rank], par, q)[tid];
        acc[tid] = s;
    }
    if (tid == 0) *status = 0ull;
}

cudaError_t launch_peer_allreduce(long long* const* mbox, int world, int rank, unsigned long long seq,
                                  long long timeout_cycles, long long* acc, unsigned long long* status,
                                  cudaStream_t stream) {
    PeerArgs P;
    memset(&P, 0, sizeof(P));
    for (int q = 0; q < world && q < kMaxPeers; ++q) P.mbox[q] = mbox[q];
    P.world = world;
    P.rank = rank;
    P.seq = seq;
    P.timeout_cycles = timeout_cycles;
    peer_allreduce_kernel<<<1, 128, 0, stream>>>(P, acc, status);
    return cudaGetLastError();
}

size_t peer_mailbox_bytes() { return peer_mbox_words() * sizeof(long long); }
int peer_max() { return kMaxPeers; }

}  // namespace pfb
