// pfb_nll_tma.cuh -- TMA-pipelined NLL kernel for the HBM-bound evaluators.
//
// One CTA per SM: a producer warp streams whole 4096-event column blocks
// into an S-stage shared-memory ring with cp.async.bulk (the TMA bulk-copy
// engine; completion tracked by mbarrier transaction counts), and sixteen
// consumer warps evaluate -ln p from shared memory and fold each block with
// the same reference-order tree as nll_kernel (element e = 2*lane + {0,1} +
// 64*w + 64*16*k; slots k streamed in bit-reversed order through a binary
// counter, then warps, lanes, x+y).  Stages are released as soon as the
// consumers have read them, so the copy engine always has S-1 blocks of
// prefetch in flight and no thread spends registers or issue slots on loads.
// The consumers never wait for each other: each posts its partial tree into a
// fold slot and the last of the sixteen to arrive folds the block.
//
// Blocks are handed out by the producer from the device work counter
// (dynamic: measured 1.2x faster than a static round-robin split); the
// ragged tail (item 0) is copied like any block and its terms are written in
// place before the split recursion.  Blocks holding an event the fast
// evaluator cannot certify are deferred to the exact fix-up launch, exactly
// as in nll_kernel.
#pragma once

#include "pfb_nll_kernel.cuh"

namespace pfb {

constexpr int kTmaConsumers = 16;                  // consumer warps = one block tree
constexpr int kTmaThreads = 32 * (kTmaConsumers + 1);
constexpr int kTmaRing = 2;  // block-fold slots (warp drift bound; 8 KB each, shared memory is full)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

#ifndef PFB_WAIT_HINT_NS
#define PFB_WAIT_HINT_NS 20000
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "PFB_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra PFB_WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// The same wait with a suspend-time hint: the waiting thread is parked until
// the phase completes (or the hint elapses) instead of re-issuing try_wait in
// a tight loop -- for waits that are long and not latency-critical (the
// producer waiting for a free stage while consumers compute) the spin would
// otherwise take issue slots from the consumer warps on its scheduler.
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "PFB_WAITS_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n"
        " @!p bra PFB_WAITS_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"(PFB_WAIT_HINT_NS)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kTmaConsumers) : "memory");
}

// Flush the per-point CTA accumulators; the last CTA exports and resets.
__device__ __forceinline__ void finish_launch_pts(const NllArgs& A, long long* sflat, int nwords,
                                                  unsigned int* s_last) {
    const int tid = threadIdx.x;
    __syncthreads();
    for (int i = tid; i < nwords; i += blockDim.x)
        if (sflat[i]) atomicAdd(A.acc + i, (unsigned long long)sflat[i]);
    __syncthreads();
    if (tid == 0) *s_last = (ticket_acq_rel(A.ticket) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!*s_last) return;
    const int nt = blockDim.x;  // independent round trips on different threads
    if (tid == nt - 1) {
        *A.work_counter = 0ull;
        *A.ticket = 0u;
    }
    if (A.mode == MODE_ACCUM) return;
    if (PFB_PEER_ON && A.peer_world > 0 && A.mode == MODE_EXPORT && nwords == PFB_ACC_WORDS) {
        peer_finish(A);
        return;
    }
    if (tid == nt - 2) A.result_i[0] = (long long)atomicExch(A.fix_counter, 0ull);
    if (tid == nt - 3) A.result_i[1] = (long long)atomicExch(A.errkey, ~0ull);
    for (int i = tid; i < nwords; i += nt) {
        const long long v = (long long)atomicExch(A.acc + i, 0ull);
        if (A.mode == MODE_EXPORT)
            A.acc_out[i] = v;
        else
            A.acc_out[i] += v;
    }
    post_seq(A);
}

template <class Ev, int S>
__global__ void __launch_bounds__(kTmaThreads, 1) nll_tma_kernel(const __grid_constant__ NllArgs A) {
    constexpr int NC = Ev::NC;
    constexpr int KPT = 64 / kTmaConsumers;  // 4 double2 slots per consumer thread
    constexpr int LK = Log2<KPT>::value;
    extern __shared__ __align__(128) double stage[];  // S x NC x 4096 doubles

    __shared__ unsigned long long full_bar[S], empty_bar[S];
    __shared__ long long s_blk[S];
    __shared__ double2 xch[kTmaRing][kTmaConsumers][32];  // warp partial trees per fold slot
    __shared__ int xbad[kTmaRing][kTmaConsumers];
    __shared__ unsigned int s_cnt[kTmaRing];
    __shared__ int s_done[kTmaRing];
    __shared__ int s_tailbad[kTmaConsumers];
    __shared__ long long sacc[kMaxPts][PFB_ACC_WORDS];
    __shared__ unsigned int s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    if (tid == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full_bar[s], 1);
            mbar_init(&empty_bar[s], kTmaConsumers);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < kMaxPts * PFB_ACC_WORDS; i += blockDim.x) (&sacc[0][0])[i] = 0;
    if (tid < kTmaRing) {
        s_cnt[tid] = 0u;
        s_done[tid] = 0;
    }
    __syncthreads();

    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    if (warp == kTmaConsumers) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            // the next item index is fetched one stage ahead, so the device-wide
            // atomic's round trip overlaps the wait for a free stage
            int64_t it_next = (int64_t)atomicAdd(A.work_counter, 1ull);
            for (int u = 0;; ++u) {
                const int s = u % S;
                mbar_wait(&empty_bar[s], ((u / S) & 1) ^ 1);
                const int64_t it = it_next;
                if (it < nitems) it_next = (int64_t)atomicAdd(A.work_counter, 1ull);
                if (it >= nitems) {
                    s_blk[s] = -1;
                    mbar_arrive(&full_bar[s]);
                    break;
                }
                const bool is_tail = A.tail && it == 0;
                const int64_t bidx = is_tail ? A.nfull : it - (A.tail ? 1 : 0);
                s_blk[s] = bidx;
                // bulk copies move multiples of 16 B: an odd tail's last event
                // is read from global memory by the consumers
                const unsigned bytes = is_tail ? (unsigned)(8 * (A.tail & ~1)) : (unsigned)(8 * kBlock);
                mbar_arrive_expect_tx(&full_bar[s], bytes * NC);
                if (bytes) {
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        bulk_g2s(stage + ((int64_t)s * NC + c) * kBlock,
                                 A.col[c] + A.begin + bidx * (int64_t)kBlock, bytes, &full_bar[s]);
                }
            }
        }
    } else {
        // ------------------------------------------------------------ consumers
        // Batched objective: the stage stays resident while every parameter
        // point is folded, so HBM traffic is one pass whatever npts is.
        const int w = warp;
        int f = 0;  // block folds posted by this warp (the same sequence in every warp)
        for (int u = 0;; ++u) {
            const int s = u % S;
            mbar_wait(&full_bar[s], (u / S) & 1);
            const int64_t bidx = s_blk[s];
            if (bidx < 0) break;
            const double* sx = stage + (int64_t)s * NC * kBlock;
            for (int m = 0; m < A.npts; ++m) {
                bool bad = false;
                double bsum = 0.0;
                const bool last_pt = m == A.npts - 1;
                if (A.tail && bidx == A.nfull) {
                    // ragged tail: terms to global scratch, then the split recursion
                    const int n = A.tail;
                    const int64_t lbase = A.nfull * (int64_t)kBlock;
                    for (int e = 2 * (w * 32 + lane); e < n; e += 64 * kTmaConsumers) {
                        const bool pair = e + 1 < n;
                        double2 x[NC];
#pragma unroll
                        for (int c = 0; c < NC; ++c) {
                            if (pair) {
                                x[c] = *reinterpret_cast<const double2*>(sx + c * kBlock + e);
                            } else {
                                const double v = __ldg(A.col[c] + A.begin + lbase + e);
                                x[c] = make_double2(v, v);
                            }
                        }
                        const double2 t = Ev::eval2(A, x, lbase + e, sacc[0], pair ? 2 : 1, bad, m);
                        A.tail_scratch[e] = t.x;
                        if (pair) A.tail_scratch[e + 1] = t.y;
                    }
                    if (last_pt) {  // the stage is no longer read
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty_bar[s]);
                    }
                    const unsigned anybad = __any_sync(0xffffffffu, bad);
                    if (lane == 0) s_tailbad[w] = anybad ? 1 : 0;
                    consumer_sync();
                    bad = false;
#pragma unroll
                    for (int q = 0; q < kTmaConsumers; ++q) bad |= s_tailbad[q] != 0;
                    if (w == 0 && !bad) bsum = pairwise_warp(A.tail_scratch, n, lane);
                    consumer_sync();
                    if (w == 0 && lane == 0) {
                        if (bad) {
                            const unsigned long long slot = atomicAdd(A.fix_counter, 1ull);
                            A.fix_list[slot] = (A.block_base + bidx) * kMaxPts + m;
                        } else {
                            if (A.block_sums && m == 0) A.block_sums[A.block_base + bidx] = bsum;
                            acc_add_shared(sacc[m], bsum);
                        }
                    }
                } else {
                    const int64_t lthr = bidx * (int64_t)kBlock + 2 * lane + 64 * w;
                    const int base = 2 * lane + 64 * w;
                    double2 lvl[LK];
                    double2 T = make_double2(0.0, 0.0);
#pragma unroll
                    for (int i = 0; i < KPT; ++i) {
                        const int k = (int)(__brev((unsigned)i) >> (32 - LK));
                        double2 cur[NC];
#pragma unroll
                        for (int c = 0; c < NC; ++c)
                            cur[c] = *reinterpret_cast<const double2*>(sx + c * kBlock + base +
                                                                       64 * kTmaConsumers * k);
                        double2 v = Ev::eval2(A, cur, lthr + 64 * kTmaConsumers * (int64_t)k, sacc[0], 2, bad, m);
#pragma unroll
                        for (int b = 0; b < LK; ++b) {
                            if ((i >> b) & 1) {
                                v.x = Add(lvl[b].x, v.x);
                                v.y = Add(lvl[b].y, v.y);
                            } else {
                                lvl[b] = v;
                                break;
                            }
                        }
                        T = v;
                    }
                    if (last_pt) {  // this warp is done with the stage: hand it back
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty_bar[s]);
                    }
                    // No barrier: each warp posts its partial tree into fold
                    // slot f % R; the last of the 16 to arrive folds the block.
                    const unsigned anybad = __any_sync(0xffffffffu, bad);
                    const int slot = f % kTmaRing;
                    if (lane == 0)
                        while (*reinterpret_cast<volatile int*>(&s_done[slot]) < f / kTmaRing) __nanosleep(20);
                    __syncwarp();
                    xch[slot][w][lane] = T;
                    unsigned arrived = 0;
                    if (lane == 0) {
                        xbad[slot][w] = anybad ? 1 : 0;
                        __threadfence_block();
                        arrived = atomicAdd(&s_cnt[slot], 1u);
                    }
                    arrived = __shfl_sync(0xffffffffu, arrived, 0);
                    const bool folder = arrived == kTmaConsumers - 1;
                    if (folder) {
                        __threadfence_block();
                        bad = false;
#pragma unroll
                        for (int q = 0; q < kTmaConsumers; ++q) bad |= xbad[slot][q] != 0;
                    }
                    if (folder && !bad) {
                        double2 Wv[kTmaConsumers];
#pragma unroll
                        for (int q = 0; q < kTmaConsumers; ++q) Wv[q] = xch[slot][q][lane];  // after the fence
#pragma unroll
                        for (int h = kTmaConsumers / 2; h >= 1; h /= 2) {
#pragma unroll
                            for (int q = 0; q < h; ++q) {
                                Wv[q].x = Add(Wv[q].x, Wv[q + h].x);
                                Wv[q].y = Add(Wv[q].y, Wv[q + h].y);
                            }
                        }
                        T = Wv[0];
#pragma unroll
                        for (int off = 16; off >= 1; off /= 2) {
                            T.x = Add(T.x, __shfl_down_sync(0xffffffffu, T.x, off));
                            T.y = Add(T.y, __shfl_down_sync(0xffffffffu, T.y, off));
                        }
                        bsum = Add(T.x, T.y);
                    }
                    if (folder) {
                        __syncwarp();
                        if (lane == 0) {
                            if (bad) {  // defer (block, point) to the exact fix-up launch
                                const unsigned long long fs = atomicAdd(A.fix_counter, 1ull);
                                A.fix_list[fs] = (A.block_base + bidx) * kMaxPts + m;
                            } else {
                                if (A.block_sums && m == 0) A.block_sums[A.block_base + bidx] = bsum;
                                acc_add_shared(sacc[m], bsum);
                            }
                            s_cnt[slot] = 0u;
                            __threadfence_block();
                            *reinterpret_cast<volatile int*>(&s_done[slot]) = f / kTmaRing + 1;
                        }
                    }
                    ++f;
                }
            }
        }
    }

    finish_launch_pts(A, &sacc[0][0], A.npts * PFB_ACC_WORDS, &s_last);
}

// Stages: as many NC x 32 KB stages as fit the 227 KB opt-in shared memory.
template <class Ev>
static cudaError_t launch_tma(const NllArgs& A, cudaStream_t stream, int sm_count) {
    constexpr int NC = Ev::NC;
    constexpr int S = NC == 1 ? 6 : (NC == 2 ? 3 : 1);
    const size_t smem = (size_t)S * NC * kBlock * sizeof(double);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(nll_tma_kernel<Ev, S>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    int64_t grid = sm_count;
    if (grid > nitems) grid = nitems > 0 ? nitems : 1;
    nll_tma_kernel<Ev, S><<<(unsigned)grid, kTmaThreads, smem, stream>>>(A);
    return cudaGetLastError();
}

}  // namespace pfb
