// pfb_nll_task.cuh -- warp-task product-mode NLL kernel (C1 / C5 SumPdf).
//
// The canonical block structure of pfb_nll_prod.cuh is unchanged: a
// 4096-event block is 8 unit rows of 512 events (row w = events
// [512w, 512w + 512)), each row's 32 lanes produce one unit value (8 rows of
// 2 events per lane, product mode), and the block value is the lane tree of
// the unit tree -- so every NLL this kernel returns is bitwise the bulk /
// TMA / SIMT product kernels' NLL.
//
// What changes is the schedule.  The work is T = 8 x blocks warp TASKS
// (block, unit row) of identical cost.  One CTA per SM (24 warps); CTA c owns
// the contiguous task range [c T / G, (c+1) T / G) -- equal shares, no global
// work counter -- and its warps claim tasks from that range through a shared
// counter, one task ahead: each warp bulk-copies its next task's 4 KB
// (cp.async.bulk, one mbarrier per buffer) while it computes the current one.
// No warp ever waits for a sibling except at the very end, so the tail of a
// launch is one task (512 events), not one block per 8-warp group (the bulk
// kernel lost ~1/4 of its samples at its end-of-launch barrier, ncu).
//   * a block whose 8 tasks all lie inside one CTA's range folds through a
//     shared-memory ring (last of the 8 to post folds; a slot is reused only
//     after its previous fold is published, as in nll_prod_bulk_kernel);
//   * a block split between CTAs (at most two per CTA boundary) folds through
//     a global slot: the 8 posts land in gfold/gbad, a release fence, a
//     global arrival counter; the last arriver folds and resets the counter.
#pragma once
#include "pfb_nll_prod.cuh"

namespace pfb {

constexpr int kTaskWarps = 24;
constexpr int kTaskThreads = 32 * kTaskWarps;
constexpr int kTaskRing = 8;  // shared fold slots (blocks in flight per CTA)

template <class Ev>
__global__ void __launch_bounds__(kTaskThreads, 1) nll_task_kernel(const __grid_constant__ NllArgs A) {
    constexpr int NC = Ev::NC;
    extern __shared__ __align__(128) double tbuf[];  // [warps][2 buffers][NC][512]
    __shared__ unsigned long long bar[kTaskWarps][2];
    __shared__ double xch[kTaskRing][8][32];
    __shared__ int xbad[kTaskRing][8];
    __shared__ unsigned int s_cnt[kTaskRing];
    __shared__ int s_done[kTaskRing];
    __shared__ long long sacc[PFB_ACC_WORDS];
    __shared__ double s_tab[kTabN];
    __shared__ unsigned long long s_next;
    __shared__ unsigned int s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int w = tid >> 5;
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    const int64_t T = 8 * nitems;
    const int64_t t_begin = (int64_t)blockIdx.x * T / gridDim.x;
    const int64_t t_end = ((int64_t)blockIdx.x + 1) * T / gridDim.x;
    // the first task of this warp is fixed (no claim latency before the first copy)
    const int64_t t_first = t_begin + w;

    double* mybuf = tbuf + (int64_t)w * 2 * NC * kUnitEvents;
    // task t = (block t / 8, unit row t % 8); the ragged tail is the last block
    auto issue = [&](int64_t t, int b) {
        const int64_t bidx = t >> 3;
        const int row = (int)(t & 7);
        const bool tail = A.tail && bidx == A.nfull;
        const int n = tail ? A.tail : kBlock;
        int nw = n - kUnitEvents * row;
        nw = nw < 0 ? 0 : (nw > kUnitEvents ? kUnitEvents : nw);
        const unsigned bytes = 8u * (unsigned)(nw & ~1);
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar[w][b], bytes * NC);
            if (bytes) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    bulk_g2s(mybuf + (b * NC + c) * kUnitEvents,
                             A.col[c] + A.begin + bidx * (int64_t)kBlock + kUnitEvents * row, bytes, &bar[w][b]);
            }
        }
    };

    if (lane == 0) {
        mbar_init(&bar[w][0], 1);
        mbar_init(&bar[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (t_first < t_end) issue(t_first, 0);  // before the CTA-wide set-up
    for (int i = tid; i < PFB_ACC_WORDS; i += kTaskThreads) sacc[i] = 0;
    init_tab<Ev>(A, s_tab, tid);
    if (tid < kTaskRing) {
        s_cnt[tid] = 0u;
        s_done[tid] = 0;
    }
    if (tid == 0) s_next = (unsigned long long)(t_begin + kTaskWarps);
    __syncthreads();

    // blocks wholly inside [t_begin, t_end) fold in shared memory; j = local
    // index of such a block (blocks are claimed in order, so ring slot j % R)
    const int64_t b_own0 = (t_begin + 7) >> 3;  // first wholly-owned block
    const int64_t b_own1 = t_end >> 3;          // one past the last
    int64_t t = t_first;
    int k = 0;  // tasks done by this warp
    while (t < t_end) {
        const int b = k & 1;
        unsigned long long tn = 0;
        if (lane == 0) tn = atomicAdd(&s_next, 1ull);
        const int64_t t_next = (int64_t)__shfl_sync(0xffffffffu, tn, 0);
        if (t_next < t_end) {
            __syncwarp();
            fence_proxy_async_smem();  // buffer b^1 was read (generic proxy) in the previous task
            issue(t_next, b ^ 1);
        }
        mbar_wait(&bar[w][b], (k >> 1) & 1);
        const int64_t bidx = t >> 3;
        const int row = (int)(t & 7);
        const double* xb = mybuf + b * NC * kUnitEvents;
        const bool tail = A.tail && bidx == A.nfull;
        Unit un;
        bool bad = false;
        if (!tail) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double2 x[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    x[c] = *reinterpret_cast<const double2*>(xb + c * kUnitEvents + r * 64 + 2 * lane);
                prod_row<Ev, false>(A, x, 0, kBlock, un, bad, s_tab, (r & 1) != 0);
            }
        } else {
            const int n = A.tail;
            const int64_t gbase = A.begin + bidx * (int64_t)kBlock;
#pragma unroll 1
            for (int r = 0; r < 8; ++r) {
                const int le = r * 64 + 2 * lane;
                const int e = kUnitEvents * row + le;
                double2 x[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    if (e + 1 < n) {
                        x[c] = *reinterpret_cast<const double2*>(xb + c * kUnitEvents + le);
                    } else {  // odd last event (not bulk-copied) or a stand-in
                        const double v = __ldg(A.col[c] + gbase + (e < n ? e : 0));
                        x[c] = make_double2(v, v);
                    }
                }
                prod_row<Ev, true>(A, x, e, n, un, bad, s_tab);
            }
        }
        bad |= !unit_in_range(un, IsRatio<Ev>::value);
        const double uval = unit_value<Ev>(A, un);
        const unsigned anybad = __any_sync(0xffffffffu, bad);
        // block fold: the last of the block's 8 tasks to post folds it
        auto fold_block = [&](auto load, int slot, bool shared_slot) {
            bool fbad = false;
#pragma unroll
            for (int q = 0; q < 8; ++q) fbad |= load(1, q) != 0.0;
            double bsum = 0.0;
            if (!fbad) {
                double v[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) v[q] = load(0, q * 32 + lane);
                double S = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
#pragma unroll
                for (int off = 16; off >= 1; off /= 2) S = S + __shfl_down_sync(0xffffffffu, S, off);
                bsum = S;
            }
            __syncwarp();
            if (lane == 0) {
                if (fbad) {
                    const unsigned long long fs = atomicAdd(A.fix_counter, 1ull);
                    A.fix_list[fs] = (A.block_base + bidx) * kMaxPts + A.fix_point;
                } else {
                    if (A.block_sums) A.block_sums[A.block_base + bidx] = bsum;
                    acc_add_shared(sacc, bsum);
                }
                if (shared_slot) {
                    s_cnt[slot] = 0u;
                    __threadfence_block();
                    st_volatile(&s_done[slot], (int)((bidx - b_own0) / kTaskRing) + 1);
                } else {
                    A.gcnt[bidx] = 0u;  // self-resetting for the next launch
                }
            }
        };
        if (bidx >= b_own0 && bidx < b_own1) {
            const int64_t j = bidx - b_own0;
            const int slot = (int)(j % kTaskRing);
            if (lane == 0)
                while (ld_volatile(&s_done[slot]) < (int)(j / kTaskRing)) __nanosleep(32);
            __syncwarp();
            xch[slot][row][lane] = uval;
            if (lane == 0) xbad[slot][row] = anybad ? 1 : 0;
            __syncwarp();
            unsigned arrived = 0;
            if (lane == 0) {
                __threadfence_block();
                arrived = atomicAdd(&s_cnt[slot], 1u);
            }
            arrived = __shfl_sync(0xffffffffu, arrived, 0);
            if (arrived == 7) {
                __threadfence_block();
                fold_block([&](int which, int i) -> double {
                    return which ? (double)ld_volatile(&xbad[slot][i]) : ld_volatile(&xch[slot][0][0] + i);
                }, slot, true);
            }
        } else {
            // a block shared with a neighbouring CTA: global slot, release /
            // acquire through gcnt
            double* gv = A.gfold + bidx * 256;
            int* gb = A.gbad + bidx * 8;
            gv[row * 32 + lane] = uval;
            if (lane == 0) gb[row] = anybad ? 1 : 0;
            __threadfence();
            __syncwarp();
            unsigned arrived = 0;
            if (lane == 0) arrived = atomicAdd(A.gcnt + bidx, 1u);
            arrived = __shfl_sync(0xffffffffu, arrived, 0);
            if (arrived == 7) {
                __threadfence();
                fold_block([&](int which, int i) -> double {
                    return which ? (double)__ldcg(gb + i) : __ldcg(gv + i);
                }, 0, false);
            }
        }
        t = t_next;
        ++k;
    }
    finish_launch<false>(A, sacc, &s_last);
}

template <class Ev>
static cudaError_t launch_task(const NllArgs& A, cudaStream_t stream, int sm_count) {
    constexpr int NC = Ev::NC;
    const size_t smem = (size_t)kTaskWarps * 2 * NC * kUnitEvents * sizeof(double);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(nll_task_kernel<Ev>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int64_t tasks = 8 * (A.nfull + (A.tail ? 1 : 0));
    int64_t grid = sm_count;
    const int64_t need = (tasks + kTaskWarps - 1) / kTaskWarps;
    if (grid > need) grid = need > 0 ? need : 1;
    nll_task_kernel<Ev><<<(unsigned)grid, kTaskThreads, smem, stream>>>(A);
    return cudaGetLastError();
}

}  // namespace pfb
