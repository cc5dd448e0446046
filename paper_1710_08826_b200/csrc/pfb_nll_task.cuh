// pfb_nll_task.cuh -- warp-task NLL kernels: one-shot (C1 / C5 SumPdf at
// large N) and persistent (any supported plan at small N: the minimiser's
// per-call latency).
//
// The canonical block structure of pfb_nll_prod.cuh is unchanged: a
// 4096-event block is 8 unit rows of 512 events (row w = events
// [512w, 512w + 512)), each row's 32 lanes produce one unit value (8 rows of
// 2 events per lane: product mode, or the row-ordered sum of 16 log-domain
// terms), and the block value is the lane tree of the unit tree -- so every
// NLL these kernels return is bitwise the bulk / TMA / SIMT kernels' NLL.
//
// The schedule: the work is T = 8 x blocks warp TASKS (block, unit row) of
// identical cost.  One CTA per SM; CTA c owns the contiguous task range
// [c T / G, (c+1) T / G) -- equal shares, no global work counter -- and its
// warps claim tasks from that range through a shared counter, one task
// ahead: each warp bulk-copies its next task's NC x 4 KB (cp.async.bulk, one
// mbarrier per buffer) while it computes the current one.  No warp waits for
// a sibling until the end, so the tail of a launch is one task (512 events),
// not one block per 8-warp group.
//   * a block whose 8 tasks all lie inside one CTA's range folds through a
//     shared-memory ring (last of the 8 to post folds; a slot is reused only
//     after its previous fold is published, as in nll_prod_bulk_kernel);
//   * a block split between CTAs (at most two per CTA boundary) folds through
//     a global slot: the 8 posts land in gfold/gbad, a release fence, a
//     global arrival counter; the last arriver folds and resets the counter.
//
// Persistent form (nll_persist_kernel): the same loop inside a kernel that
// stays resident between minimiser calls.  The host writes the call's
// NllArgs into a mapped pinned mailbox and bumps a sequence number (the
// doorbell); CTA 0 polls it over PCIe, copies the mailbox into device memory
// and releases the other CTAs through a global word; every CTA copies the
// arguments into its shared memory and runs the pass; the last CTA exports
// the result into mapped host memory and posts the sequence number.  One
// call costs the doorbell round trip plus the pass -- no launch, no stream
// synchronisation (per-call host floor).
#pragma once
#include "pfb_nll_prod.cuh"

namespace pfb {

constexpr int kTaskWarps = 24;
constexpr int kTaskRing = 8;  // shared fold slots (blocks in flight per CTA)

template <int NC>
struct TaskWarps {
    static constexpr int value = NC == 1 ? 24 : 12;  // 2 x NC x 4 KB per warp in <= 192 KB
};

// Shared state of a task pass (one per CTA).
struct TaskShared {
    double xch[kTaskRing][8][32];
    int xbad[kTaskRing][8];
    unsigned int s_cnt[kTaskRing];
    int s_done[kTaskRing];
    long long sacc[PFB_ACC_WORDS];
    double s_tab[kTabN];
    unsigned long long s_next;
    unsigned int s_last;
};

// task t = (block t / 8, unit row t % 8); the ragged tail is the last block
template <int NC>
__device__ __forceinline__ void task_issue(const NllArgs& A, int64_t t, double* mybuf, unsigned long long* bar,
                                           int lane) {
    const int64_t bidx = t >> 3;
    const int row = (int)(t & 7);
    const bool tail = A.tail && bidx == A.nfull;
    const int n = tail ? A.tail : kBlock;
    int nw = n - kUnitEvents * row;
    nw = nw < 0 ? 0 : (nw > kUnitEvents ? kUnitEvents : nw);
    const unsigned bytes = 8u * (unsigned)(nw & ~1);
    if (lane == 0) {
        mbar_arrive_expect_tx(bar, bytes * NC);
        if (bytes) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
                bulk_g2s(mybuf + c * kUnitEvents, A.col[c] + A.begin + bidx * (int64_t)kBlock + kUnitEvents * row,
                         bytes, bar);
        }
    }
}

// Per-pass reset of the shared state (before the CTA barrier that starts a pass).
template <class Ev, int WARPS>
__device__ __forceinline__ void task_reset(const NllArgs& A, TaskShared& S, int64_t t_begin) {
    const int tid = threadIdx.x;
    for (int i = tid; i < PFB_ACC_WORDS; i += 32 * WARPS) S.sacc[i] = 0;
    init_tab<Ev>(A, S.s_tab, tid);
    if (tid < kTaskRing) {
        S.s_cnt[tid] = 0u;
        S.s_done[tid] = 0;
    }
    if (tid == 0) S.s_next = (unsigned long long)(t_begin + WARPS);
}

// The warp's part of one pass: tasks t_first, then claimed ones, until the
// CTA's range is done.  The first task's copy into buffer (k & 1) must have
// been issued.  k counts this warp's tasks over the kernel's lifetime (the
// mbarrier phases continue across persistent passes).
template <class Ev, bool PROD, int WARPS>
__device__ __forceinline__ void task_loop(const NllArgs& A, TaskShared& S, double* mybuf,
                                          unsigned long long (*bar)[2], int64_t t_first, int64_t t_begin,
                                          int64_t t_end, int& k) {
    constexpr int NC = Ev::NC;
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    // blocks wholly inside [t_begin, t_end) fold in shared memory; j = local
    // index of such a block (blocks are claimed in order, so ring slot j % R)
    const int64_t b_own0 = (t_begin + 7) >> 3;  // first wholly-owned block
    const int64_t b_own1 = t_end >> 3;          // one past the last
    int64_t t = t_first;
    while (t < t_end) {
        const int b = k & 1;
        unsigned long long tn = 0;
        if (lane == 0) tn = atomicAdd(&S.s_next, 1ull);
        const int64_t t_next = (int64_t)__shfl_sync(0xffffffffu, tn, 0);
        if (t_next < t_end) {
            __syncwarp();
            fence_proxy_async_smem();  // buffer b^1 was read (generic proxy) in the previous task
            task_issue<NC>(A, t_next, mybuf + (b ^ 1) * NC * kUnitEvents, &bar[w][b ^ 1], lane);
        }
        mbar_wait(&bar[w][b], (k >> 1) & 1);
        const int64_t bidx = t >> 3;
        const int row = (int)(t & 7);
        const double* xb = mybuf + b * NC * kUnitEvents;
        const bool tail = A.tail && bidx == A.nfull;
        Unit un;
        bool bad = false;
        double acc = 0.0;
        if (!tail) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double2 x[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    x[c] = *reinterpret_cast<const double2*>(xb + c * kUnitEvents + r * 64 + 2 * lane);
                if constexpr (PROD) {
                    prod_row<Ev, false>(A, x, 0, kBlock, un, bad, S.s_tab, (r & 1) != 0);
                } else {
                    const double2 v = Ev::eval2(A, x, 0, S.sacc, 2, bad, 0);
                    acc = (acc + v.x) + v.y;
                }
            }
        } else {
            const int n = A.tail;
            const int64_t gbase = A.begin + bidx * (int64_t)kBlock;
#pragma unroll 1
            for (int r = 0; r < 8; ++r) {
                const int le = r * 64 + 2 * lane;
                const int e = kUnitEvents * row + le;
                if constexpr (!PROD) {
                    if (e >= n) break;  // rows ascend: nothing further in this lane
                }
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
                if constexpr (PROD) {
                    prod_row<Ev, true>(A, x, e, n, un, bad, S.s_tab);
                } else {
                    const int nv = e + 1 < n ? 2 : 1;
                    const double2 v = Ev::eval2(A, x, 0, S.sacc, nv, bad, 0);
                    acc = acc + v.x;
                    if (nv == 2) acc = acc + v.y;
                }
            }
        }
        double uval = acc;
        if constexpr (PROD) {
            bad |= !unit_ok<Ev>(A, un);
            uval = unit_value<Ev>(A, un);
        }
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
                double T = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
#pragma unroll
                for (int off = 16; off >= 1; off /= 2) T = T + __shfl_down_sync(0xffffffffu, T, off);
                bsum = T;
            }
            __syncwarp();
            if (lane == 0) {
                if (fbad) {
                    const unsigned long long fs = atomicAdd(A.fix_counter, 1ull);
                    A.fix_list[fs] = (A.block_base + bidx) * kMaxPts + A.fix_point;
                } else {
                    if (A.block_sums) A.block_sums[A.block_base + bidx] = bsum;
                    acc_add_shared(S.sacc, bsum);
                }
                if (shared_slot) {
                    S.s_cnt[slot] = 0u;
                    __threadfence_block();
                    st_volatile(&S.s_done[slot], (int)((bidx - b_own0) / kTaskRing) + 1);
                } else {
                    A.gcnt[bidx] = 0u;  // self-resetting for the next launch
                }
            }
        };
        if (bidx >= b_own0 && bidx < b_own1) {
            const int64_t j = bidx - b_own0;
            const int slot = (int)(j % kTaskRing);
            if (lane == 0)
                while (ld_volatile(&S.s_done[slot]) < (int)(j / kTaskRing)) __nanosleep(32);
            __syncwarp();
            S.xch[slot][row][lane] = uval;
            if (lane == 0) S.xbad[slot][row] = anybad ? 1 : 0;
            __syncwarp();
            unsigned arrived = 0;
            if (lane == 0) {
                __threadfence_block();
                arrived = atomicAdd(&S.s_cnt[slot], 1u);
            }
            arrived = __shfl_sync(0xffffffffu, arrived, 0);
            if (arrived == 7) {
                __threadfence_block();
                fold_block([&](int which, int i) -> double {
                    return which ? (double)ld_volatile(&S.xbad[slot][i]) : ld_volatile(&S.xch[slot][0][0] + i);
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
}

__device__ __forceinline__ void task_range(int64_t nitems, int64_t& t_begin, int64_t& t_end) {
    const int64_t T = 8 * nitems;
    t_begin = (int64_t)blockIdx.x * T / gridDim.x;
    t_end = ((int64_t)blockIdx.x + 1) * T / gridDim.x;
}

template <class Ev, bool PROD = true>
__global__ void __launch_bounds__(32 * TaskWarps<Ev::NC>::value, 1) nll_task_kernel(const __grid_constant__ NllArgs A) {
    constexpr int NC = Ev::NC;
    constexpr int WARPS = TaskWarps<NC>::value;
    extern __shared__ __align__(128) double tbuf[];  // [warps][2 buffers][NC][512]
    __shared__ unsigned long long bar[WARPS][2];
    __shared__ TaskShared S;

    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    int64_t t_begin, t_end;
    task_range(A.nfull + (A.tail ? 1 : 0), t_begin, t_end);
    const int64_t t_first = t_begin + w;  // fixed: no claim latency before the first copy
    double* mybuf = tbuf + (int64_t)w * 2 * NC * kUnitEvents;
    if (lane == 0) {
        mbar_init(&bar[w][0], 1);
        mbar_init(&bar[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    if (t_first < t_end) task_issue<NC>(A, t_first, mybuf, &bar[w][0], lane);  // before the CTA set-up
    task_reset<Ev, WARPS>(A, S, t_begin);
    __syncthreads();
    int k = 0;
    task_loop<Ev, PROD, WARPS>(A, S, mybuf, bar, t_first, t_begin, t_end, k);
    finish_launch<false>(A, S.sacc, &S.s_last);
}

template <class Ev, bool PROD = true>
static cudaError_t launch_task(const NllArgs& A, cudaStream_t stream, int sm_count) {
    constexpr int NC = Ev::NC;
    constexpr int WARPS = TaskWarps<NC>::value;
    const size_t smem = (size_t)WARPS * 2 * NC * kUnitEvents * sizeof(double);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(nll_task_kernel<Ev, PROD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    const int64_t tasks = 8 * (A.nfull + (A.tail ? 1 : 0));
    int64_t grid = sm_count;
    const int64_t need = (tasks + WARPS - 1) / WARPS;
    if (grid > need) grid = need > 0 ? need : 1;
    nll_task_kernel<Ev, PROD><<<(unsigned)grid, 32 * WARPS, smem, stream>>>(A);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Persistent form.
constexpr int kArgWords = kMaxArgChunks * kArgChunk / 8;
static_assert(sizeof(NllArgs) <= (size_t)kMaxArgChunks * kArgChunk, "mailbox chunks");

template <class Ev, bool PROD = true>
__global__ void __launch_bounds__(32 * TaskWarps<Ev::NC>::value, 1) nll_persist_kernel(const __grid_constant__ PersistCtl P) {
    constexpr int NC = Ev::NC;
    constexpr int WARPS = TaskWarps<NC>::value;
    constexpr int NT = 32 * WARPS;
    constexpr int kChunks = (int)((sizeof(NllArgs) + kArgChunk - 1) / kArgChunk);
    extern __shared__ __align__(128) double tbuf[];
    __shared__ unsigned long long bar[WARPS][2];
    __shared__ TaskShared S;
    // the call's arguments, kept across calls: each call updates the chunks
    // that changed
    __shared__ __align__(16) unsigned char sA_raw[kChunks * kArgChunk];
    __shared__ unsigned int s_idx[kMaxArgChunks];
    __shared__ unsigned long long s_seq, s_op, s_n;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int w = tid >> 5;
    double* mybuf = tbuf + (int64_t)w * 2 * NC * kUnitEvents;
    if (lane == 0) {
        mbar_init(&bar[w][0], 1);
        mbar_init(&bar[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    unsigned long long seen = P.start_seq;
    int k = 0;
    for (;;) {
        // 1. the doorbell: CTA 0 polls the mapped host word, copies the
        //    changed argument chunks to device memory and releases the
        //    others.  With no call for P.idle_ns the kernel leaves by itself
        //    (go[2]), so a forgotten session never holds the GPU (the host
        //    restarts it on demand).
        if (tid == 0) {
            unsigned long long s = seen;
            bool quit = false;
            if (blockIdx.x == 0) {
                unsigned long long t0, now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
                for (;;) {
                    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(s) : "l"(P.host_seq) : "memory");
                    if (s != seen) break;
                    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                    if (now - t0 > P.idle_ns) {
                        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(P.go + 2), "l"(1ull) : "memory");
                        quit = true;
                        break;
                    }
                }
            } else {
                for (;;) {
                    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(s) : "l"(P.go) : "memory");
                    if (s != seen) break;
                    if (__ldcg(P.go + 2)) {
                        quit = true;
                        break;
                    }
                    __nanosleep(32);
                }
            }
            s_seq = s;
            s_op = quit ? 2ull : 0ull;
            if (P.trace && blockIdx.x == 0) P.trace[0] = gtimer();  // doorbell seen
        }
        __syncthreads();
        if (s_op == 2ull) break;  // idle timeout
        if (blockIdx.x == 0) {
            // mailbox header, then the changed chunks (16 B per thread)
            const PersistBox* box = P.host_args;
            if (tid == 0) {
                unsigned long long n, op;
                asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(n) : "l"(&box->nchunks) : "memory");
                asm volatile("ld.relaxed.sys.global.u64 %0, [%1];" : "=l"(op) : "l"(P.host_seq + 1) : "memory");
                s_n = n;
                P.go[1] = op;
                P.dev_chunks[0] = (unsigned int)n;
            }
            if (tid < kMaxArgChunks) {
                unsigned int v;
                asm volatile("ld.relaxed.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(&box->idx[tid]) : "memory");
                s_idx[tid] = v;
                P.dev_chunks[1 + tid] = v;
            }
            __syncthreads();
            const int nparts = (int)s_n * (kArgChunk / 16);
            unsigned char* dst = reinterpret_cast<unsigned char*>(P.dev_args);
            for (int i = tid; i < nparts; i += NT) {
                const int c = i / (kArgChunk / 16), part = i % (kArgChunk / 16);
                unsigned long long a, b;
                asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];"
                             : "=l"(a), "=l"(b)
                             : "l"(&box->payload[c][part * 16])
                             : "memory");
                *reinterpret_cast<ulonglong2*>(dst + (size_t)s_idx[c] * kArgChunk + part * 16) = make_ulonglong2(a, b);
            }
            __syncthreads();
            if (tid == 0) {
                __threadfence();
                asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(P.go), "l"(s_seq) : "memory");
                if (P.trace) P.trace[1] = gtimer();  // arguments copied, CTAs released
            }
        }
        // 2. the changed chunks into this CTA's resident copy (L2, never a stale L1 line)
        if (tid == 0) {
            s_n = __ldcg(P.dev_chunks);
            s_op = __ldcg(P.go + 1);
        }
        if (tid < kMaxArgChunks) s_idx[tid] = __ldcg(P.dev_chunks + 1 + tid);
        __syncthreads();
        {
            const int nparts = (int)s_n * (kArgChunk / 16);
            const unsigned char* src = reinterpret_cast<const unsigned char*>(P.dev_args);
            for (int i = tid; i < nparts; i += NT) {
                const int c = i / (kArgChunk / 16), part = i % (kArgChunk / 16);
                const size_t off = (size_t)s_idx[c] * kArgChunk + part * 16;
                *reinterpret_cast<ulonglong2*>(sA_raw + off) = __ldcg(reinterpret_cast<const ulonglong2*>(src + off));
            }
        }
        __syncthreads();
        seen = s_seq;
        if (s_op != 0) break;  // stop
        // 3. one pass
        const NllArgs& A = *reinterpret_cast<const NllArgs*>(sA_raw);
        int64_t t_begin, t_end;
        task_range(A.nfull + (A.tail ? 1 : 0), t_begin, t_end);
        const int64_t t_first = t_begin + w;
        task_reset<Ev, WARPS>(A, S, t_begin);
        __syncthreads();
        if (P.trace && tid == 0 && blockIdx.x == gridDim.x - 1) P.trace[2] = gtimer();  // last CTA starts its pass
        if (t_first < t_end) {
            __syncwarp();
            fence_proxy_async_smem();
            task_issue<NC>(A, t_first, mybuf + (k & 1) * NC * kUnitEvents, &bar[w][k & 1], lane);
        }
        task_loop<Ev, PROD, WARPS>(A, S, mybuf, bar, t_first, t_begin, t_end, k);
        __syncthreads();
        if (P.trace && tid == 0 && blockIdx.x == gridDim.x - 1) P.trace[3] = gtimer();  // last CTA's pass done
        finish_launch<false>(A, S.sacc, &S.s_last);
        if (P.trace && tid == 0 && S.s_last) P.trace[4] = gtimer();  // result posted
        __syncthreads();
    }
}

template <class Ev, bool PROD = true>
static cudaError_t launch_persist(const PersistCtl& P, cudaStream_t stream, int sm_count) {
    constexpr int NC = Ev::NC;
    constexpr int WARPS = TaskWarps<NC>::value;
    const size_t smem = (size_t)WARPS * 2 * NC * kUnitEvents * sizeof(double);
    static bool configured = false;
    if (!configured) {
        cudaError_t e = cudaFuncSetAttribute(nll_persist_kernel<Ev, PROD>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured = true;
    }
    nll_persist_kernel<Ev, PROD><<<(unsigned)sm_count, 32 * WARPS, smem, stream>>>(P);
    return cudaGetLastError();
}

}  // namespace pfb
