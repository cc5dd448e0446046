// pfb_nll_prod.cuh -- product-mode NLL kernel for transcendental-bound models.
//
// -sum_i ln p_i equals -ln prod_i p_i.  For models whose per-event density
// costs exponentials anyway (SumPdf C1/C5, Dalitz C3/C4) the kernel evaluates
// p_i in the linear domain -- the reference's own formula, pdf.py:205-227 /
// dalitz.py:217-230 -- and multiplies: one log per 16 events instead of one
// per event.
//
// Canonical structure of one 4096-event block (independent of warps per
// block P, of grid size and of GPU count, so every invariance the reference
// tests -- serial == pool == shards -- holds bit for bit):
//   row r = e / 64 (64 rows), column = e % 64, thread column = 2*lane + {0,1};
//   unit u = rows [8u, 8u+8) x one lane's 2 columns = 16 events;
//   unit value  v(u, lane) = -(ln m + ex ln 2)  with  m 2^ex = prod p  (rows in
//   ascending order, x then y, renormalised to m in [1, 2) after every row);
//   block value = lane tree (shuffle-down 16..1) of the unit tree
//   ((v0+v1)+(v2+v3))+((v4+v5)+(v6+v7)).
// A ragged tail block uses the same structure with p = 1 for absent events.
//
// Guard: an event is certified when its p lies in [2^-500, 2^500] (so every
// partial product is a normal double and the reference's p is far from 0 and
// inf) and the evaluator reports no out-of-range intermediate.  A block with
// any uncertified event is deferred to the exact fix-up launch (literal
// reference arithmetic, reference errors) exactly like the log-domain kernel.
//
// Accuracy: the product of 16 correctly-rounded factors has relative error
// <= 16 u, i.e. an absolute error <= 4e-15 in each unit's -ln -- orders of
// magnitude inside the 1e-10 relative NLL tolerance.
#pragma once
#include "pfb_nll_kernel.cuh"

namespace pfb {

// ln 2 split so that ex * kLn2Hi is exact for |ex| < 2^21 (fdlibm split).
static constexpr double kLn2Hi = 6.93147180369123816490e-01;
static constexpr double kLn2Lo = 1.90821492927058770002e-10;

// p in [2^-500, 2^500]: biased exponent in [523, 1523]; 0, subnormal, negative,
// inf and NaN all fail.
__device__ __forceinline__ bool p_in_range(double p) {
    const int hi = __double2hiint(p);
    return (unsigned)((hi >> 20) - 523) <= 1000u;
}

// m * 2^ex  ->  m in [1, 2), exponent moved into ex (m positive normal).
__device__ __forceinline__ void renorm(double& m, int& ex) {
    const int hi = __double2hiint(m);
    ex += (hi >> 20) - 1023;
    m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(m));
}

// SumPdf(gaussian, exponential) on one column (C1 / C5), linear domain:
//   p = c0 exp((-0.5 z) z) + c1 exp(alpha x),  z = (x - mu) / sigma,
//   c_t = weight_t / (norm_t * norm_root)  (pdf.py:122-127, 141-144, 205-219).
// Leaf/term layout fixed by the dispatcher: leaf 0 gaussian (ptv[0][0..1] =
// mu, 1/sigma), leaf 1 exponential (ptv[0][2] = alpha), term t = leaf t.
// A subnormal term is negligible next to a certified p when |ln c_t| < 200
// (checked by the dispatcher), so no per-leaf guard is needed.
struct EvSum2GE {
    static constexpr int NC = 1;
    static constexpr int U = 4;
    static constexpr int MINB = 3;

    __device__ static __forceinline__ double one(const NllArgs& A, double x) {
        const double z = (x - A.ptv[0][0]) * A.ptv[0][1];
        const double g = exp((-0.5 * z) * z);
        const double e = exp(A.ptv[0][2] * x);
        return fma(A.term[0].coef, g, A.term[1].coef * e);
    }

    __device__ static __forceinline__ double2 prob2(const NllArgs& A, const double2 (&x)[1], bool& okx,
                                                    bool& oky) {
        okx = oky = true;
        return make_double2(one(A, x[0].x), one(A, x[0].y));
    }
};

template <int P, class Ev>
__global__ void __launch_bounds__(kThreads, Ev::MINB) nll_prod_kernel(const __grid_constant__ NllArgs A) {
    static_assert(P == 1 || P == 2 || P == 4 || P == 8, "P");
    constexpr int NC = Ev::NC;
    constexpr int GROUPS = kThreads / (32 * P);
    constexpr int ROWS = 64 / P;  // rows per warp
    constexpr int W = Ev::U;      // row loads kept in flight
    static_assert(W <= ROWS, "window");

    __shared__ double xch[GROUPS][8][32];
    __shared__ int xbad[GROUPS][P];
    __shared__ long long s_item[GROUPS];
    __shared__ long long sacc[PFB_ACC_WORDS];
    __shared__ unsigned int s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int grp = warp / P;
    const int wig = warp % P;
    for (int i = tid; i < PFB_ACC_WORDS; i += blockDim.x) sacc[i] = 0;
    __syncthreads();

    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    const int r0 = wig * ROWS;
    for (;;) {
        if (wig == 0 && lane == 0) s_item[grp] = (long long)atomicAdd(A.work_counter, 1ull);
        group_sync<P>(grp);
        const int64_t it = s_item[grp];
        group_sync<P>(grp);
        if (it >= nitems) break;
        const bool is_tail = A.tail && it == 0;
        const int64_t bidx = is_tail ? A.nfull : it - (A.tail ? 1 : 0);
        const int64_t lbase = bidx * (int64_t)kBlock;
        const int n = is_tail ? A.tail : kBlock;
        const double* col[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) col[c] = A.col[c] + A.begin + lbase;

        auto load = [&](int row, double2 (&dst)[NC]) {
            const int e = row * 64 + 2 * lane;
            if (!is_tail || e + 1 < n) {
#pragma unroll
                for (int c = 0; c < NC; ++c) dst[c] = ld2(col[c] + e);
            } else {  // ragged tail: a lone last event, or a stand-in (masked below)
                const int j = e < n ? e : 0;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double v = __ldg(col[c] + j);
                    dst[c] = make_double2(v, v);
                }
            }
        };

        double2 win[W][NC];
#pragma unroll
        for (int q = 0; q < W; ++q) load(r0 + q, win[q]);
        double m = 1.0;
        int ex = 0;
        bool bad = false;
#pragma unroll 1
        for (int i = 0; i < ROWS; ++i) {
            double2 cur[NC];
#pragma unroll
            for (int c = 0; c < NC; ++c) cur[c] = win[0][c];
#pragma unroll
            for (int q = 0; q + 1 < W; ++q)
#pragma unroll
                for (int c = 0; c < NC; ++c) win[q][c] = win[q + 1][c];
            if (i + W < ROWS) load(r0 + i + W, win[W - 1]);
            bool okx, oky;
            double2 p = Ev::prob2(A, cur, okx, oky);
            if (is_tail) {
                const int e = (r0 + i) * 64 + 2 * lane;
                if (e >= n) {
                    p.x = 1.0;
                    okx = true;
                }
                if (e + 1 >= n) {
                    p.y = 1.0;
                    oky = true;
                }
            }
            bad |= !(okx && oky && p_in_range(p.x) && p_in_range(p.y));
            m = (m * p.x) * p.y;
            renorm(m, ex);
            if ((i & 7) == 7) {
                const double fe = (double)ex;
                xch[grp][(r0 + i) >> 3][lane] = -fma(fe, kLn2Hi, fma(fe, kLn2Lo, log(m)));
                m = 1.0;
                ex = 0;
            }
        }
        const unsigned anybad = __any_sync(0xffffffffu, bad);
        if (lane == 0) xbad[grp][wig] = anybad ? 1 : 0;
        group_sync<P>(grp);
        bad = false;
#pragma unroll
        for (int w = 0; w < P; ++w) bad |= xbad[grp][w] != 0;
        double bsum = 0.0;
        if (wig == 0 && !bad) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = xch[grp][u][lane];
            double T = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
#pragma unroll
            for (int off = 16; off >= 1; off /= 2) T = T + __shfl_down_sync(0xffffffffu, T, off);
            bsum = T;
        }
        group_sync<P>(grp);  // xch / xbad reused by the next item
        if (wig == 0 && lane == 0) {
            if (bad) {  // defer the whole block to the exact fix-up launch
                const unsigned long long slot = atomicAdd(A.fix_counter, 1ull);
                A.fix_list[slot] = (A.block_base + bidx) * kMaxPts + A.fix_point;
            } else {
                if (A.block_sums) A.block_sums[A.block_base + bidx] = bsum;
                acc_add_shared(sacc, bsum);
            }
        }
    }
    finish_launch<false>(A, sacc, &s_last);
}

template <int P, class Ev>
static cudaError_t launch_prod_one(const NllArgs& A, cudaStream_t stream, int sm_count) {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nll_prod_kernel<P, Ev>, kThreads, 0);
        if (occ < 1) occ = 1;
    }
    constexpr int GROUPS = kThreads / (32 * P);
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    int64_t grid = (nitems + GROUPS - 1) / GROUPS;
    const int64_t cap = (int64_t)sm_count * occ;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    nll_prod_kernel<P, Ev><<<(unsigned)grid, kThreads, 0, stream>>>(A);
    return cudaGetLastError();
}

// Block values do not depend on P (see the header), so A.warps is a pure
// tuning knob here too.
template <class Ev>
static cudaError_t launch_prod(const NllArgs& A, cudaStream_t stream, int sm_count) {
    switch (A.warps) {
        case 1:
            return launch_prod_one<1, Ev>(A, stream, sm_count);
        case 2:
            return launch_prod_one<2, Ev>(A, stream, sm_count);
        case 4:
            return launch_prod_one<4, Ev>(A, stream, sm_count);
        default:
            return launch_prod_one<8, Ev>(A, stream, sm_count);
    }
}

}  // namespace pfb
