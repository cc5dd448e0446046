// pfb_nll_sop.cu -- sum-of-products (log-domain) instantiations.
// Shape-specialised (exact leaf/term counts and leaf kinds) for the common
// trees -- streamed through the TMA pipeline -- and a generic instantiation
// (<= 4 leaves, <= 4 terms) on the SIMT kernel for the rest.
#include "pfb_nll_prod.cuh"
#include "pfb_nll_task.cuh"
#include "pfb_nll_tma.cuh"

namespace pfb {

#ifndef PFB_TMA1_ITEMS_PER_SM
#define PFB_TMA1_ITEMS_PER_SM 24  // C1 / C5 single points: the TMA unit kernel from ~14.5M events
#endif

static constexpr int kG = PFB_GAUSSIAN, kE = PFB_EXPONENTIAL, kP = PFB_POLYNOMIAL;

static int kinds_of(const NllArgs& A) {
    int k = 0;
    for (int l = 0; l < A.nleaf && l < kMaxLeaves; ++l) k |= (A.leaf[l].kind & 3) << (2 * l);
    return k;
}

// EvSum2GE's fixed layout (leaf 0 gaussian, leaf 1 exponential, term t =
// leaf t alone) and |ln c_t| < 200 (see EvSum2GE).
static bool sum2ge_ok(const NllArgs& A) {
    if (A.leaf[0].voff != 0 || A.leaf[1].voff != 2) return false;
    if (A.term[0].emask != 1u || A.term[1].emask != 2u || A.term[0].vmask || A.term[1].vmask) return false;
    const int npts = A.npts > 0 ? A.npts : 1;
    for (int m = 0; m < npts; ++m)  // every parameter point's log coefficients (the ptv rows)
        for (int t = 0; t < 2; ++t)
            if (!(fabs(A.ptv[m][kPtLeafWords + 2 * t]) < 200.0)) return false;
    return true;
}

// EvGaussPoly's fixed layout: leaf 0 gaussian, leaf 1 polynomial, one term
// multiplying both (gaussian in the log sum, polynomial as a value).
static bool gp_ok(const NllArgs& A) {
    if (A.leaf[0].voff != 0 || A.leaf[1].voff != 2 || A.leaf[1].nv < 1) return false;
    if (A.term[0].emask != 1u || A.term[0].vmask != 2u) return false;
    const int npts = A.npts > 0 ? A.npts : 1;
    for (int m = 0; m < npts; ++m)  // every parameter point's log coefficient (the ptv rows)
        if (!(fabs(A.ptv[m][kPtLeafWords]) < 600.0)) return false;
    return true;
}

// EvProd1's layout: one term, exp-type leaves in its emask, polynomials in its
// vmask, at least one polynomial (without one the log-domain unit sums need
// no logarithm at all).
static bool prod1_ok(const NllArgs& A) {
    if (A.nterm != 1) return false;
    const int npts = A.npts > 0 ? A.npts : 1;
    for (int m = 0; m < npts; ++m)  // every parameter point's log coefficient (the ptv rows)
        if (!(fabs(A.ptv[m][kPtLeafWords]) < 600.0)) return false;
    bool value = false;
    for (int l = 0; l < A.nleaf; ++l) {
        const SopLeaf& L = A.leaf[l];
        const bool e = (A.term[0].emask >> l) & 1u, v = (A.term[0].vmask >> l) & 1u;
        if (L.kind == PFB_POLYNOMIAL) {
            if (!v || e || L.nv < 1) return false;
            value = true;
        } else if (!e || v) {
            return false;
        }
    }
    return value;
}

// True when launch_sop runs the TMA pipeline kernel for this plan -- the
// kernel that evaluates A.npts parameter points per pass over the data.
bool sop_batched_in_kernel(const NllArgs& A, int nc) {
    if (!A.tma) return false;
    const int nl = A.nleaf, nt = A.nterm, kinds = kinds_of(A);
    // C1 / C5 SumPdf(gaussian, exponential): product mode with per-point
    // constants and tables in the TMA unit kernel (EvSum2GE::POINTS); the
    // caller re-checks sum2ge_ok once every point is filled
    if (nc == 1 && nl == 2 && nt == 2 && kinds == (kG | kE << 2) && A.warps == 0) return sum2ge_ok(A);
    if (nc == 2 && nl == 2 && nt == 1 && kinds == (kG | kP << 2) && A.warps == 0) return gp_ok(A);  // EvGaussPoly
    // EvProd1 on one or two columns (a lone polynomial; exp-type x polynomial)
    if (nc == 1 && nl == 1 && kinds == kP && A.warps == 0) return prod1_ok(A);
    if (nc == 2 && nl == 2 && A.warps == 0 && prod1_ok(A)) return true;
    if (nc == 1) return nl == 1 && nt == 1 && kinds == kG;
    if (nc == 2) return nl == 2 && nt == 1 && kinds == (kG | kE << 2);
    return false;
}

// pipeline 1: the unit-sum TMA kernel; 2: the reference-tree TMA kernel;
// 0: the SIMT streaming kernel
template <class Ev>
static cudaError_t launch_stream(const NllArgs& A, cudaStream_t stream, int sm_count) {
    if (A.tma == 1) return launch_unit_sum<Ev>(A, stream, sm_count);
    if (A.tma) return launch_tma<Ev>(A, stream, sm_count);
    return launch_p<Ev>(A, stream, sm_count);
}

// Persistent kernels (pfb_nll_task.cuh) for the shapes the minimiser calls
// most: 1 = SumPdf(gaussian, exponential) product mode (C1 / C5), 2 =
// ProdPdf(gaussian(x), exponential(y)) unit sums (C2).  0: none (one-shot
// launches).  The kind is re-derived from every call's arguments.
int persist_kind_sop(const NllArgs& A, int nc) {
    if (!A.tma || A.warps || A.npts != 1 || A.evaluator != EV_SOP) return 0;
    const int nl = A.nleaf, nt = A.nterm, kinds = kinds_of(A);
    if (nc == 1 && nl == 2 && nt == 2 && kinds == (kG | kE << 2) && sum2ge_ok(A)) return 1;
    if (nc == 2 && nl == 2 && nt == 1 && kinds == (kG | kE << 2)) return 2;
    return 0;
}

cudaError_t launch_persist_sop(int kind, const PersistCtl& P, cudaStream_t stream, int sm_count) {
    if (kind == 1) return launch_persist<EvSum2GE<>, true>(P, stream, sm_count);
    if (kind == 2) return launch_persist<EvSop<2, 2, 1, true, kG | kE << 2>, false>(P, stream, sm_count);
    return cudaErrorInvalidValue;
}

cudaError_t launch_sop(const NllArgs& A, cudaStream_t stream, int sm_count, int nc) {
    const int nl = A.nleaf, nt = A.nterm, kinds = kinds_of(A);
    if (nc == 1) {
        // SumPdf(gaussian, exponential): C1 / C5.  FP64-bound: product mode
        // (two exp per event, one log per 16 events) on the SIMT streaming
        // kernel; the log-domain kernel (one exp + one log per event) when
        // the pipeline is off or the shape's preconditions do not hold.
        // pipeline 1: per-warp bulk prefetch below 24 blocks per SM, the TMA
        // unit kernel above (its single-point instance: 10M 27.6 vs 27.6 us,
        // 20M 42.0 vs 46.1, 40M 72.7 vs 76.8 for the warp-task kernel, 100M
        // 160.8 vs 164.8 -- measured); 2: bulk prefetch; 3: the TMA unit
        // kernel; 4: the warp-task kernel (pfb_nll_task.cuh) -- the same
        // canonical blocks, the same bits
        if (nl == 2 && nt == 2 && kinds == (kG | kE << 2) && A.tma && sum2ge_ok(A)) {
            const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
            if (A.npts > 1)  // batched points: one pass, the stage reused by every point
                return A.g2_qcert ? launch_tma_unit<EvSum2GE<true>, true>(A, stream, sm_count)
                                  : launch_tma_unit<EvSum2GE<>, true>(A, stream, sm_count);
            if (A.task_shell && A.warps == 0)
                return A.g2_qcert ? launch_task<EvSum2GE<true>>(A, stream, sm_count)
                                  : launch_task<EvSum2GE<>>(A, stream, sm_count);
            if (A.tma == 1 && A.warps == 0 && nitems >= PFB_TMA1_ITEMS_PER_SM * (int64_t)sm_count)
                return A.g2_qcert ? launch_tma_unit<EvSum2GE<true>, true>(A, stream, sm_count)
                                  : launch_tma_unit<EvSum2GE<>, true>(A, stream, sm_count);
            return A.g2_qcert ? launch_prod<EvSum2GE<true>>(A, stream, sm_count)
                              : launch_prod<EvSum2GE<>>(A, stream, sm_count);
        }
        if (nl == 2 && nt == 2 && kinds == (kG | kE << 2))
            return launch_p<EvSop<1, 2, 2, true, kG | kE << 2>>(A, stream, sm_count);
        if (nl == 1 && nt == 1 && kinds == kG)
            return launch_stream<EvSop<1, 1, 1, true, kG>>(A, stream, sm_count);
        // a lone polynomial: product mode (one log per 16 events)
        if (nl == 1 && kinds == kP && A.tma && prod1_ok(A))
            return A.npts > 1 ? launch_tma_unit<EvProd1<1, 1, kP>, true>(A, stream, sm_count)
                              : launch_prod<EvProd1<1, 1, kP>>(A, stream, sm_count);
        if (nl == 1 && nt == 1) return launch_p<EvSop<1, 1, 1, true>>(A, stream, sm_count);
        if (nl == 2 && nt == 2) return launch_p<EvSop<1, 2, 2, true>>(A, stream, sm_count);
        return launch_p<EvSop<1>>(A, stream, sm_count);
    }
    if (nc == 2) {
        // ProdPdf(gaussian(x), exponential(y)): C2
        if (nl == 2 && nt == 1 && kinds == (kG | kE << 2))
            return launch_stream<EvSop<2, 2, 1, true, kG | kE << 2>>(A, stream, sm_count);
        // ProdPdf(gaussian(x), polynomial(y)): C2p -- product mode (one log
        // per 16 events) with the pipeline on; the log-domain EvSop (108 us at
        // 10M, XU-bound) without; the generic SIMT instantiation took 290 us
        if (nl == 2 && nt == 1 && kinds == (kG | kP << 2) && A.tma && gp_ok(A)) {
            switch (A.leaf[1].nv) {
                case 1: return launch_prod<EvGaussPoly<1>>(A, stream, sm_count);
                case 2: return launch_prod<EvGaussPoly<2>>(A, stream, sm_count);
                case 3: return launch_prod<EvGaussPoly<3>>(A, stream, sm_count);
                case 4: return launch_prod<EvGaussPoly<4>>(A, stream, sm_count);
                default: return launch_prod<EvGaussPoly<>>(A, stream, sm_count);
            }
        }
        if (nl == 2 && nt == 1 && kinds == (kG | kP << 2))
            return launch_stream<EvSop<2, 2, 1, true, kG | kP << 2>>(A, stream, sm_count);
        // other single-term products with a polynomial factor: product mode
        if (nl == 2 && A.tma && prod1_ok(A)) return launch_prod<EvProd1<2, 2, -1>>(A, stream, sm_count);
        return launch_p<EvSop<2>>(A, stream, sm_count);
    }
    // the kernels stream exactly the plan's columns (NC of them)
    if (nc == 3 && nl == 3 && A.tma && prod1_ok(A)) return launch_prod<EvProd1<3, 3, -1>>(A, stream, sm_count);
    if (nc == 3) return launch_p<EvSop<3>>(A, stream, sm_count);
    return launch_p<EvSop<4>>(A, stream, sm_count);
}

}  // namespace pfb

#ifdef PFB_TRACE
extern "C" int pfb_debug_trace(unsigned long long* out, int nblocks) {
    return (int)pfb::read_trace(out, nblocks);
}
#endif
