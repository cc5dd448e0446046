// pfb_nll_dal.cu -- Dalitz instantiations: recompute path with K known at
// compile time (batch-inverted denominators), optionally with the term
// structure (pair, spin per term) fixed at compile time; the generic /
// lineshape-cache path for everything else.
#include "pfb_nll_prod.cuh"
#include "pfb_nll_task.cuh"

namespace pfb {

// (pair, spin) signature, 3 bits per term (see EvDalitz)
static constexpr int sig_term(int pair, int spin) { return dal_pair_code(pair) | (spin << 2); }
// C3 / C4: D0 -> pi+ pi- pi0 with rho+ (13, P-wave), rho- (23), rho0 (12), NR (12, S-wave)
// pi+ pi- equal masses: the 12 Zemach term has no 1/s12 part (need 13, 23 only)
static constexpr int kSigD0 = sig_term(13, 1) | sig_term(23, 1) << 3 | sig_term(12, 1) << 6 |
                              sig_term(12, 0) << 9 | 1 << 13 | 1 << 14;

static int signature_of(const DalDesc& D) {
    int sig = 0;
    for (int k = 0; k < D.K; ++k) sig |= sig_term(D.t[k].pair, D.t[k].spin) << (3 * k);
    return sig | (D.need12 ? 1 << 12 : 0) | (D.need13 ? 1 << 13 : 0) | (D.need23 ? 1 << 14 : 0);
}

// Batched parameter points in one pass (pfb_nll_batch): the D0 ratio form,
// pipeline 1, the coefficients of every point in the ptv rows.
bool dal_batched_in_kernel(const NllArgs& A) {
    return A.tma == 1 && A.warps == 0 && A.evaluator == EV_DALITZ && A.dal.K == 4 && signature_of(A.dal) == kSigD0;
}

cudaError_t launch_dalitz(const NllArgs& A, cudaStream_t stream, int sm_count) {
    if (A.evaluator == EV_DALITZ_CACHED) return launch_p<EvDalitzCached>(A, stream, sm_count);
    const bool d0 = A.dal.K == 4 && signature_of(A.dal) == kSigD0;
    if (A.npts > 1 && dal_batched_in_kernel(A))
        return launch_tma_unit<EvDalitzR<4, kSigD0, true>, true>(A, stream, sm_count);
    if (A.tma) {
        // product kernels.  D0 -> pi+ pi- pi0 (C3/C4): the reciprocal-free
        // ratio form with the term structure fixed at compile time.  Other
        // models with 2..4 terms: the batch-inverted form (the ratio form with
        // the structure read at run time measured 14-40% slower there);
        // 5..6 terms: the run-time ratio form (1.9x faster than the per-term
        // reciprocal kernel they used before, K = 5 measured)
        if (d0) return launch_prod<EvDalitzR<4, kSigD0>>(A, stream, sm_count);
        switch (A.dal.K) {
            case 2: return launch_prod<EvDalitz<2>>(A, stream, sm_count);
            case 3: return launch_prod<EvDalitz<3>>(A, stream, sm_count);
            case 4: return launch_prod<EvDalitz<4>>(A, stream, sm_count);
            case 5: return launch_prod<EvDalitzR<5>>(A, stream, sm_count);
            case 6: return launch_prod<EvDalitzR<6>>(A, stream, sm_count);
            default: break;
        }
    }
    // pipeline 0 (log-domain SIMT kernels) and K > 6
    switch (A.dal.K) {
        case 2:
            return launch_p<EvDalitz<2>>(A, stream, sm_count);
        case 3:
            return launch_p<EvDalitz<3>>(A, stream, sm_count);
        case 4:
            if (d0) return launch_p<EvDalitz<4, kSigD0>>(A, stream, sm_count);
            return launch_p<EvDalitz<4>>(A, stream, sm_count);
        default:  // any K: per-term reciprocals, no cache rows
            return launch_p<EvDalitzCached>(A, stream, sm_count);
    }
}

// Persistent kernel for the D0 -> pi+ pi- pi0 ratio form (C3 / C4): kind 3.
int persist_kind_dal(const NllArgs& A) {
    if (!A.tma || A.warps || A.npts != 1 || A.evaluator != EV_DALITZ) return 0;
    return A.dal.K == 4 && signature_of(A.dal) == kSigD0 ? 3 : 0;
}

cudaError_t launch_persist_dal(int kind, const PersistCtl& P, cudaStream_t stream, int sm_count) {
    if (kind == 3) return launch_persist<EvDalitzR<4, kSigD0>, true>(P, stream, sm_count);
    return cudaErrorInvalidValue;
}

}  // namespace pfb

#ifdef PFB_TRACE
extern "C" int pfb_debug_trace_dal(unsigned long long* out, int nblocks) {
    return (int)pfb::read_trace(out, nblocks);
}
#endif
