// pfb_nll_dal.cu -- Dalitz instantiations: recompute path with K known at
// compile time (batch-inverted denominators), generic/lineshape-cache path.
#include "pfb_nll_kernel.cuh"

namespace pfb {

cudaError_t launch_dalitz(const NllArgs& A, cudaStream_t stream, int sm_count) {
    if (A.evaluator == EV_DALITZ_CACHED) return launch_p<EvDalitzCached>(A, stream, sm_count);
    switch (A.dal.K) {
        case 2:
            return launch_p<EvDalitz<2>>(A, stream, sm_count);
        case 3:
            return launch_p<EvDalitz<3>>(A, stream, sm_count);
        case 4:
            return launch_p<EvDalitz<4>>(A, stream, sm_count);
        default:  // any K: per-term reciprocals, no cache rows
            return launch_p<EvDalitzCached>(A, stream, sm_count);
    }
}

}  // namespace pfb
