// pfb_nll_sop.cu -- sum-of-products (log-domain) instantiations: 1, 2 or 4
// observable columns x P in {1,2,4,8}.
#include "pfb_nll_kernel.cuh"

namespace pfb {

cudaError_t launch_sop(const NllArgs& A, cudaStream_t stream, int sm_count, int nc) {
    switch (nc) {
        case 1:
            return launch_p<EvSop<1>>(A, stream, sm_count);
        case 2:
            return launch_p<EvSop<2>>(A, stream, sm_count);
        default:
            return launch_p<EvSop<4>>(A, stream, sm_count);
    }
}

}  // namespace pfb
