// pfb_binned.cu -- binned data on the device.
//
//   * bin_fill_kernel: BinnedDataSet.fill (core.py:370-379) -- per event the
//     row-major flat bin of clip(int64(floor((x - lower) / width)), 0, nb-1)
//     over the axes, counted with integer atomics (bit-exact; the count of a
//     bin does not depend on the order of the reference's np.add.at).
//   * binned_nll_kernel: binned_nll (engine.py:246-276) -- per bin the density
//     at the bin centre through the literal interpreter (reference operation
//     order), nu = (total * p) * volume, term = nu - n ln nu for observed bins
//     (nu alone otherwise), summed through the exact integer accumulator
//     (= math.fsum of the terms).  Node-kernel errors are keyed like the
//     unbinned path; a non-positive expectation in an observed bin is keyed
//     by its bin index (NonPositiveExpectation, errors.py:102-108).
#include <climits>

#include "pfb_nll_kernel.cuh"

namespace pfb {

// numpy's float64 -> int64 cast (astype) on x86-64 (cvttsd2si): NaN, +-inf and
// values outside [-2^63, 2^63) become INT64_MIN ("integer indefinite").
__device__ __forceinline__ long long np_floor_to_i64(double v) {
    const double f = floor(v);
    if (!(f >= -9223372036854775808.0 && f < 9223372036854775808.0)) return LLONG_MIN;
    return (long long)f;
}

__global__ void bin_fill_kernel(const BinAxes B, int64_t begin, int64_t n, unsigned long long* counts) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x) {
        long long idx = 0;
        for (int a = 0; a < B.naxes; ++a) {
            const double x = B.col[a][begin + j];
            long long k = np_floor_to_i64(__ddiv_rn(__dsub_rn(x, B.lower[a]), B.width[a]));
            k = k < 0 ? 0 : (k > B.nbins[a] - 1 ? B.nbins[a] - 1 : k);
            idx = idx * B.nbins[a] + k;
        }
        atomicAdd(counts + idx, 1ull);
    }
}

__global__ void __launch_bounds__(kThreads) binned_nll_kernel(const __grid_constant__ NllArgs A,
                                                               const double* contents, int64_t nbins,
                                                               double total, double volume,
                                                               unsigned long long* expkey) {
    __shared__ long long sacc[PFB_ACC_WORDS];
    __shared__ unsigned int s_last;
    for (int i = threadIdx.x; i < PFB_ACC_WORDS; i += blockDim.x) sacc[i] = 0;
    __syncthreads();
    // warp-uniform trip count (acc_add_warp needs the whole warp)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t b0 = blockIdx.x * (int64_t)blockDim.x; b0 < nbins; b0 += stride) {
        const int64_t b = b0 + threadIdx.x;
        bool act = b < nbins;
        double term = 0.0;
        if (act) {
            int rank = -1;
            double val = 0.0;
            const double p = literal_density(A, A.begin + b, &rank, &val);
            if (rank >= 0) {
                record_failure(A, rank, b, sacc);
                act = false;
            } else {
                const double nu = Mul(Mul(total, p), volume);
                const double c = contents[b];
                const bool observed = c > 0.0;
                if (observed && !(nu > 0.0)) {
                    atomicMin(expkey, (unsigned long long)b);
                    act = false;
                } else {
                    term = observed ? Sub(nu, Mul(c, log(nu))) : nu;
                }
            }
        }
        acc_add_warp(sacc, term, act);
    }
    finish_launch<false>(A, sacc, &s_last);
}

// Normalisation integral by quadrature (north_star item 4): sum_j w_j * f(x_j)
// over the abscissas of a store (one column per observable), f = the plan's
// literal density with the root norm set to 1 (pdf._polynomial_norm,
// pdf.py:192-199, or any subtree over a tensor grid).  Each product is
// rounded once and the sum is exact (accumulator), i.e. the correctly
// rounded dot product.  Node-kernel errors are keyed by abscissa index as the
// reference's kernel on the abscissa array reports them.
__global__ void __launch_bounds__(kThreads) quadrature_kernel(const __grid_constant__ NllArgs A,
                                                               const double* weights, int64_t n) {
    __shared__ long long sacc[PFB_ACC_WORDS];
    __shared__ unsigned int s_last;
    for (int i = threadIdx.x; i < PFB_ACC_WORDS; i += blockDim.x) sacc[i] = 0;
    __syncthreads();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j0 = blockIdx.x * (int64_t)blockDim.x; j0 < n; j0 += stride) {
        const int64_t j = j0 + threadIdx.x;
        bool act = j < n;
        double term = 0.0;
        if (act) {
            int rank = -1;
            double val = 0.0;
            const double f = literal_density(A, A.begin + j, &rank, &val);
            if (rank >= 0) {
                record_failure(A, rank, j, sacc);
                act = false;
            } else {
                term = Mul(weights[j], f);
            }
        }
        acc_add_warp(sacc, term, act);
    }
    finish_launch<false>(A, sacc, &s_last);
}

// nu of one bin (the NonPositiveExpectation value).
__global__ void binned_probe_kernel(const __grid_constant__ NllArgs A, int64_t b, double total, double volume,
                                    double* out) {
    int rank = -1;
    double val = 0.0;
    const double p = literal_density(A, A.begin + b, &rank, &val);
    out[0] = Mul(Mul(total, p), volume);
}

cudaError_t launch_bin_fill(const BinAxes& B, int64_t begin, int64_t n, unsigned long long* counts,
                            cudaStream_t stream, int sm_count) {
    if (n <= 0) return cudaSuccess;
    int64_t grid = (n + 255) / 256;
    if (grid > (int64_t)sm_count * 8) grid = (int64_t)sm_count * 8;
    bin_fill_kernel<<<(unsigned)grid, 256, 0, stream>>>(B, begin, n, counts);
    return cudaGetLastError();
}

cudaError_t launch_binned_nll(const NllArgs& A, const double* contents, int64_t nbins, double total,
                              double volume, unsigned long long* expkey, cudaStream_t stream, int sm_count) {
    int64_t grid = (nbins + kThreads - 1) / kThreads;
    if (grid > (int64_t)sm_count * 2) grid = (int64_t)sm_count * 2;
    if (grid < 1) grid = 1;
    binned_nll_kernel<<<(unsigned)grid, kThreads, 0, stream>>>(A, contents, nbins, total, volume, expkey);
    return cudaGetLastError();
}

cudaError_t launch_quadrature(const NllArgs& A, const double* weights, int64_t n, cudaStream_t stream,
                              int sm_count) {
    int64_t grid = (n + kThreads - 1) / kThreads;
    if (grid > (int64_t)sm_count * 2) grid = (int64_t)sm_count * 2;
    if (grid < 1) grid = 1;
    quadrature_kernel<<<(unsigned)grid, kThreads, 0, stream>>>(A, weights, n);
    return cudaGetLastError();
}

cudaError_t launch_binned_probe(const NllArgs& A, int64_t b, double total, double volume, double* out,
                                cudaStream_t stream) {
    binned_probe_kernel<<<1, 1, 0, stream>>>(A, b, total, volume, out);
    return cudaGetLastError();
}

}  // namespace pfb
