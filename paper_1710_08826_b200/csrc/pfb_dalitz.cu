// pfb_dalitz.cu -- Dalitz normalisation grid, overlap integrals, lineshape cache.
//
// integration_grid (dalitz.py:246-264): midpoint centres lo + (i+0.5)*dx and
// the kinematic mask (dalitz.py:127-150) computed with the reference's exact
// IEEE operation sequence -> the mask is bit-exact.  In-boundary nodes are
// compacted in row-major order (s12 outer) exactly as g12[mask].
//
// compute_integrals (dalitz.py:282-329): amplitude rows for stale terms only,
// then I[i][j] = sum_nodes A_i conj(A_j) for every pair touching a stale term.
// Sums go through the exact integer accumulator (the correctly rounded sum of
// the per-node products); the host multiplies by the cell area, as the
// reference does after its own sum.
#include "pfb_internal.cuh"
#include "pfb_math.cuh"

namespace pfb {

__device__ __forceinline__ double centre(double lo, int i, double d) {
    return Add(lo, Mul((double)i + 0.5, d));
}

__global__ void grid_mask_kernel(GridConsts g, uint8_t* mask, int* row_count) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (int64_t)g.nx * g.ny) return;
    const int i = (int)(idx / g.ny), j = (int)(idx % g.ny);
    const bool in = in_boundary_exact(g, centre(g.lo12, i, g.dx), centre(g.lo13, j, g.dy));
    mask[idx] = in ? 1 : 0;
    if (in) atomicAdd(&row_count[i], 1);
}

// One warp per row: ordered compaction with ballots.
__global__ void grid_compact_kernel(GridConsts g, const uint8_t* mask, const int* row_offset,
                                    double* p12, double* p13) {
    const int row = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const int lane = threadIdx.x & 31;
    if (row >= g.nx) return;
    int out = row_offset[row];
    const double s12 = centre(g.lo12, row, g.dx);
    for (int j0 = 0; j0 < g.ny; j0 += 32) {
        const int j = j0 + lane;
        const bool in = j < g.ny && mask[(int64_t)row * g.ny + j];
        const unsigned bal = __ballot_sync(0xffffffffu, in);
        if (in) {
            const int pos = out + __popc(bal & ((1u << lane) - 1u));
            p12[pos] = s12;
            p13[pos] = centre(g.lo13, j, g.dy);
        }
        out += __popc(bal);
    }
}

// Amplitude row of one term over the compacted nodes (literal arithmetic).
__global__ void grid_amp_kernel(DalDesc D, DalTerm T, const double* p12, const double* p13,
                                int64_t n, double2* out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = dalitz_amp_literal(D, T, p12[i], p13[i]);
}

// Overlap sums.  blockIdx.y = pair index; each pair has two accumulators
// (real, imaginary) of PFB_ACC_WORDS words in `acc`.
__global__ void grid_overlap_kernel(const double2* amps, int64_t n, const int2* pairs,
                                    unsigned long long* acc) {
    __shared__ long long s[2][PFB_ACC_WORDS];
    for (int i = threadIdx.x; i < 2 * PFB_ACC_WORDS; i += blockDim.x) (&s[0][0])[i] = 0;
    __syncthreads();
    const int2 pr = pairs[blockIdx.y];
    const double2* Ai = amps + (int64_t)pr.x * n;
    const double2* Aj = amps + (int64_t)pr.y * n;
    // warp-uniform trip count: the accumulator adds are warp-aggregated
    // (acc_add_warp; per-thread 64-bit shared atomics on the same few limbs
    // serialised this kernel: 233 us for one 4-term overlap matrix, ncu)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k0 = (int64_t)blockIdx.x * blockDim.x; k0 < n; k0 += stride) {
        const int64_t k = k0 + threadIdx.x;
        const bool act = k < n;
        double re = 0.0, im = 0.0;
        if (act) {
            const double2 a = Ai[k], b = Aj[k];
            if (pr.x == pr.y) {
                re = Add(Mul(a.x, a.x), Mul(a.y, a.y));
            } else {
                const double bni = Sub(0.0, b.y);  // conj(b)
                re = Sub(Mul(a.x, b.x), Mul(a.y, bni));
                im = Add(Mul(a.x, bni), Mul(a.y, b.x));
            }
        }
        acc_add_warp(s[0], re, act);
        if (pr.x != pr.y) acc_add_warp(s[1], im, act);  // block-uniform branch
    }
    __syncthreads();
    unsigned long long* dst = acc + (int64_t)blockIdx.y * 2 * PFB_ACC_WORDS;
    for (int i = threadIdx.x; i < 2 * PFB_ACC_WORDS; i += blockDim.x) {
        const long long v = (&s[0][0])[i];
        if (v) atomicAdd(dst + i, (unsigned long long)v);
    }
}

// Per-event lineshape cache row: A_k(event) with the literal arithmetic, so
// cached amplitudes are the reference's amplitudes.
__global__ void lineshape_cache_kernel(DalDesc D, DalTerm T, const double* s12, const double* s13,
                                       int64_t n, double2* row) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        row[i] = dalitz_amp_literal(D, T, __ldg(s12 + i), __ldg(s13 + i));
}

cudaError_t launch_grid_mask(const GridConsts& g, uint8_t* mask, int* row_count,
                             cudaStream_t st) {
    const int64_t total = (int64_t)g.nx * g.ny;
    grid_mask_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(g, mask, row_count);
    return cudaGetLastError();
}

cudaError_t launch_grid_compact(const GridConsts& g, const uint8_t* mask, const int* row_offset,
                                double* p12, double* p13, cudaStream_t st) {
    const int warps = 8;
    grid_compact_kernel<<<(g.nx + warps - 1) / warps, warps * 32, 0, st>>>(g, mask, row_offset,
                                                                          p12, p13);
    return cudaGetLastError();
}

cudaError_t launch_grid_amp(const DalDesc& D, const DalTerm& T, const double* p12,
                            const double* p13, int64_t n, double2* out, cudaStream_t st,
                            int sm_count) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sm_count * 8) blocks = (int64_t)sm_count * 8;
    if (blocks < 1) blocks = 1;
    grid_amp_kernel<<<(unsigned)blocks, 256, 0, st>>>(D, T, p12, p13, n, out);
    return cudaGetLastError();
}

cudaError_t launch_grid_overlap(const double2* amps, int64_t n, const int2* pairs, int npairs,
                                unsigned long long* acc, cudaStream_t st, int sm_count) {
    int64_t bx = (n + 255 * 8) / (256 * 8);
    if (bx < 1) bx = 1;
    const int64_t cap = ((int64_t)sm_count * 8 + npairs - 1) / npairs;
    if (bx > cap) bx = cap > 0 ? cap : 1;
    dim3 grid((unsigned)bx, (unsigned)npairs);
    grid_overlap_kernel<<<grid, 256, 0, st>>>(amps, n, pairs, acc);
    return cudaGetLastError();
}

cudaError_t launch_lineshape_cache(const DalDesc& D, const DalTerm& T, const double* s12,
                                   const double* s13, int64_t n, double2* row, cudaStream_t st,
                                   int sm_count) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sm_count * 16) blocks = (int64_t)sm_count * 16;
    if (blocks < 1) blocks = 1;
    lineshape_cache_kernel<<<(unsigned)blocks, 256, 0, st>>>(D, T, s12, s13, n, row);
    return cudaGetLastError();
}

}  // namespace pfb
