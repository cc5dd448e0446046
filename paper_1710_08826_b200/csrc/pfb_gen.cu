// pfb_gen.cu -- device synthetic-event generation (toy Monte Carlo).
//
// The reference samples with numpy PCG64 accept-reject (mcgen.py:68-257);
// generating 100M Dalitz events that way takes minutes on the host.  Here
// candidates are drawn with a counter-based Philox4x32-10 stream (candidate
// c uses counter c, so any thread can draw any candidate), accepted with the
// same rule as the reference (flat in the (s12, s13) box, kinematic boundary,
// u * envelope < intensity) and compacted IN CANDIDATE ORDER (per-CTA counts,
// one exclusive scan, a second pass that rewrites the survivors), so the
// output is deterministic for a given seed.  Streams are not bit-identical
// to numpy's PCG64 (documented in DESIGN.md); parity never depends on them
// because the device and the CPU reference consume the same arrays.
#include "pfb_internal.cuh"
#include "pfb_math.cuh"

namespace pfb {

struct Philox {
    uint32_t c0, c1, c2, c3;
};

__device__ __forceinline__ Philox philox4x32_10(uint32_t k0, uint32_t k1, uint32_t c0, uint32_t c1,
                                                uint32_t c2, uint32_t c3) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u, W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
        const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
        k0 += W0;
        k1 += W1;
    }
    return {c0, c1, c2, c3};
}

// Uniform double in [0, 1) with 53 random bits (as numpy: (u64 >> 11) * 2^-53).
__device__ __forceinline__ double u53(uint32_t hi, uint32_t lo) {
    const unsigned long long v = (((unsigned long long)hi << 32) | lo) >> 11;
    return (double)v * (1.0 / 9007199254740992.0);
}

// candidate -> accepted?  (s12, s13) written when accepted
__device__ __forceinline__ bool dalitz_candidate(const GenDalitz& G, unsigned long long c, double* o12,
                                                 double* o13) {
    const Philox a = philox4x32_10(G.seed_lo, G.seed_hi, (uint32_t)c, (uint32_t)(c >> 32), 0u, 0x6a09e667u);
    const Philox b = philox4x32_10(G.seed_lo, G.seed_hi, (uint32_t)c, (uint32_t)(c >> 32), 1u, 0x6a09e667u);
    const double s12 = G.lo12 + (G.hi12 - G.lo12) * u53(a.c0, a.c1);
    const double s13 = G.lo13 + (G.hi13 - G.lo13) * u53(a.c2, a.c3);
    const double u = G.envelope * u53(b.c0, b.c1);
    // kinematic boundary (dalitz.py:127-150)
    const double rs = sqrt(s12);
    const double e1 = (s12 + G.m1sq - G.m2sq) / (2.0 * rs);
    const double e3 = (G.M2 - s12 - G.m3sq) / (2.0 * rs);
    const double p1 = sqrt(e1 * e1 - G.m1sq), p3 = sqrt(e3 * e3 - G.m3sq);
    const double es = (e1 + e3) * (e1 + e3);
    const bool inside = (s13 >= es - (p1 + p3) * (p1 + p3)) && (s13 <= es - (p1 - p3) * (p1 - p3));
    if (!inside) return false;
    double tr = 0.0, ti = 0.0;
    for (int k = 0; k < G.D.K; ++k) {
        const DalTerm& T = G.D.t[k];
        const double2 amp = dalitz_amp_literal(G.D, T, s12, s13);
        tr += T.cre * amp.x - T.cim * amp.y;
        ti += T.cre * amp.y + T.cim * amp.x;
    }
    const double I = tr * tr + ti * ti;
    if (!(u < I)) return false;
    *o12 = s12;
    *o13 = s13;
    return true;
}

__device__ __forceinline__ double trunc_gauss(const Gen1D& G, unsigned long long i, uint32_t stream) {
    for (uint32_t t = 0;; ++t) {
        const Philox r = philox4x32_10(G.seed_lo, G.seed_hi, (uint32_t)i, (uint32_t)(i >> 32), stream, t);
        const double u1 = 1.0 - u53(r.c0, r.c1), u2 = u53(r.c2, r.c3);  // u1 in (0,1]
        const double rad = sqrt(-2.0 * log(u1));
        double s, cth;
        sincospi(2.0 * u2, &s, &cth);
        const double x0 = G.mu + G.sigma * rad * cth, x1 = G.mu + G.sigma * rad * s;
        if (x0 >= G.lo && x0 <= G.hi) return x0;
        if (x1 >= G.lo && x1 <= G.hi) return x1;
    }
}

__device__ __forceinline__ double trunc_exp(const Gen1D& G, unsigned long long i, uint32_t stream) {
    const Philox r = philox4x32_10(G.seed_lo, G.seed_hi, (uint32_t)i, (uint32_t)(i >> 32), stream, 0x5bd1e995u);
    const double u = u53(r.c0, r.c1);
    if (G.alpha == 0.0) return G.lo + (G.hi - G.lo) * u;
    const double a = exp(G.alpha * G.lo), b = exp(G.alpha * G.hi);
    const double x = log(a + u * (b - a)) / G.alpha;
    return fmin(fmax(x, G.lo), G.hi);
}

__global__ void gen_1d_kernel(Gen1D G, int64_t n, double* x, double* y) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        if (G.kind == 0) {
            const Philox r = philox4x32_10(G.seed_lo, G.seed_hi, (uint32_t)i, (uint32_t)(i >> 32), 7u, 0u);
            x[i] = (u53(r.c0, r.c1) < G.f) ? trunc_gauss(G, i, 1u) : trunc_exp(G, i, 2u);
        } else {
            x[i] = trunc_gauss(G, i, 3u);
            y[i] = trunc_exp(G, i, 4u);
        }
    }
}

constexpr int kGenThreads = 256;
constexpr int kGenPerThread = 8;
constexpr int64_t kGenPerCta = (int64_t)kGenThreads * kGenPerThread;

// pass 1: accepted count per CTA for candidates [base, base + grid*kGenPerCta)
__global__ void gen_dalitz_count(GenDalitz G, unsigned long long base, int* counts) {
    __shared__ int s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    int mine = 0;
    const unsigned long long c0 = base + (unsigned long long)blockIdx.x * kGenPerCta;
    for (int j = 0; j < kGenPerThread; ++j) {
        double a, b;
        mine += dalitz_candidate(G, c0 + (unsigned long long)j * kGenThreads + threadIdx.x, &a, &b) ? 1 : 0;
    }
    atomicAdd(&s, mine);
    __syncthreads();
    if (threadIdx.x == 0) counts[blockIdx.x] = s;
}

// exclusive scan of the per-CTA counts (one CTA); offsets[nblk] = total
__global__ void gen_scan(const int* counts, int nblk, long long* offsets) {
    __shared__ long long part[1024];
    const int per = (nblk + blockDim.x - 1) / blockDim.x;
    long long sum = 0;
    for (int i = 0; i < per; ++i) {
        const int j = threadIdx.x * per + i;
        if (j < nblk) sum += counts[j];
    }
    part[threadIdx.x] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long run = 0;
        for (int t = 0; t < (int)blockDim.x; ++t) {
            const long long v = part[t];
            part[t] = run;
            run += v;
        }
        offsets[nblk] = run;
    }
    __syncthreads();
    long long run = part[threadIdx.x];
    for (int i = 0; i < per; ++i) {
        const int j = threadIdx.x * per + i;
        if (j < nblk) {
            offsets[j] = run;
            run += counts[j];
        }
    }
}

// pass 2: rewrite the survivors in candidate order at out_base + offset
__global__ void gen_dalitz_write(GenDalitz G, unsigned long long base, const long long* offsets,
                                 long long out_base, long long n_want, double* s12, double* s13) {
    __shared__ int warp_tot[kGenThreads / 32];
    __shared__ long long run;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (threadIdx.x == 0) run = offsets[blockIdx.x];
    __syncthreads();
    const unsigned long long c0 = base + (unsigned long long)blockIdx.x * kGenPerCta;
    for (int j = 0; j < kGenPerThread; ++j) {
        double a = 0.0, b = 0.0;
        const bool acc = dalitz_candidate(G, c0 + (unsigned long long)j * kGenThreads + threadIdx.x, &a, &b);
        const unsigned bal = __ballot_sync(0xffffffffu, acc);
        if (lane == 0) warp_tot[wid] = __popc(bal);
        __syncthreads();
        long long pre = run;
        for (int w = 0; w < wid; ++w) pre += warp_tot[w];
        pre += __popc(bal & ((1u << lane) - 1u));
        const long long dst = out_base + pre;
        if (acc && dst < n_want) {
            s12[dst] = a;
            s13[dst] = b;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            long long tot = 0;
            for (int w = 0; w < kGenThreads / 32; ++w) tot += warp_tot[w];
            run += tot;
        }
        __syncthreads();
    }
}

cudaError_t launch_gen_1d(const Gen1D& G, int64_t n, double* x, double* y, cudaStream_t st, int sm) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > (int64_t)sm * 16) blocks = (int64_t)sm * 16;
    if (blocks < 1) blocks = 1;
    gen_1d_kernel<<<(unsigned)blocks, 256, 0, st>>>(G, n, x, y);
    return cudaGetLastError();
}

// Host driver: rounds of candidates until n events are accepted.
cudaError_t run_gen_dalitz(const GenDalitz& G, int64_t n, double* s12, double* s13, cudaStream_t st,
                           int sm, int64_t* candidates_used) {
    const int nblk = sm * 64;
    int* counts = nullptr;
    long long* offsets = nullptr;
    cudaError_t e = cudaMalloc(&counts, sizeof(int) * nblk);
    if (e != cudaSuccess) return e;
    e = cudaMalloc(&offsets, sizeof(long long) * (nblk + 1));
    if (e != cudaSuccess) {
        cudaFree(counts);
        return e;
    }
    long long got = 0;
    unsigned long long base = 0;
    while (got < n) {
        gen_dalitz_count<<<nblk, kGenThreads, 0, st>>>(G, base, counts);
        gen_scan<<<1, 1024, 0, st>>>(counts, nblk, offsets);
        gen_dalitz_write<<<nblk, kGenThreads, 0, st>>>(G, base, offsets, got, n, s12, s13);
        long long tot = 0;
        e = cudaMemcpyAsync(&tot, offsets + nblk, sizeof(long long), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        got += tot;
        base += (unsigned long long)nblk * kGenPerCta;
        if (tot == 0 && base > (1ull << 40)) {
            e = cudaErrorInvalidValue;  // envelope / model cannot accept anything
            break;
        }
    }
    if (candidates_used) *candidates_used = (int64_t)base;
    cudaFree(counts);
    cudaFree(offsets);
    return e == cudaSuccess ? cudaGetLastError() : e;
}

}  // namespace pfb
