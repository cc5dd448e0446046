// pfb_pcg.cu -- the reference's toy generator on the GPU, stream for stream
// (mcgen.py:56-97, 155-257).
//
// numpy's PCG64 (XSL-RR 128/64: state <- state * M + inc mod 2^128, output
// rotr64(hi ^ lo, hi >> 58) of the new state) and Generator.uniform(lo, hi)
// = lo + (hi - lo) * ((next >> 11) * 2^-53) are reproduced bit for bit.  The
// accept-reject loop of the reference draws chunks of k <= 8192 candidates:
//   1-D:    x = uniform(lo, hi, k), u = uniform(0, envelope, k)      (2k draws)
//   Dalitz: s12, s13 = uniform over the box (k each), u (k)           (3k draws)
// and keeps candidates with u < density (Dalitz: inside the kinematic
// boundary first).  Here every chunk's draw offsets are known in advance, so a
// whole batch of chunks is generated in parallel from jumped-ahead states:
//   count kernel  -- per chunk: accepted count, max density (envelope check),
//                    in-boundary count;
//   host          -- walks the chunks in order exactly like the reference loop
//                    (envelope hit, budget, how many to take from each chunk);
//   write kernel  -- one CTA per needed chunk regenerates its candidates and
//                    writes the accepted ones in candidate order.
// Densities come from the literal interpreter / literal Dalitz intensity
// (reference operation order), so an accept decision can differ from numpy's
// only when u falls within a few ulps of the density (probability ~2^-50 per
// candidate); the in-boundary mask is bit-exact.  Such candidates are
// counted (|u - density| <= 2^-47 density, and chunks whose maximum density
// lies that close to the envelope) and reported as pfb_gen_stats.ambiguous:
// a run with ambiguous == 0 is the reference's sample bit for bit (given
// device densities within 2^-47 relative of numpy's).
#include <cstring>
#include <vector>

#include "pfb_nll_kernel.cuh"

namespace pfb {

typedef unsigned __int128 u128;

static constexpr uint64_t kPcgMultHi = 0x2360ED051FC65DA4ull;
static constexpr uint64_t kPcgMultLo = 0x4385DF649FCCF645ull;
static constexpr int kChunk = 8192;      // mcgen.py:31 CHUNK
static constexpr int kRun = 32;          // consecutive candidates per thread
static constexpr int kGenThreads = kChunk / kRun;

__host__ __device__ __forceinline__ u128 pcg_mult() { return ((u128)kPcgMultHi << 64) | kPcgMultLo; }

// s -> A s + C (mod 2^128) for 2^b steps, b = 0..13 (within-chunk offsets)
struct PcgJump {
    u128 a[14], c[14];
};

struct PcgChunk {
    u128 base[3];  // stream state before the chunk's first draw of each run
    int32_t k;     // candidates in the chunk
};

struct PcgParams {
    int32_t dalitz;
    int32_t nch;
    double lo0, scale0, lo1, scale1;  // candidate boxes (scale = hi - lo)
    double envelope;
    u128 inc;
    PcgJump jump;
    GridConsts g;  // Dalitz boundary
    const PcgChunk* chunks;
    unsigned long long* count;   // [nch] accepted
    unsigned long long* dmax;    // [nch] max density (bits of a non-negative double)
    unsigned long long* inside;  // [nch] in-boundary candidates (Dalitz)
    unsigned long long* ambig;   // [nch] candidates with u within 2^-47 of the density
    unsigned long long* errflag; // density kernel error (1-D)
    // write phase
    const int64_t* pos;   // [nch] output offset of the chunk's first taken event
    const int64_t* take;  // [nch] events taken from the chunk
    double* out0;
    double* out1;
};

__device__ __forceinline__ u128 pcg_step(u128 s, u128 inc) { return s * pcg_mult() + inc; }

__device__ __forceinline__ uint64_t pcg_out(u128 s) {
    const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    const uint64_t x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
}

// next_double (numpy: (next_uint64 >> 11) * 2^-53)
__device__ __forceinline__ double u53(uint64_t v) { return (double)(v >> 11) * (1.0 / 9007199254740992.0); }

// advance a state by `d` steps (d < 2^14) with the jump table
__device__ __forceinline__ u128 pcg_advance(const PcgJump& J, u128 s, int d) {
#pragma unroll
    for (int b = 0; b < 14; ++b)
        if ((d >> b) & 1) s = J.a[b] * s + J.c[b];
    return s;
}

// One run of kRun candidates of chunk `ch` starting at candidate i0: calls
// f(i, x0, x1, u) for every candidate i < k in order.
template <class F>
__device__ __forceinline__ void pcg_run(const PcgParams& P, const PcgChunk& ch, int i0, F&& f) {
    const int nd = P.dalitz ? 3 : 2;
    u128 s0 = pcg_advance(P.jump, ch.base[0], i0);
    u128 s1 = pcg_advance(P.jump, ch.base[1], i0);
    u128 s2 = nd == 3 ? pcg_advance(P.jump, ch.base[2], i0) : (u128)0;
    const int n = ch.k - i0 < kRun ? ch.k - i0 : kRun;
    for (int t = 0; t < n; ++t) {
        s0 = pcg_step(s0, P.inc);
        s1 = pcg_step(s1, P.inc);
        double x0, x1 = 0.0, u;
        x0 = Add(P.lo0, Mul(P.scale0, u53(pcg_out(s0))));
        if (nd == 3) {
            s2 = pcg_step(s2, P.inc);
            x1 = Add(P.lo1, Mul(P.scale1, u53(pcg_out(s1))));
            u = Add(0.0, Mul(P.envelope, u53(pcg_out(s2))));
        } else {
            u = Add(0.0, Mul(P.envelope, u53(pcg_out(s1))));
        }
        f(i0 + t, x0, x1, u);
    }
}

// density of a candidate; *inside for Dalitz; sets *err on a 1-D kernel error
__device__ __forceinline__ double pcg_density(const NllArgs& A, const PcgParams& P, double x0, double x1,
                                              bool* inside, bool* err) {
    if (P.dalitz) {
        *inside = in_boundary_exact(P.g, x0, x1);
        return *inside ? dalitz_intensity_literal(A.dal, x0, x1) : 0.0;
    }
    *inside = true;
    int rank = -1;
    double val = 0.0;
    ValLoader ld;
    ld.v[0] = x0;
    ld.v[1] = x1;
    const double d = literal_density_t(A, ld, &rank, &val);
    *err = rank >= 0;
    return d;
}

__global__ void __launch_bounds__(kGenThreads) pcg_count_kernel(const __grid_constant__ NllArgs A,
                                                                const __grid_constant__ PcgParams P) {
    const int c = blockIdx.x;
    const PcgChunk& ch = P.chunks[c];
    unsigned cnt = 0, ins = 0, amb = 0;
    double dm = 0.0;
    bool err = false;
    pcg_run(P, ch, threadIdx.x * kRun, [&](int, double x0, double x1, double u) {
        bool inside = false, e = false;
        const double d = pcg_density(A, P, x0, x1, &inside, &e);
        err |= e;
        ins += inside ? 1u : 0u;
        cnt += (u < d) ? 1u : 0u;
        amb += (d > 0.0 && fabs(u - d) <= d * 0x1p-47) ? 1u : 0u;
        dm = d > dm ? d : dm;  // NaN never raises the maximum (numpy: nan > env is False)
    });
    __shared__ unsigned s_cnt, s_ins, s_amb;
    __shared__ unsigned long long s_max;
    if (threadIdx.x == 0) {
        s_cnt = 0;
        s_ins = 0;
        s_amb = 0;
        s_max = 0;
    }
    __syncthreads();
    atomicAdd(&s_cnt, cnt);
    atomicAdd(&s_ins, ins);
    if (amb) atomicAdd(&s_amb, amb);
    atomicMax(&s_max, (unsigned long long)__double_as_longlong(dm));  // dm >= 0: bit order = value order
    if (err) atomicOr(P.errflag, 1ull);
    __syncthreads();
    if (threadIdx.x == 0) {
        P.count[c] = s_cnt;
        P.inside[c] = s_ins;
        P.ambig[c] = s_amb;
        P.dmax[c] = s_max;
    }
}

__global__ void __launch_bounds__(kGenThreads) pcg_write_kernel(const __grid_constant__ NllArgs A,
                                                                const __grid_constant__ PcgParams P) {
    const int c = blockIdx.x;
    const PcgChunk& ch = P.chunks[c];
    const int64_t take = P.take[c];
    if (take <= 0) return;
    // pass 1: accepted count of this thread's run
    unsigned cnt = 0;
    pcg_run(P, ch, threadIdx.x * kRun, [&](int, double x0, double x1, double u) {
        bool inside = false, e = false;
        const double d = pcg_density(A, P, x0, x1, &inside, &e);
        cnt += (u < d) ? 1u : 0u;
    });
    // exclusive scan over the block in thread (= candidate) order
    __shared__ unsigned warp_tot[kGenThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    unsigned incl = cnt;
#pragma unroll
    for (int off = 1; off < 32; off *= 2) {
        const unsigned v = __shfl_up_sync(0xffffffffu, incl, off);
        if (lane >= off) incl += v;
    }
    if (lane == 31) warp_tot[w] = incl;
    __syncthreads();
    unsigned before = 0;
    for (int q = 0; q < w; ++q) before += warp_tot[q];
    int64_t slot = (int64_t)before + incl - cnt;
    if (slot >= take || cnt == 0) return;
    // pass 2: write accepted candidates in order
    const int64_t base = P.pos[c];
    pcg_run(P, ch, threadIdx.x * kRun, [&](int, double x0, double x1, double u) {
        bool inside = false, e = false;
        const double d = pcg_density(A, P, x0, x1, &inside, &e);
        if (u < d) {
            if (slot < take) {
                P.out0[base + slot] = x0;
                if (P.dalitz) P.out1[base + slot] = x1;
            }
            ++slot;
        }
    });
}

// Envelope scans (mcgen.py:52-54 and 209-222): the maximum density over
// midpoint grids, as bits of a non-negative double.
__global__ void pcg_scan_1d_kernel(const __grid_constant__ NllArgs A, double lo, double step, int64_t points,
                                   unsigned long long* out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < points; i += (int64_t)gridDim.x * blockDim.x) {
        const double x = Add(lo, Mul((double)i + 0.5, step));
        int rank = -1;
        double val = 0.0;
        ValLoader ld;
        ld.v[0] = x;
        ld.v[1] = 0.0;
        const double d = literal_density_t(A, ld, &rank, &val);
        m = d > m ? d : m;
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

__global__ void pcg_scan_dalitz_kernel(const __grid_constant__ NllArgs A, GridConsts g, unsigned long long* out) {
    double m = 0.0;
    const int64_t total = (int64_t)g.nx * g.ny;
    for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(idx / g.ny), j = (int)(idx % g.ny);
        const double s12 = Add(g.lo12, Mul((double)i + 0.5, g.dx));
        const double s13 = Add(g.lo13, Mul((double)j + 0.5, g.dy));
        if (!in_boundary_exact(g, s12, s13)) continue;
        const double d = dalitz_intensity_literal(A.dal, s12, s13);
        m = d > m ? d : m;
    }
    atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

// ---------------------------------------------------------------------------
// host side

static u128 host_mul_add(u128 a, u128 s, u128 c) { return a * s + c; }

// (A, C) of n steps: s -> A s + C  (pcg_advance_lcg_128)
static void pcg_jump_of(uint64_t n, u128 inc, u128* A, u128* C) {
    u128 acc_a = 1, acc_c = 0, cur_a = pcg_mult(), cur_c = inc;
    while (n) {
        if (n & 1) {
            acc_a *= cur_a;
            acc_c = acc_c * cur_a + cur_c;
        }
        cur_c = (cur_a + 1) * cur_c;
        cur_a *= cur_a;
        n >>= 1;
    }
    *A = acc_a;
    *C = acc_c;
}

static u128 pcg_skip(u128 s, u128 inc, uint64_t n) {
    u128 a, c;
    pcg_jump_of(n, inc, &a, &c);
    return host_mul_add(a, s, c);
}

struct PcgHostResult {
    int status;  // 0 ok, 2 density error, 10 envelope hit, 11 attempts exhausted
    int64_t attempts, accepted, in_boundary, produced;
    double observed;
    int64_t ambiguous;  // candidates of the consumed chunks within 2^-47 of their decision
};

// The reference's chunk loop over one stream (mcgen.py:66-97 / 232-257).
cudaError_t pcg_generate(const NllArgs& A, PcgParams P, u128 state, int64_t n_wanted, int64_t budget,
                         double* out0, double* out1, cudaStream_t stream, PcgHostResult* R) {
    memset(R, 0, sizeof(*R));
    for (int b = 0; b < 14; ++b) pcg_jump_of(1ull << b, P.inc, &P.jump.a[b], &P.jump.c[b]);
    const int nd = P.dalitz ? 3 : 2;
    int64_t got = 0, attempts = 0;
    int64_t out_pos = 0;
    const int kMaxBatch = 2048;
    PcgChunk* d_chunks = nullptr;
    unsigned long long* d_words = nullptr;  // count, dmax, inside, ambig (4 x kMaxBatch) + errflag
    int64_t* d_pt = nullptr;                // pos, take
    cudaError_t e = cudaMalloc(&d_chunks, sizeof(PcgChunk) * kMaxBatch);
    if (e == cudaSuccess) e = cudaMalloc(&d_words, sizeof(unsigned long long) * (4 * kMaxBatch + 1));
    if (e == cudaSuccess) e = cudaMalloc(&d_pt, sizeof(int64_t) * 2 * kMaxBatch);
    std::vector<PcgChunk> h_chunks(kMaxBatch);
    std::vector<unsigned long long> h_words(4 * kMaxBatch + 1);
    std::vector<int64_t> h_pt(2 * kMaxBatch);
    double rate = 0.0;  // accepted per candidate, from the batches so far
    bool done = false;
    while (e == cudaSuccess && !done) {
        if (attempts >= budget) {
            R->status = 11;  // AttemptsExhausted
            break;
        }
        // batch size: enough chunks for the remaining events at the observed rate
        const int64_t remaining = n_wanted - got;
        int64_t want = rate > 0.0 ? (int64_t)(1.15 * (double)remaining / (rate * kChunk)) + 1 : 8;
        int nch = (int)(want < 1 ? 1 : (want > kMaxBatch ? kMaxBatch : want));
        int64_t a = attempts;
        int used = 0;
        for (int c = 0; c < nch && a < budget; ++c) {
            const int64_t k = budget - a < kChunk ? budget - a : kChunk;
            PcgChunk& ch = h_chunks[c];
            ch.k = (int)k;
            for (int r = 0; r < nd; ++r) ch.base[r] = pcg_skip(state, P.inc, (uint64_t)(r * k));
            state = pcg_skip(state, P.inc, (uint64_t)(nd * k));
            a += k;
            ++used;
        }
        nch = used;
        P.nch = nch;
        P.chunks = d_chunks;
        P.count = d_words;
        P.dmax = d_words + kMaxBatch;
        P.inside = d_words + 2 * kMaxBatch;
        P.ambig = d_words + 3 * kMaxBatch;
        P.errflag = d_words + 4 * kMaxBatch;
        P.pos = d_pt;
        P.take = d_pt + kMaxBatch;
        P.out0 = out0;
        P.out1 = out1;
        if ((e = cudaMemcpyAsync(d_chunks, h_chunks.data(), sizeof(PcgChunk) * nch, cudaMemcpyHostToDevice, stream)))
            break;
        if ((e = cudaMemsetAsync(P.errflag, 0, sizeof(unsigned long long), stream))) break;
        pcg_count_kernel<<<nch, kGenThreads, 0, stream>>>(A, P);
        if ((e = cudaGetLastError())) break;
        if ((e = cudaMemcpyAsync(h_words.data(), d_words, sizeof(unsigned long long) * (4 * kMaxBatch + 1),
                                 cudaMemcpyDeviceToHost, stream)))
            break;
        if ((e = cudaStreamSynchronize(stream))) break;
        if (h_words[4 * kMaxBatch]) {
            R->status = 2;  // a density kernel raised (NonFiniteDensity)
            break;
        }
        // walk the chunks exactly like the reference loop
        int last = -1;
        int64_t batch_acc = 0, batch_k = 0;
        for (int c = 0; c < nch; ++c) {
            const double dmax = __builtin_bit_cast(double, h_words[kMaxBatch + c]);
            const int64_t k = h_chunks[c].k;
            R->ambiguous += (int64_t)h_words[3 * kMaxBatch + c];
            if (fabs(dmax - P.envelope) <= P.envelope * 0x1p-47) ++R->ambiguous;  // the envelope check
            if (dmax > P.envelope) {  // _EnvelopeHit(max(dens)) before this chunk's acceptance
                R->status = 10;
                R->observed = dmax;
                attempts += k;
                break;
            }
            attempts += k;
            R->in_boundary += (int64_t)h_words[2 * kMaxBatch + c];
            const int64_t acc = (int64_t)h_words[c];
            batch_acc += acc;
            batch_k += k;
            const int64_t take = acc < n_wanted - got ? acc : n_wanted - got;
            h_pt[c] = out_pos;
            h_pt[kMaxBatch + c] = take;
            out_pos += take;
            // 1-D counts every accepted candidate (mcgen.py:91-92), Dalitz only those taken (250-253)
            R->accepted += P.dalitz ? take : acc;
            got += take;
            last = c;
            if (got >= n_wanted) {
                done = true;
                break;
            }
            if (attempts >= budget) break;
        }
        if (batch_k > 0) rate = (double)batch_acc / (double)batch_k;
        if (rate <= 0.0) rate = 0.0;
        if (last >= 0) {
            if ((e = cudaMemcpyAsync(d_pt, h_pt.data(), sizeof(int64_t) * kMaxBatch, cudaMemcpyHostToDevice, stream)))
                break;
            if ((e = cudaMemcpyAsync(d_pt + kMaxBatch, h_pt.data() + kMaxBatch, sizeof(int64_t) * (last + 1),
                                     cudaMemcpyHostToDevice, stream)))
                break;
            pcg_write_kernel<<<last + 1, kGenThreads, 0, stream>>>(A, P);
            if ((e = cudaGetLastError())) break;
            if ((e = cudaStreamSynchronize(stream))) break;
        }
        if (R->status) break;
    }
    R->attempts = attempts;
    R->produced = got;
    cudaFree(d_chunks);
    cudaFree(d_words);
    cudaFree(d_pt);
    return e;
}

cudaError_t pcg_generate_entry(const NllArgs& A, int dalitz, const double* box, double envelope,
                               const GridConsts* g, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                               uint64_t inc_lo, int64_t n_wanted, int64_t budget, double* out0, double* out1,
                               cudaStream_t stream, PcgHostResult* R) {
    PcgParams P;
    memset(&P, 0, sizeof(P));
    P.dalitz = dalitz;
    P.lo0 = box[0];
    P.scale0 = box[1];
    P.lo1 = box[2];
    P.scale1 = box[3];
    P.envelope = envelope;
    P.inc = ((u128)inc_hi << 64) | inc_lo;
    if (g) P.g = *g;
    const u128 state = ((u128)state_hi << 64) | state_lo;
    return pcg_generate(A, P, state, n_wanted, budget, out0, out1, stream, R);
}

cudaError_t pcg_scan_1d(const NllArgs& A, double lo, double hi, int64_t points, double* out_max,
                        unsigned long long* scratch, cudaStream_t stream, int sm_count) {
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(unsigned long long), stream);
    if (e) return e;
    const double step = (hi - lo) / (double)points;  // (hi - lo) / points, as numpy
    int64_t grid = (points + 255) / 256;
    if (grid > sm_count * 4) grid = sm_count * 4;
    pcg_scan_1d_kernel<<<(unsigned)grid, 256, 0, stream>>>(A, lo, step, points, scratch);
    if ((e = cudaGetLastError())) return e;
    unsigned long long bits = 0;
    if ((e = cudaMemcpyAsync(&bits, scratch, sizeof(bits), cudaMemcpyDeviceToHost, stream))) return e;
    if ((e = cudaStreamSynchronize(stream))) return e;
    *out_max = __builtin_bit_cast(double, bits);
    return cudaSuccess;
}

cudaError_t pcg_scan_dalitz(const NllArgs& A, const GridConsts& g, double* out_max, unsigned long long* scratch,
                            cudaStream_t stream, int sm_count) {
    cudaError_t e = cudaMemsetAsync(scratch, 0, sizeof(unsigned long long), stream);
    if (e) return e;
    pcg_scan_dalitz_kernel<<<sm_count * 4, 256, 0, stream>>>(A, g, scratch);
    if ((e = cudaGetLastError())) return e;
    unsigned long long bits = 0;
    if ((e = cudaMemcpyAsync(&bits, scratch, sizeof(bits), cudaMemcpyDeviceToHost, stream))) return e;
    if ((e = cudaStreamSynchronize(stream))) return e;
    *out_max = __builtin_bit_cast(double, bits);
    return cudaSuccess;
}

}  // namespace pfb
