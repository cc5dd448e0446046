// pfb_internal.cuh -- device-side plan layout, exact accumulator, IEEE helpers.
//
// Shared by the NLL kernels (pfb_nll.cu), the Dalitz grid kernels (pfb_dalitz.cu)
// and the C ABI (pfb_api.cu).  The accumulator helpers are __host__ __device__
// so the CPU test-suite exercises the very code the GPU runs.
#pragma once
#include <climits>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/pfb200.h"

#define PFB_HD __host__ __device__ __forceinline__
#ifdef __CUDA_ARCH__
// keep the 68-limb working set of the (once per launch) rounding in local memory
#define PFB_NOUNROLL _Pragma("unroll 1")
#else
#define PFB_NOUNROLL
#endif

namespace pfb {

PFB_HD double __longlong_as_double_hd(long long v) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(v);
#else
    double d;
    __builtin_memcpy(&d, &v, 8);
    return d;
#endif
}

constexpr int kBlock = PFB_BLOCK;        // 4096 events per reduction block
constexpr int kMaxNodes = 16;            // post-order ops of the literal interpreter
constexpr int kMaxCols = 4;              // distinct observable columns
constexpr int kMaxVals = 128;            // derived per-call values (literal path)
constexpr int kMaxLeaves = 4;            // sum-of-products leaves (fast path)
constexpr int kMaxTerms = 4;             // sum-of-products terms (fast path)
constexpr int kMaxDal = PFB_MAX_DALITZ_TERMS;
constexpr int kThreads = 256;            // CTA size of the NLL kernels
constexpr int kMaxPts = 16;              // parameter points evaluated in one pass
constexpr int kMaxPeers = 16;            // ranks of a peer-memory exchange
constexpr int kPeerSlotWords = 80;       // mailbox slot: 72 limbs + status word, padded
constexpr int kPtLeafWords = 16;         // per-point leaf values (mu, 1/sigma, alpha, coeffs)
constexpr int kPtWords = kPtLeafWords + 2 * kMaxTerms;  // + (log coef, threshold) per term

enum Evaluator : int32_t { EV_LITERAL = 0, EV_SOP = 1, EV_DALITZ = 2, EV_DALITZ_CACHED = 3 };

// ---------------------------------------------------------------------------
// Literal interpreter: one op per tree node, post-order.  Evaluates exactly
// the reference operation sequence (eval_batch recursion, pdf.py:251-269).
struct LitOp {
    int32_t kind;
    int32_t nchild;
    int32_t col0, col1;   // column slots (index into NllArgs::col)
    int32_t voff;         // offset of this node's derived values in NllArgs::v
    int32_t nv;
    int32_t rank;         // rank of this node's first check (evaluation order)
    int32_t dal;          // dalitz: index into NllArgs dalitz tables
};

// Sum-of-products flattening of add/prod trees over gaussian/exponential/
// polynomial leaves:  p(x) = sum_t coef_t * prod_{l in t} leaf_l(x).
struct SopLeaf {
    int32_t kind;  // PFB_GAUSSIAN / PFB_EXPONENTIAL / PFB_POLYNOMIAL
    int32_t col;   // column slot
    int32_t voff;  // gaussian: mu, 1/sigma; exponential: alpha; polynomial: coeffs
    int32_t nv;
};
struct SopTerm {
    uint32_t emask;   // exp-type leaves (gaussian/exponential) multiplied in
    uint32_t vmask;   // value-type leaves (polynomial) multiplied in
    double logcoef;   // log(coef_t)
    double coef;      // coef_t
    double thr;       // guard threshold on sum |u_l| (+ value-leaf exponent budget)
};

// Dalitz fast evaluator (dalitz.py:162-230): per-term constants.
struct DalTerm {
    int32_t pair;     // 12, 13, 23
    int32_t spin;     // 0, 1
    int32_t cached;   // amplitude read from the lineshape cache
    int32_t zinv;     // spin-1 Zemach needs 1/s_pair (constant != 0)
    double m2;        // m*m
    double mg;        // m*width
    double mg2;       // (m*width)^2
    double cre, cim;  // magnitude*(cos phase, sin phase)
    double alpha;     // cre*m^2 - cim*m*G
    double beta;      // cre*m*G + cim*m^2
    // the same four scaled by sqrt(1/norm) (ratio evaluator: |N|^2 / norm
    // without a per-event multiply)
    double scre, scim, salpha, sbeta;
};

struct DalDesc {
    int32_t K;
    int32_t ninv;     // number of 1/s_pair the Zemach factors need
    int32_t need12, need13, need23;
    double mss;       // M^2+m1^2+m2^2+m3^2 (DecayChannel.mass_sum_sq)
    double zc12, zc13, zc23;  // Zemach constants (M^2-m_k^2)(m_j^2-m_i^2)
    DalTerm t[kMaxDal];
    const double2* cache;     // lineshape cache base (K rows of n events, double2)
    int64_t cache_stride;     // events per row
};

struct NllArgs {
    const double* col[kMaxCols];
    int32_t ncols;
    int32_t vec2;             // double2 loads allowed
    int64_t begin;            // first event (store index)
    int64_t nfull;            // number of full 4096-blocks
    int32_t tail;             // events in the trailing partial block
    int32_t evaluator;
    int32_t warps;            // warps cooperating on one block (1,2,4,8)
    int32_t tma;              // 1: TMA bulk-copy pipeline for HBM-bound evaluators
    int32_t task_shell;       // pipeline 4: C1 / C5 single points on the warp-task kernel
    int32_t mode;             // KernelMode: export / add-export / accumulate
    int64_t idx_base;         // added to local event indices in error keys
    int64_t block_base;       // global block index of this range's block 0
    double* block_sums;       // optional per-block output (indexed block_base + b)
    unsigned long long* acc;  // PFB_ACC_WORDS persistent accumulator (self-resetting)
    unsigned int* ticket;     // CTA completion counter (self-resetting)
    unsigned long long* work_counter;  // dynamic block scheduler (self-resetting)
    unsigned long long* errkey;  // min (rank<<40 | local index), ~0 when clean
    unsigned long long* xkey;    // binned: first non-positive-expectation bin, exported into result_i[2]
    double* tail_scratch;     // 4096 doubles
    long long* acc_out;       // PFB_ACC_WORDS export target
    long long* result_i;      // [0] deferred-block count, [1] error key, [4] completion sequence
    long long seq;            // > 0: the exporting CTA posts it to result_i[4] last (host polls)

    unsigned long long* fix_counter;  // deferred-block list fill (self-resetting)
    int64_t* fix_list;        // deferred global block indices
    const long long* fix_count;       // list length for the fix-up launch (device)
    // task kernel (pfb_nll_task.cuh): fold slots of blocks split across CTAs
    double* gfold;            // [block][8 unit rows][32 lanes] unit values
    int* gbad;                // [block][8] uncertified flags
    unsigned int* gcnt;       // [block] arrivals (self-resetting)
    // literal interpreter
    int32_t nops;
    int32_t final_rank;       // rank of the root p > 0 check
    LitOp ops[kMaxNodes];
    double norm[kMaxNodes];   // per-node normalisation
    double v[kMaxVals];       // derived per-call values
    // sum-of-products
    int32_t nleaf, nterm;
    SopLeaf leaf[kMaxLeaves];  // voff indexes a ptv row
    SopTerm term[kMaxTerms];
    // SumPdf(gaussian, exponential) constants per parameter point (EvSum2GE):
    // c2 = -1/(2 sigma^2), alpha mu, the term coefficients c0 / c1, and the high
    // word of the certified bound on |x - mu|
    double g2_c2[kMaxPts], g2_amu[kMaxPts], g2_c0[kMaxPts], g2_c1[kMaxPts];
    int32_t g2_wlim[kMaxPts];
    int32_t g2_qcert;  // every point: q = c1 + c0 e^d provably in [2^-249, 2^249] for every x
    // batched objective: npts parameter points per pass over the data
    int32_t npts;
    int32_t fix_point;         // fix-up launch: the point whose deferred blocks it redoes
    double ptv[kMaxPts][kPtWords];
    // dalitz
    double inv_norm;          // 1/norm_root (fast paths)
    DalDesc dal;
    // fused cross-GPU exchange of the exact accumulator (pfb_nll_peer): the
    // CTA that finishes the launch trades its limbs with every rank's
    // mailbox over NVLink peer memory and exports the global sum
    long long* peer_mbox[kMaxPeers];
    int32_t peer_world;       // 0: no exchange
    int32_t peer_rank;
    unsigned long long peer_seq;
    long long peer_timeout;   // clock64 cycles of the bounded wait
};

// Persistent NLL kernel control (pfb_nll_task.cuh nll_persist_kernel): the
// doorbell [seq, op] and the call's NllArgs in mapped pinned host memory,
// their device copy and the CTA-release word [seq, op] in device memory.
// Mailbox of one call: the 128-byte chunks of the call's NllArgs that differ
// from the previous call (chunk indices, then their payloads).
constexpr int kArgChunk = 128;
constexpr int kMaxArgChunks = 64;  // >= ceil(sizeof(NllArgs) / 128)
struct PersistBox {
    unsigned long long nchunks;
    unsigned int idx[kMaxArgChunks];
    unsigned long long pad[7];
    unsigned char payload[kMaxArgChunks][kArgChunk];
};
struct NllArgs;
struct PersistCtl {
    const unsigned long long* host_seq;  // mapped: [0] sequence, [1] op (0 run, 1 stop)
    const PersistBox* host_args;         // mapped mailbox (changed chunks)
    unsigned int* dev_chunks;            // device: [0] count, [1..] changed chunk indices
    NllArgs* dev_args;                   // device copy of the mailbox
    unsigned long long* go;              // device: [0] released sequence, [1] op, [2] idle exit
    unsigned long long start_seq;        // the doorbell value at launch (== go[0])
    unsigned long long idle_ns;          // leave after this long without a call
    unsigned long long* trace;           // optional (mapped): %globaltimer stamps of the last call
};

// Peer mailbox layout (64-bit words): data [2][kMaxPeers][kPeerSlotWords],
// flags [2][kMaxPeers] (the separate exchange kernel), then the fused
// exchange's flag-in-line region [2][kMaxPeers][kPeerSlotWords] 16-byte lines
// {(seq << 32) | lo32, (seq << 32) | hi32}; parity = call sequence number & 1.
constexpr size_t kPeerLineBase = 2 * kMaxPeers * kPeerSlotWords + 2 * kMaxPeers;  // in 64-bit words
__host__ __device__ constexpr size_t peer_mbox_words() {
    return kPeerLineBase + 2 * 2 * kMaxPeers * kPeerSlotWords;
}
__device__ __forceinline__ ulonglong2* peer_line(long long* m, int par, int r, int w) {
    return reinterpret_cast<ulonglong2*>(m + kPeerLineBase) + ((size_t)par * kMaxPeers + r) * kPeerSlotWords + w;
}
// One limb split into two 64-bit elements, each carrying the call number in
// its high half.  A vector access is a set of element accesses in no
// particular order, but each 64-bit element is single-copy atomic: a reader
// that sees seq in both elements has both halves of this call's value, so no
// fence or separate flag orders data before a flag.
__device__ __forceinline__ void st_line(ulonglong2* p, long long v, unsigned seq) {
    const unsigned long long u = (unsigned long long)v;
    const unsigned long long tag = (unsigned long long)seq << 32;
    asm volatile("st.relaxed.sys.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(tag | (u & 0xffffffffull)),
                 "l"(tag | (u >> 32))
                 : "memory");
}
__device__ __forceinline__ bool ld_line(const ulonglong2* p, unsigned seq, long long* v) {
    unsigned long long a, b;
    asm volatile("ld.relaxed.sys.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
    if ((unsigned)(a >> 32) != seq || (unsigned)(b >> 32) != seq) return false;
    *v = (long long)(((b & 0xffffffffull) << 32) | (a & 0xffffffffull));
    return true;
}
__device__ __forceinline__ long long* peer_slot(long long* m, int par, int r) {
    return m + ((size_t)par * kMaxPeers + r) * kPeerSlotWords;
}
__device__ __forceinline__ unsigned long long* peer_flag(long long* m, int par, int r) {
    return reinterpret_cast<unsigned long long*>(m + 2 * kMaxPeers * kPeerSlotWords) + par * kMaxPeers + r;
}
__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Synthetic-event generators (pfb_gen.cu).
struct GenDalitz {
    DalDesc D;
    double lo12, hi12, lo13, hi13, m1sq, m2sq, m3sq, M2;
    double envelope;
    uint32_t seed_lo, seed_hi;
};
struct Gen1D {
    int kind;  // 0: f*Gauss + (1-f)*Exp on [lo,hi] (1 column); 1: Gauss(x) x Exp(y) (2 columns)
    double mu, sigma, alpha, f, lo, hi;
    uint32_t seed_lo, seed_hi;
};

// BinnedDataSet axes for bin_fill_kernel (core.py:339-379).
struct BinAxes {
    int32_t naxes;
    const double* col[kMaxCols];
    double lower[kMaxCols];
    double width[kMaxCols];
    long long nbins[kMaxCols];
};

// Dalitz integration grid constants (dalitz.py:246-264).
struct GridConsts {
    int nx, ny;
    double lo12, hi12, lo13, dx, dy;
    double m1sq, m2sq, m3sq, M2;
};

// ---------------------------------------------------------------------------
// Exact accumulator.  A finite double x = m * 2^(b-1074) with integer m < 2^53
// and b >= 0 is added as three signed 32-bit digits into int64 limbs
// [b/32, b/32+1, b/32+2].  Integer addition is associative, so any grouping of
// blocks, CTAs, shards and GPUs yields the same limbs; pfb::acc_round then
// returns the correctly rounded (round-half-even) exact sum == math.fsum.

struct Digits {
    int32_t limb;        // index of the lowest limb
    long long d[3];      // signed digits
    int32_t special;     // 0 finite, PFB_ACC_POSINF / NEGINF / NAN
};

PFB_HD Digits split_double(double x) {
    Digits r;
    r.limb = 0;
    r.d[0] = r.d[1] = r.d[2] = 0;
    r.special = 0;
    unsigned long long bits;
#ifdef __CUDA_ARCH__
    bits = (unsigned long long)__double_as_longlong(x);
#else
    __builtin_memcpy(&bits, &x, 8);
#endif
    const unsigned E = (unsigned)((bits >> 52) & 0x7ffu);
    const unsigned long long frac = bits & 0xfffffffffffffull;
    const bool neg = (bits >> 63) != 0;
    if (E == 0x7ffu) {
        r.special = frac ? PFB_ACC_NAN : (neg ? PFB_ACC_NEGINF : PFB_ACC_POSINF);
        return r;
    }
    unsigned long long m;
    unsigned b;
    if (E == 0) {
        m = frac;
        b = 0;
    } else {
        m = frac | (1ull << 52);
        b = E - 1;
    }
    if (m == 0) return r;
    const unsigned s = b & 31u;
    r.limb = (int32_t)(b >> 5);
    const unsigned long long lo = m << s;
    const unsigned long long hi = s ? (m >> (64 - s)) : 0ull;
    long long d0 = (long long)(lo & 0xffffffffull);
    long long d1 = (long long)(lo >> 32);
    long long d2 = (long long)hi;
    if (neg) {
        d0 = -d0;
        d1 = -d1;
        d2 = -d2;
    }
    r.d[0] = d0;
    r.d[1] = d1;
    r.d[2] = d2;
    return r;
}

#ifdef __CUDACC__
// Exact accumulation of one double into a CTA's shared accumulator (the
// digits of split_double added with integer atomics).
__device__ __forceinline__ void acc_add_shared(long long* sacc, double x) {
    const Digits d = split_double(x);
    if (d.special) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&sacc[d.special]), 1ull);
        return;
    }
#pragma unroll
    for (int i = 0; i < 3; ++i)
        if (d.d[i])
            atomicAdd(reinterpret_cast<unsigned long long*>(&sacc[d.limb + i]),
                      (unsigned long long)d.d[i]);
}

// Warp-aggregated acc_add_shared for kernels that produce one term per thread
// (quadrature, binned): the 32 lanes' digits are summed per limb with
// shuffles (integer, exact) and one lane adds each limb sum, so a CTA issues
// ~8 shared atomics per warp instead of 3 per thread (64-bit shared atomics
// are CAS loops; 256 threads on the same few limbs serialise for tens of us).
// Must be called by all 32 lanes; inactive lanes pass act = false.  Terms
// spread over more than kWarpSpan limbs, and inf/NaN, take the per-lane path.
__device__ __forceinline__ void acc_add_warp(long long* sacc, double x, bool act) {
    constexpr unsigned kFull = 0xffffffffu;
    constexpr int kWarpSpan = 6;
    const Digits d = split_double(x);
    if (act && d.special) {
        atomicAdd(reinterpret_cast<unsigned long long*>(&sacc[d.special]), 1ull);
        act = false;
    }
    if (act && !(d.d[0] | d.d[1] | d.d[2])) act = false;
    const int lo = __reduce_min_sync(kFull, act ? d.limb : INT_MAX);
    const int hi = __reduce_max_sync(kFull, act ? d.limb : INT_MIN);
    if (lo == INT_MAX) return;
    if (hi - lo > kWarpSpan) {
        if (act) acc_add_shared(sacc, x);
        return;
    }
    const bool lead = (threadIdx.x & 31) == 0;
    for (int k = lo; k <= hi + 2; ++k) {
        const int off = k - d.limb;
        long long c = !act ? 0 : off == 0 ? d.d[0] : off == 1 ? d.d[1] : off == 2 ? d.d[2] : 0;
#pragma unroll
        for (int s = 16; s; s >>= 1) c += __shfl_xor_sync(kFull, c, s);
        if (lead && c) atomicAdd(reinterpret_cast<unsigned long long*>(&sacc[k]), (unsigned long long)c);
    }
}

#endif  // __CUDACC__

PFB_HD void acc_add_host(long long* acc, double x) {
    Digits d = split_double(x);
    if (d.special) {
        acc[d.special] += 1;
        return;
    }
    acc[d.limb] += d.d[0];
    acc[d.limb + 1] += d.d[1];
    acc[d.limb + 2] += d.d[2];
}

PFB_HD int clz32(unsigned v) {
#ifdef __CUDA_ARCH__
    return __clz((int)v);
#else
    return v ? __builtin_clz(v) : 32;
#endif
}

PFB_HD double ldexp_exact(double m, int e) {
    // m * 2^e for an exactly representable result (or overflow to inf).
#ifdef __CUDA_ARCH__
    return ldexp(m, e);
#else
    return __builtin_ldexp(m, e);
#endif
}

// Correctly rounded value of the accumulator.  Returns PFB_OK or
// PFB_E_INVALID_SUM (+inf and -inf both present, as math.fsum raises).
PFB_HD int acc_round(const long long* acc_in, double* out) {
    const long long pinf = acc_in[PFB_ACC_POSINF], ninf = acc_in[PFB_ACC_NEGINF];
    if (acc_in[PFB_ACC_NAN] > 0) {
        *out = __longlong_as_double_hd(0x7ff8000000000000ll);
        return PFB_OK;
    }
    if (pinf > 0 && ninf > 0) {
        *out = __longlong_as_double_hd(0x7ff8000000000000ll);
        return PFB_E_INVALID_SUM;
    }
    if (pinf > 0) {
        *out = __longlong_as_double_hd(0x7ff0000000000000ll);
        return PFB_OK;
    }
    if (ninf > 0) {
        *out = __longlong_as_double_hd((long long)0xfff0000000000000ull);
        return PFB_OK;
    }
    long long L[PFB_NLIMBS];
    PFB_NOUNROLL for (int i = 0; i < PFB_NLIMBS; ++i) L[i] = acc_in[i];
    // carry-normalise: limbs 0..66 into [0, 2^32), the top limb keeps the sign
    PFB_NOUNROLL for (int i = 0; i < PFB_NLIMBS - 1; ++i) {
        const long long c = L[i] >> 32;  // arithmetic shift = floor division
        L[i] -= (long long)((unsigned long long)c << 32);
        L[i + 1] += c;
    }
    bool neg = L[PFB_NLIMBS - 1] < 0;
    if (neg) {
        PFB_NOUNROLL for (int i = 0; i < PFB_NLIMBS; ++i) L[i] = -L[i];
        PFB_NOUNROLL for (int i = 0; i < PFB_NLIMBS - 1; ++i) {
            const long long c = L[i] >> 32;
            L[i] -= (long long)((unsigned long long)c << 32);
            L[i + 1] += c;
        }
    }
    if (L[PFB_NLIMBS - 1] >= (1ll << 32)) {  // far beyond DBL_MAX
        *out = neg ? __longlong_as_double_hd((long long)0xfff0000000000000ull)
                   : __longlong_as_double_hd(0x7ff0000000000000ll);
        return PFB_OK;
    }
    int h = PFB_NLIMBS - 1;
    PFB_NOUNROLL while (h >= 0 && L[h] == 0) --h;
    if (h < 0) {
        *out = 0.0;  // math.fsum of zeros is +0.0
        return PFB_OK;
    }
    const int bitlen = 32 * h + (32 - clz32((unsigned)L[h]));
    double r;
    if (bitlen <= 64) {
        unsigned long long k = 0;
        PFB_NOUNROLL for (int i = h; i >= 0; --i) k = (k << 32) | (unsigned long long)L[i];
        unsigned long long m = k;
        int e = -1074;
        if (bitlen > 53) {  // round k to 53 significant bits, half-even
            const int sh = bitlen - 53;
            const unsigned long long rem = k & ((1ull << sh) - 1);
            const unsigned long long half = 1ull << (sh - 1);
            m = k >> sh;
            if (rem > half || (rem == half && (m & 1ull))) m += 1;
            e += sh;
        }
        r = ldexp_exact((double)m, e);
    } else {
        const int top = bitlen - 64;  // bit index of the window's lsb
        const int i0 = top >> 5, s = top & 31;
        unsigned long long w;
        {
            const unsigned long long a0 = (unsigned long long)L[i0];
            const unsigned long long a1 = (i0 + 1 < PFB_NLIMBS) ? (unsigned long long)L[i0 + 1] : 0;
            const unsigned long long a2 = (i0 + 2 < PFB_NLIMBS) ? (unsigned long long)L[i0 + 2] : 0;
            const unsigned long long lo64 = a0 | (a1 << 32);
            w = s ? ((lo64 >> s) | (a2 << (64 - s))) : lo64;
        }
        bool sticky = s ? (((unsigned long long)L[i0] & ((1ull << s) - 1)) != 0) : false;
        PFB_NOUNROLL for (int i = 0; i < i0 && !sticky; ++i) sticky = L[i] != 0;
        unsigned long long m = w >> 11;
        const unsigned long long rem = w & 0x7ffull;
        if (rem > 0x400ull || (rem == 0x400ull && (sticky || (m & 1ull)))) m += 1;
        // m may become 2^53: still exact as a double, ldexp handles it
        r = ldexp_exact((double)m, top + 11 - 1074);
    }
    *out = neg ? -r : r;
    return PFB_OK;
}

}  // namespace pfb
