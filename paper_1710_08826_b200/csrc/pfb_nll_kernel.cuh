// pfb_nll_kernel.cuh -- evaluators and the fused NLL kernel template.
//
// One launch evaluates -ln(p) for every event of a range, reduces each
// 4096-event block with the reference's half-folding tree (reduction.py:28-42),
// sums the ragged tail block with the reference's split recursion
// (reduction.py:45-56), and adds every block sum into an exact integer
// accumulator (replacing math.fsum, engine.py:240-243).  The last CTA to finish
// rounds the accumulator once, so one launch returns the NLL bit-for-bit equal
// to the reference's block structure, independent of grid size or GPU count.
//
// Mapping of one 4096-event block onto P warps (P = 1, 2, 4, 8):
//   element e = 2*lane + {0,1} + 64*w + 64*P*k,   k in [0, 64/P)
// bit 0 lives inside a thread (double2 loads), bits 1..5 are the lane, the
// next log2(P) bits the warp, the top bits the per-thread slot k.  The
// reference tree combines element bit 11 first and bit 0 last, so the fold
// order is: slots (registers, streamed in bit-reversed chunks and combined
// with a binary counter) -> warps (shared memory) -> lanes (shuffles) -> the
// final x+y.  Every addition pairs exactly the operands the reference pairs,
// hence identical bits.
#pragma once
#include <math.h>

#include "pfb_internal.cuh"
#include "pfb_math.cuh"

namespace pfb {


__device__ __forceinline__ bool finite(double x) { return isfinite(x); }

// 16-byte streaming load of two consecutive events (the host guarantees an
// even range start and 16-byte aligned columns, re-staging otherwise).
__device__ __forceinline__ double2 ld2(const double* __restrict__ p) {
    return __ldg(reinterpret_cast<const double2*>(p));
}

__device__ __forceinline__ void record_failure(const NllArgs& A, int rank, int64_t local,
                                               long long* sacc) {
    const unsigned long long key =
        ((unsigned long long)(unsigned)rank << 40) | (unsigned long long)(A.idx_base + local);
    atomicMin(A.errkey, key);
    atomicAdd(reinterpret_cast<unsigned long long*>(&sacc[PFB_ACC_FAILS]), 1ull);
}

// |sum_k c_k A_k|^2, reference order (dalitz.py:217-230).
__device__ __forceinline__ double dalitz_intensity_literal(const DalDesc& D, double s12,
                                                           double s13) {
    double tr = 0.0, ti = 0.0;
    for (int k = 0; k < D.K; ++k) {
        const DalTerm& T = D.t[k];
        const double2 a = dalitz_amp_literal(D, T, s12, s13);
        const double cr = Sub(Mul(T.cre, a.x), Mul(T.cim, a.y));
        const double ci = Add(Mul(T.cre, a.y), Mul(T.cim, a.x));
        if (k == 0) {
            tr = cr;
            ti = ci;
        } else {
            tr = Add(tr, cr);
            ti = Add(ti, ci);
        }
    }
    return Sub(Mul(tr, tr), Mul(ti, Sub(0.0, ti)));
}

// ---------------------------------------------------------------------------
// Literal interpreter: the exact reference evaluation of one event.  Used for
// trees without a fast evaluator and, per event, whenever a fast evaluator's
// guard cannot prove that the reference computation is free of underflow,
// overflow and density errors.  Returns -ln p, or NaN with `rank` set.
static __device__ __noinline__ double literal_event(const NllArgs& A, int64_t j, int* rank, double* val) {
    double st[kMaxNodes];
    int sid[kMaxNodes];
    int sp = 0;
    for (int o = 0; o < A.nops; ++o) {
        const LitOp& op = A.ops[o];
        double v = 0.0;
        switch (op.kind) {
            case PFB_GAUSSIAN: {
                const double x = A.col[op.col0][j];
                const double z = Div(Sub(x, A.v[op.voff]), A.v[op.voff + 1]);
                v = exp(Mul(Mul(-0.5, z), z));
                if (!finite(v)) {
                    *rank = op.rank;
                    *val = __longlong_as_double(0x7ff8000000000000ll);
                    return *val;
                }
                break;
            }
            case PFB_EXPONENTIAL: {
                const double x = A.col[op.col0][j];
                v = exp(Mul(A.v[op.voff], x));
                if (!finite(v)) {
                    *rank = op.rank;
                    *val = __longlong_as_double(0x7ff8000000000000ll);
                    return *val;
                }
                break;
            }
            case PFB_POLYNOMIAL: {
                const double x = A.col[op.col0][j];
                const double* c = A.v + op.voff;
                const int n = op.nv;
                v = Add(c[n - 1], Mul(x, 0.0));
                for (int i = 2; i <= n; ++i) v = Add(c[n - i], Mul(v, x));
                if (!finite(v)) {
                    *rank = op.rank;
                    *val = __longlong_as_double(0x7ff8000000000000ll);
                    return *val;
                }
                if (v < 0.0) {
                    *rank = op.rank + 1;
                    *val = v;
                    return __longlong_as_double(0x7ff8000000000000ll);
                }
                break;
            }
            case PFB_ADD: {
                const int k = op.nchild, base = sp - k;
                const double* w = A.v + op.voff;
                v = Mul(w[0], Div(st[base], A.norm[sid[base]]));
                for (int c = 1; c < k; ++c)
                    v = Add(v, Mul(w[c], Div(st[base + c], A.norm[sid[base + c]])));
                sp = base;
                break;
            }
            case PFB_PROD: {
                const int k = op.nchild, base = sp - k;
                v = Div(st[base], A.norm[sid[base]]);
                for (int c = 1; c < k; ++c) v = Mul(v, Div(st[base + c], A.norm[sid[base + c]]));
                sp = base;
                break;
            }
            case PFB_DALITZ: {
                v = dalitz_intensity_literal(A.dal, A.col[op.col0][j], A.col[op.col1][j]);
                break;
            }
            default:
                break;
        }
        st[sp] = v;
        sid[sp] = o;
        ++sp;
    }
    const double p = Div(st[0], A.norm[A.nops - 1]);
    if (!(p > 0.0)) {
        *rank = A.final_rank;
        *val = p;
        return __longlong_as_double(0x7ff8000000000000ll);
    }
    return -log(p);
}

__device__ __forceinline__ double literal_or_fail(const NllArgs& A, int64_t local,
                                                  long long* sacc) {
    int rank = -1;
    double val = 0.0;
    const double t = literal_event(A, A.begin + local, &rank, &val);
    if (rank >= 0) record_failure(A, rank, local, sacc);
    return t;
}

// ---------------------------------------------------------------------------
// Evaluators.  eval2 computes -ln p for the events (local, local+1) whose
// column values are x[c]; events the fast path cannot certify go through the
// literal interpreter (which also reports the reference's errors).

// Reduction known-answer mode: column 0 already holds the terms.
struct EvTerms {
    static constexpr int NC = 1;
    static constexpr int U = 8;
    __device__ static __forceinline__ double2 eval2(const NllArgs&, const double2 (&x)[1], int64_t,
                                                    long long*, int) {
        return x[0];
    }
};

// Literal interpreter for every event (arbitrary trees).
template <int NC_>
struct EvLiteral {
    static constexpr int NC = NC_;
    static constexpr int U = 1;
    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&)[NC_],
                                                    int64_t local, long long* sacc, int nvalid) {
        double2 t;
        t.x = literal_or_fail(A, local, sacc);
        t.y = nvalid > 1 ? literal_or_fail(A, local + 1, sacc) : 0.0;
        return t;
    }
};

// Sum of products in the log domain:
//   p = sum_t coef_t * V_t * exp(U_t),  U_t = sum of gaussian/exponential
//   exponents in term t, V_t = product of polynomial values in term t.
// Guard: every exponent |u| <= 600 and every term's log-magnitude budget below
// its host-computed threshold => the reference computation has no underflow,
// overflow, non-finite or non-positive value, so both agree to rounding.
template <int NC_>
struct EvSop {
    static constexpr int NC = NC_;
    static constexpr int U = 4;

    __device__ static __forceinline__ double pick(const double2 (&x)[NC_], int col, int which) {
        double r = which ? x[0].y : x[0].x;
#pragma unroll
        for (int c = 1; c < NC_; ++c)
            if (col == c) r = which ? x[c].y : x[c].x;
        return r;
    }

    __device__ static __forceinline__ double one(const NllArgs& A, const double2 (&x)[NC_],
                                                 int which, bool* ok) {
        double u[kMaxLeaves];
        double lv[kMaxLeaves];  // |log2| budget of value leaves
        bool good = true;
#pragma unroll
        for (int l = 0; l < kMaxLeaves; ++l) {
            u[l] = 0.0;
            lv[l] = 0.0;
            if (l < A.nleaf) {
                const SopLeaf& L = A.leaf[l];
                const double xv = pick(x, L.col, which);
                if (L.kind == PFB_GAUSSIAN) {
                    const double z = (xv - A.v[L.voff]) * A.v[L.voff + 1];
                    u[l] = -0.5 * z * z;
                    good &= (u[l] >= -600.0) || (u[l] < -746.0);
                } else if (L.kind == PFB_EXPONENTIAL) {
                    u[l] = A.v[L.voff] * xv;
                    good &= (fabs(u[l]) <= 600.0) || (u[l] < -746.0);
                } else {  // polynomial value (Horner, as np.polynomial.polynomial.polyval)
                    const double* c = A.v + L.voff;
                    double acc = c[L.nv - 1];
                    for (int i = 2; i <= L.nv; ++i) acc = fma(acc, xv, c[L.nv - i]);
                    u[l] = acc;
                    const int e = ((__double2hiint(acc) >> 20) & 0x7ff) - 1023;
                    good &= (acc > 0.0) && (e > -900) && (e < 900);
                    lv[l] = fabs((double)e) * 0.6931471805599453 + 1.0;
                }
            }
        }
        double L0 = 0.0, V0 = 1.0, Lm = -1e300, s = 0.0;
        bool live = false;
        double Lt[kMaxTerms], Vt[kMaxTerms];
#pragma unroll
        for (int t = 0; t < kMaxTerms; ++t) {
            Lt[t] = -1e300;
            Vt[t] = 1.0;
            if (t < A.nterm) {
                const SopTerm& T = A.term[t];
                double lsum = T.logcoef, budget = 0.0, vprod = 1.0;
                bool dead = false;  // a leaf underflows to exactly 0 in the reference
#pragma unroll
                for (int l = 0; l < kMaxLeaves; ++l) {
                    if ((T.emask >> l) & 1u) {
                        lsum += u[l];
                        budget += fabs(u[l]);
                        dead |= (u[l] < -746.0);
                    }
                    if ((T.vmask >> l) & 1u) {
                        vprod *= u[l];
                        budget += lv[l];
                    }
                }
                good &= dead || (budget <= T.thr);
                live |= !dead;
                Lt[t] = dead ? -1e300 : lsum;
                Vt[t] = vprod;
                Lm = fmax(Lm, Lt[t]);
            }
        }
        *ok = good && live;
        if (A.nterm == 1) {
            L0 = Lt[0];
            V0 = Vt[0];
            return (A.term[0].vmask ? -(L0 + log(V0)) : -L0);
        }
        if (A.nterm == 2) {
            const double d = Lt[0] - Lt[1];
            const double e = exp(-fabs(d));
            s = d >= 0.0 ? fma(Vt[1], e, Vt[0]) : fma(Vt[0], e, Vt[1]);
            return -(fmax(Lt[0], Lt[1]) + log(s));
        }
#pragma unroll
        for (int t = 0; t < kMaxTerms; ++t)
            if (t < A.nterm) s = fma(Vt[t], exp(Lt[t] - Lm), s);
        return -(Lm + log(s));
    }

    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&x)[NC_],
                                                    int64_t local, long long* sacc, int nvalid) {
        bool ok0, ok1;
        double2 t;
        t.x = one(A, x, 0, &ok0);
        t.y = one(A, x, 1, &ok1);
        if (!ok0) t.x = literal_or_fail(A, local, sacc);
        if (!ok1 && nvalid > 1) t.y = literal_or_fail(A, local + 1, sacc);
        return t;
    }
};

// Dalitz coherent sum, recompute path, K terms known at compile time.
// All K Breit-Wigner denominators and the Zemach 1/s_pair share ONE
// reciprocal through Montgomery batch inversion.
template <int K>
struct EvDalitz {
    static constexpr int NC = 2;
    static constexpr int U = 2;

    __device__ static __forceinline__ double one(const NllArgs& A, double s12, double s13,
                                                 bool* ok) {
        const DalDesc& D = A.dal;
        constexpr int KK = (K > 0 ? K : 1);
        const double s23 = (D.mss - s12) - s13;
        double a[KK], d[KK + 3], P[KK + 3];
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            const DalTerm& T = D.t[k];
            const double s = T.pair == 12 ? s12 : (T.pair == 13 ? s13 : s23);
            a[k] = T.m2 - s;
            d[k] = fma(a[k], a[k], T.mg2);
        }
        int n = KK;
        d[KK] = s12;
        d[KK + 1] = s13;
        d[KK + 2] = s23;
        // prefix products over the used denominators
        P[0] = d[0];
#pragma unroll
        for (int k = 1; k < KK; ++k) P[k] = P[k - 1] * d[k];
        double last = P[KK - 1];
        if (D.need12) last = last * s12;
        P[KK] = last;
        if (D.need13) last = last * s13;
        P[KK + 1] = last;
        if (D.need23) last = last * s23;
        P[KK + 2] = last;
        (void)n;
        double inv = 1.0 / last;
        bool good = (last > 1e-280) && (last < 1e280);
        double r23 = 0.0, r13 = 0.0, r12 = 0.0;
        if (D.need23) {
            r23 = inv * P[KK + 1];
            inv = inv * s23;
        }
        if (D.need13) {
            r13 = inv * P[KK];
            inv = inv * s13;
        }
        if (D.need12) {
            r12 = inv * P[KK - 1];
            inv = inv * s12;
        }
        double r[KK];
#pragma unroll
        for (int k = KK - 1; k >= 1; --k) {
            r[k] = inv * P[k - 1];
            inv = inv * d[k];
        }
        r[0] = inv;
        double tr = 0.0, ti = 0.0;
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            const DalTerm& T = D.t[k];
            double br = a[k] * r[k];
            double bi = T.mg * r[k];
            if (T.spin == 1) {
                double z;
                if (T.pair == 12)
                    z = fma(D.zc12, r12, s13 - s23);
                else if (T.pair == 13)
                    z = fma(D.zc13, r13, s12 - s23);
                else
                    z = fma(D.zc23, r23, s12 - s13);
                br *= z;
                bi *= z;
            }
            tr = fma(T.cre, br, fma(-T.cim, bi, tr));
            ti = fma(T.cre, bi, fma(T.cim, br, ti));
        }
        const double I = fma(tr, tr, ti * ti);
        const double p = I * A.inv_norm;
        good &= (p > 1e-300) && (p < 1e300);
        *ok = good;
        return -log(p);
    }

    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&x)[2],
                                                    int64_t local, long long* sacc, int nvalid) {
        bool ok0, ok1;
        double2 t;
        t.x = one(A, x[0].x, x[1].x, &ok0);
        t.y = one(A, x[0].y, x[1].y, &ok1);
        if (!ok0) t.x = literal_or_fail(A, local, sacc);
        if (!ok1 && nvalid > 1) t.y = literal_or_fail(A, local + 1, sacc);
        return t;
    }
};

// Dalitz with the lineshape cache: amplitudes of cached terms are read from
// HBM (K rows of double2 per event); the remaining terms are recomputed.
struct EvDalitzCached {
    static constexpr int NC = 2;
    static constexpr int U = 2;

    __device__ static __forceinline__ double one(const NllArgs& A, double s12, double s13,
                                                 int64_t local, bool* ok) {
        const DalDesc& D = A.dal;
        const double s23 = (D.mss - s12) - s13;
        double tr = 0.0, ti = 0.0;
        for (int k = 0; k < D.K; ++k) {
            const DalTerm& T = D.t[k];
            double br, bi;
            if (T.cached) {
                const double2 amp = __ldg(D.cache + (int64_t)k * D.cache_stride + local);
                br = amp.x;
                bi = amp.y;
            } else {
                const double s = T.pair == 12 ? s12 : (T.pair == 13 ? s13 : s23);
                const double a = T.m2 - s;
                const double r = 1.0 / fma(a, a, T.mg2);
                br = a * r;
                bi = T.mg * r;
                if (T.spin == 1) {
                    double z;
                    if (T.pair == 12)
                        z = (s13 - s23) + D.zc12 / s12;
                    else if (T.pair == 13)
                        z = (s12 - s23) + D.zc13 / s13;
                    else
                        z = (s12 - s13) + D.zc23 / s23;
                    br *= z;
                    bi *= z;
                }
            }
            tr = fma(T.cre, br, fma(-T.cim, bi, tr));
            ti = fma(T.cre, bi, fma(T.cim, br, ti));
        }
        const double I = fma(tr, tr, ti * ti);
        const double p = I * A.inv_norm;
        *ok = (p > 1e-300) && (p < 1e300);
        return -log(p);
    }

    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&x)[2],
                                                    int64_t local, long long* sacc, int nvalid) {
        bool ok0, ok1;
        double2 t;
        t.x = one(A, x[0].x, x[1].x, local, &ok0);
        t.y = one(A, x[0].y, x[1].y, local + 1, &ok1);
        if (!ok0) t.x = literal_or_fail(A, local, sacc);
        if (!ok1 && nvalid > 1) t.y = literal_or_fail(A, local + 1, sacc);
        return t;
    }
};

// ---------------------------------------------------------------------------
// Reference split-recursion pairwise sum (reduction.py:45-56) of a[0..n).
static __device__ __noinline__ double pairwise_serial(const double* a, int n) {
    // explicit stack of (start, len, state); depth <= log2(4096/8)+1
    if (n <= 0) return 0.0;
    struct Frame {
        int start, len, stage;
        double left;
    };
    Frame st[16];
    int sp = 0;
    st[0] = {0, n, 0, 0.0};
    double ret = 0.0;
    while (sp >= 0) {
        Frame& f = st[sp];
        if (f.len <= 8) {
            double s = a[f.start];
            for (int k = 1; k < f.len; ++k) s = Add(s, a[f.start + k]);
            ret = s;
            --sp;
            continue;
        }
        const int half = f.len / 2;
        if (f.stage == 0) {
            f.stage = 1;
            st[sp + 1] = {f.start, half, 0, 0.0};
            ++sp;
        } else if (f.stage == 1) {
            f.left = ret;
            f.stage = 2;
            st[sp + 1] = {f.start + half, f.len - half, 0, 0.0};
            ++sp;
        } else {
            ret = Add(f.left, ret);
            --sp;
        }
    }
    return ret;
}

// Warp-parallel evaluation of the same recursion: the top D levels of the
// recursion tree (all of whose nodes split) are spread over 2^D lanes.
static __device__ __noinline__ double pairwise_warp(const double* a, int n, int lane) {
    int D = 0;
    while (D < 5 && (n >> D) > 8 * 2) ++D;  // every node above depth D has > 8 elements
    // Nodes at depth < D have size >= floor(n / 2^(D-1)) > 16 > 8, so they split.
    double v = 0.0;
    if (lane < (1 << D)) {
        int start = 0, len = n;
        for (int b = D - 1; b >= 0; --b) {
            const int half = len / 2;
            if ((lane >> b) & 1) {
                start += half;
                len -= half;
            } else {
                len = half;
            }
        }
        v = pairwise_serial(a + start, len);
    }
    // combine bottom-up: depth D-1 pairs lanes (2i, 2i+1), ...
    for (int b = 0; b < D; ++b) {
        const double o = __shfl_down_sync(0xffffffffu, v, 1 << b);
        if ((lane & ((2 << b) - 1)) == 0) v = Add(v, o);
    }
    return __shfl_sync(0xffffffffu, v, 0);
}

template <int P>
__device__ __forceinline__ void group_sync(int grp) {
    if (P == 1) {
        __syncwarp();
    } else {
        asm volatile("bar.sync %0, %1;" ::"r"(grp + 1), "r"(P * 32) : "memory");
    }
}

template <int BITS>
__device__ __forceinline__ constexpr int bitrev(int v) {
    int r = 0;
#pragma unroll
    for (int i = 0; i < BITS; ++i) r |= ((v >> i) & 1) << (BITS - 1 - i);
    return r;
}

template <int N>
struct Log2 {
    static constexpr int value = 1 + Log2<N / 2>::value;
};
template <>
struct Log2<1> {
    static constexpr int value = 0;
};

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

// Rounding runs once per launch in one thread: keep its 68-limb working set
// out of the kernel's register allocation.
static __device__ __noinline__ int acc_round_dev(const long long* acc, double* out) {
    return acc_round(acc, out);
}

// ---------------------------------------------------------------------------
template <int P, class Ev>
__global__ void __launch_bounds__(kThreads, 1) nll_kernel(const __grid_constant__ NllArgs A) {
    constexpr int NC = Ev::NC;
    constexpr int GROUPS = kThreads / (32 * P);
    constexpr int KPT = 64 / P;                       // double2 slots per thread per block
    constexpr int U = Ev::U < KPT ? Ev::U : KPT;      // slots per streamed chunk
    constexpr int G = KPT / U;                        // chunks
    constexpr int LG = Log2<G>::value;

    __shared__ double2 xch[GROUPS][P][32];
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
    for (int64_t it = (int64_t)blockIdx.x * GROUPS + grp; it < nitems;
         it += (int64_t)gridDim.x * GROUPS) {
        double bsum = 0.0;
        int64_t bidx;
        if (A.tail && it == 0) {
            // ---- ragged tail block: terms to scratch, then split recursion
            bidx = A.nfull;
            const int64_t lbase = A.nfull * (int64_t)kBlock;  // local index of tail start
            const int n = A.tail;
#pragma unroll 1
            for (int e = 2 * (wig * 32 + lane); e < n; e += 64 * P) {
                double2 x[NC];
                const bool pair = e + 1 < n;
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const double* p = A.col[c] + A.begin + lbase + e;
                    x[c] = pair ? ld2(p) : make_double2(__ldg(p), __ldg(p));
                }
                const double2 t = Ev::eval2(A, x, lbase + e, sacc, pair ? 2 : 1);
                A.tail_scratch[e] = t.x;
                if (pair) A.tail_scratch[e + 1] = t.y;
            }
            __threadfence_block();
            group_sync<P>(grp);
            if (wig == 0) bsum = pairwise_warp(A.tail_scratch, n, lane);
            group_sync<P>(grp);
        } else {
            // ---- full block, reference half-folding tree
            bidx = it - (A.tail ? 1 : 0);
            const int64_t lbase = bidx * (int64_t)kBlock;
            const int64_t lthr = lbase + 2 * lane + 64 * wig;
            double2 lvl[LG > 0 ? LG : 1];
            double2 T = make_double2(0.0, 0.0);
#pragma unroll 1
            for (int g = 0; g < G; ++g) {
                const int cidx = LG ? (int)(__brev((unsigned)g) >> (32 - LG)) : 0;
                double2 x[U][NC];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int64_t off = lthr + 64 * P * (int64_t)(cidx + G * q);
#pragma unroll
                    for (int c = 0; c < NC; ++c) x[q][c] = ld2(A.col[c] + A.begin + off);
                }
                double2 t[U];
#pragma unroll
                for (int q = 0; q < U; ++q)
                    t[q] = Ev::eval2(A, x[q], lthr + 64 * P * (int64_t)(cidx + G * q), sacc, 2);
#pragma unroll
                for (int h = U / 2; h >= 1; h /= 2) {
#pragma unroll
                    for (int q = 0; q < h; ++q) {
                        t[q].x = Add(t[q].x, t[q + h].x);
                        t[q].y = Add(t[q].y, t[q + h].y);
                    }
                }
                // binary counter over chunks: chunk g is the right sibling at
                // every level b where bit b of g is set
                double2 c = t[0];
#pragma unroll
                for (int b = 0; b < LG; ++b) {
                    if ((g >> b) & 1) {
                        c.x = Add(lvl[b].x, c.x);
                        c.y = Add(lvl[b].y, c.y);
                    } else {
                        lvl[b] = c;
                        break;
                    }
                }
                T = c;  // meaningful after the last chunk (g = G-1: all bits set)
            }
            if (P > 1) {
                xch[grp][wig][lane] = T;
                group_sync<P>(grp);
                if (wig == 0) {
                    double2 W[P];
#pragma unroll
                    for (int w = 0; w < P; ++w) W[w] = xch[grp][w][lane];
#pragma unroll
                    for (int h = P / 2; h >= 1; h /= 2) {
#pragma unroll
                        for (int w = 0; w < h; ++w) {
                            W[w].x = Add(W[w].x, W[w + h].x);
                            W[w].y = Add(W[w].y, W[w + h].y);
                        }
                    }
                    T = W[0];
                }
                group_sync<P>(grp);
            }
            if (wig == 0) {
#pragma unroll
                for (int off = 16; off >= 1; off /= 2) {
                    T.x = Add(T.x, __shfl_down_sync(0xffffffffu, T.x, off));
                    T.y = Add(T.y, __shfl_down_sync(0xffffffffu, T.y, off));
                }
                bsum = Add(T.x, T.y);
            }
        }
        if (wig == 0 && lane == 0) {
            if (A.block_sums) A.block_sums[bidx] = bsum;
            acc_add_shared(sacc, bsum);
        }
    }

    // ---- flush the CTA accumulator, last CTA finalises --------------------
    __syncthreads();
    for (int i = tid; i < PFB_ACC_WORDS; i += blockDim.x)
        if (sacc[i]) atomicAdd(A.acc + i, (unsigned long long)sacc[i]);
    __threadfence();
    __syncthreads();
    if (tid == 0) s_last = (atomicAdd(A.ticket, 1u) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!s_last) return;
    if (A.mode == 2) {  // chained launches: the accumulator and error key stay put
        if (tid == 0) *A.ticket = 0u;
        return;
    }
    __threadfence();
    for (int i = tid; i < PFB_ACC_WORDS; i += blockDim.x) {
        sacc[i] = (long long)atomicExch(A.acc + i, 0ull);
        if (A.mode == 1) A.acc_out[i] = sacc[i];
    }
    __syncthreads();
    if (tid == 0) {
        const unsigned long long key = atomicExch(A.errkey, ~0ull);
        *A.ticket = 0u;
        A.result[1] = (double)sacc[PFB_ACC_FAILS];
        A.result[2] = __longlong_as_double((long long)key);
        if (A.mode == 0) {
            double r;
            const int st = acc_round_dev(sacc, &r);
            A.result[0] = r;
            A.result[3] = (double)st;
        }
    }
}

// ---------------------------------------------------------------------------
// Host-side launch of one instantiation (grid = min(work, resident capacity)).
template <int P, class Ev>
static cudaError_t launch_one(const NllArgs& A, cudaStream_t stream, int sm_count) {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nll_kernel<P, Ev>, kThreads, 0);
        if (occ < 1) occ = 1;
    }
    constexpr int GROUPS = kThreads / (32 * P);
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    int64_t grid = (nitems + GROUPS - 1) / GROUPS;
    const int64_t cap = (int64_t)sm_count * occ;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    nll_kernel<P, Ev><<<(unsigned)grid, kThreads, 0, stream>>>(A);
    return cudaGetLastError();
}

template <class Ev>
static cudaError_t launch_p(const NllArgs& A, cudaStream_t stream, int sm_count) {
    switch (A.warps) {
        case 1:
            return launch_one<1, Ev>(A, stream, sm_count);
        case 2:
            return launch_one<2, Ev>(A, stream, sm_count);
        case 4:
            return launch_one<4, Ev>(A, stream, sm_count);
        default:
            return launch_one<8, Ev>(A, stream, sm_count);
    }
}

}  // namespace pfb
