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

#include <climits>

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
// overflow and density errors.  literal_density returns p = root / norm_root
// (eval_batch(...) / norms[pdf.id], engine.py:181, 265), or NaN with `rank`
// set when a node kernel raises; literal_event adds the p > 0 check and -ln.
// Observable values of one event: from the store columns (event j) or from
// registers (candidates of the toy generator, pfb_pcg.cu).
struct ColLoader {
    int64_t j;
    __device__ __forceinline__ double operator()(const NllArgs& A, int c) const { return A.col[c][j]; }
};
struct ValLoader {
    double v[kMaxCols];
    __device__ __forceinline__ double operator()(const NllArgs&, int c) const { return v[c]; }
};

template <class Ld>
static __device__ __noinline__ double literal_density_t(const NllArgs& A, const Ld ld, int* rank, double* val) {
    double st[kMaxNodes];
    int sid[kMaxNodes];
    int sp = 0;
    for (int o = 0; o < A.nops; ++o) {
        const LitOp& op = A.ops[o];
        double v = 0.0;
        switch (op.kind) {
            case PFB_GAUSSIAN: {
                const double x = ld(A, op.col0);
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
                const double x = ld(A, op.col0);
                v = exp(Mul(A.v[op.voff], x));
                if (!finite(v)) {
                    *rank = op.rank;
                    *val = __longlong_as_double(0x7ff8000000000000ll);
                    return *val;
                }
                break;
            }
            case PFB_POLYNOMIAL: {
                const double x = ld(A, op.col0);
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
                v = dalitz_intensity_literal(A.dal, ld(A, op.col0), ld(A, op.col1));
                break;
            }
            default:
                break;
        }
        st[sp] = v;
        sid[sp] = o;
        ++sp;
    }
    return Div(st[0], A.norm[A.nops - 1]);
}

static __device__ __forceinline__ double literal_density(const NllArgs& A, int64_t j, int* rank, double* val) {
    return literal_density_t(A, ColLoader{j}, rank, val);
}

static __device__ __forceinline__ double literal_event(const NllArgs& A, int64_t j, int* rank, double* val) {
    const double p = literal_density(A, j, rank, val);
    if (*rank >= 0) return p;
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
    static constexpr int MINB = 4;
    __device__ static __forceinline__ double2 eval2(const NllArgs&, const double2 (&x)[1], int64_t,
                                                    long long*, int, bool&, int = 0) {
        return x[0];
    }
};

// Literal interpreter for every event (arbitrary trees).
template <int NC_>
struct EvLiteral {
    static constexpr int NC = NC_;
    static constexpr int U = 1;
    static constexpr int MINB = 1;
    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&)[NC_],
                                                    int64_t local, long long* sacc, int nvalid, bool&, int = 0) {
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
// NL / NT are the leaf and term counts when EXACT (a shape-specialised
// instantiation), else upper bounds checked against the plan at run time.
// KINDS (optional) fixes the leaf kinds at compile time, 2 bits per leaf
// (1 gaussian, 2 exponential, 3 polynomial).
template <int NC_, int NL = kMaxLeaves, int NT = kMaxTerms, bool EXACT = false, int KINDS = 0>
struct EvSop {
    static constexpr int NC = NC_;
    static constexpr int U = 4;
    static constexpr int MINB = EXACT ? 3 : 1;

    __device__ static __forceinline__ constexpr bool has_value_leaf() {
        if (KINDS == 0) return true;
        for (int l = 0; l < NL; ++l)
            if (((KINDS >> (2 * l)) & 3) == PFB_POLYNOMIAL) return true;
        return false;
    }

    __device__ static __forceinline__ double pick(const double2 (&x)[NC_], int col, int which) {
        double r = which ? x[0].y : x[0].x;
#pragma unroll
        for (int c = 1; c < NC_; ++c)
            if (col == c) r = which ? x[c].y : x[c].x;
        return r;
    }

    __device__ static __forceinline__ double one(const NllArgs& A, const double2 (&x)[NC_],
                                                 int which, bool* ok, int m) {
        double u[NL];
        double lv[NL];  // |log| budget of value leaves
        bool good = true;
#pragma unroll
        for (int l = 0; l < NL; ++l) {
            u[l] = 0.0;
            lv[l] = 0.0;
            if (EXACT || l < A.nleaf) {
                const SopLeaf& L = A.leaf[l];
                const double xv = pick(x, L.col, which);
                const int kind = KINDS ? ((KINDS >> (2 * l)) & 3) : L.kind;
                // With a single term the term budget (sum |u| <= thr < 700)
                // already bounds every leaf, so the per-leaf check is dropped.
                constexpr bool kLeafGuard = !(EXACT && NT == 1);
                if (kind == PFB_GAUSSIAN) {
                    const double z = (xv - A.ptv[m][L.voff]) * A.ptv[m][L.voff + 1];
                    u[l] = -0.5 * z * z;
                    if (kLeafGuard) good &= (u[l] >= -600.0) || (u[l] < -746.0);
                } else if (kind == PFB_EXPONENTIAL) {
                    u[l] = A.ptv[m][L.voff] * xv;
                    if (kLeafGuard) good &= (fabs(u[l]) <= 600.0) || (u[l] < -746.0);
                } else if (has_value_leaf()) {  // polynomial (Horner, as polyval)
                    const double* c = A.ptv[m] + L.voff;
                    double acc = c[L.nv - 1];
                    for (int i = 2; i <= L.nv; ++i) acc = fma(acc, xv, c[L.nv - i]);
                    u[l] = acc;
                    const int e = ((__double2hiint(acc) >> 20) & 0x7ff) - 1023;
                    good &= (acc > 0.0) && (e > -900) && (e < 900);
                    lv[l] = fabs((double)e) * 0.6931471805599453 + 1.0;
                }
            }
        }
        double Lm = -1e300, s = 0.0;
        bool live = false;
        double Lt[NT], Vt[NT];
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            Lt[t] = -1e300;
            Vt[t] = 1.0;
            if (EXACT || t < A.nterm) {
                const SopTerm& T = A.term[t];
                const double lc = A.ptv[m][kPtLeafWords + 2 * t];
                double lsum = lc, budget = 0.0, vprod = 1.0;
                // dead: a zero weight (lc = -inf) or a leaf that underflows to
                // exactly 0 in the reference -- the term contributes exactly 0
                bool dead = !(lc > -1e300);
#pragma unroll
                for (int l = 0; l < NL; ++l) {
                    if ((T.emask >> l) & 1u) {
                        lsum += u[l];
                        budget += fabs(u[l]);
                        dead |= (u[l] < -746.0);
                    }
                    if (has_value_leaf() && ((T.vmask >> l) & 1u)) {
                        vprod *= u[l];
                        budget += lv[l];
                    }
                }
                good &= dead || (budget <= A.ptv[m][kPtLeafWords + 2 * t + 1]);
                live |= !dead;
                Lt[t] = dead ? -1e300 : lsum;
                Vt[t] = vprod;
                Lm = fmax(Lm, Lt[t]);
            }
        }
        *ok = good && live;
        if (NT == 1 || (!EXACT && A.nterm == 1)) {
            if (!has_value_leaf()) return -Lt[0];
            return (A.term[0].vmask ? -(Lt[0] + fast_log(Vt[0])) : -Lt[0]);
        }
        if (NT == 2 || (!EXACT && A.nterm == 2)) {
            const double d = Lt[0] - Lt[1];
            const double e = exp(-fabs(d));
            s = d >= 0.0 ? fma(Vt[1], e, Vt[0]) : fma(Vt[0], e, Vt[1]);
            return -(fmax(Lt[0], Lt[1]) + fast_log(s));
        }
#pragma unroll
        for (int t = 0; t < NT; ++t)
            if (EXACT || t < A.nterm) s = fma(Vt[t], exp(Lt[t] - Lm), s);
        return -(Lm + fast_log(s));
    }

    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&x)[NC_],
                                                    int64_t, long long*, int nvalid, bool& bad, int m = 0) {
        bool ok0, ok1;
        double2 t;
        t.x = one(A, x, 0, &ok0, m);
        t.y = one(A, x, 1, &ok1, m);
        bad |= !ok0 || (nvalid > 1 && !ok1);
        return t;
    }
};

// 1/x for normal x: MUFU.RCP64H seed refined by two Newton-Raphson steps.
__device__ __forceinline__ double rcp_nr(double x) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
    double e = fma(-x, r, 1.0);
    r = fma(r, e, r);
    e = fma(-x, r, 1.0);
    return fma(r, e, r);
}

#ifndef PFB_DALR_MINB
#define PFB_DALR_MINB 2  // resident CTAs per SM for EvDalitzR: 128 registers, no spills (A/B: 3% faster than 3)
#endif

// Dalitz coherent sum, recompute path, K terms known at compile time.
// All K Breit-Wigner denominators and the Zemach 1/s_pair share ONE
// reciprocal through Montgomery batch inversion.  SIG >= 0 fixes each term's
// (pair, spin) at compile time -- 3 bits per term: pair code (0: 12, 1: 13,
// 2: 23) and the spin bit -- and, in bits 12..14, which Zemach 1/s_pair
// factors the batch inversion carries (need12/13/23: a P-wave on that pair
// with a nonzero mass-difference coefficient), removing the per-term selects
// and branches.
__host__ __device__ constexpr int dal_pair_code(int pair) { return pair == 12 ? 0 : (pair == 13 ? 1 : 2); }

template <int K, int SIG = -1>
struct EvDalitz {
    static constexpr int NC = 2;
    static constexpr int U = 2;
    static constexpr int MINB = 3;  // 24 warps/SM (measured: 5% faster than 16 warps at 128 regs)

    // p = |sum_k c_k BW_k Z_k|^2 / norm; *ok = the batch inversion stayed in range
    __device__ static __forceinline__ double prob(const NllArgs& A, double s12, double s13,
                                                  bool* ok) {
        const DalDesc& D = A.dal;
        constexpr int KK = (K > 0 ? K : 1);
        const double s23 = (D.mss - s12) - s13;
        int pc[KK], sp[KK];
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            pc[k] = SIG >= 0 ? ((SIG >> (3 * k)) & 3) : dal_pair_code(D.t[k].pair);
            sp[k] = SIG >= 0 ? ((SIG >> (3 * k + 2)) & 1) : D.t[k].spin;
        }
        double sv[KK], d[KK], P[KK + 3];
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            const DalTerm& T = D.t[k];
            sv[k] = pc[k] == 0 ? s12 : (pc[k] == 1 ? s13 : s23);
            const double a = T.m2 - sv[k];
            d[k] = fma(a, a, T.mg2);
        }
        // prefix products over the used denominators
        P[0] = d[0];
#pragma unroll
        for (int k = 1; k < KK; ++k) P[k] = P[k - 1] * d[k];
        const bool n12 = SIG >= 0 ? ((SIG >> 12) & 1) : D.need12;
        const bool n13 = SIG >= 0 ? ((SIG >> 13) & 1) : D.need13;
        const bool n23 = SIG >= 0 ? ((SIG >> 14) & 1) : D.need23;
        double last = P[KK - 1];
        if (n12) last = last * s12;
        P[KK] = last;
        if (n13) last = last * s13;
        P[KK + 1] = last;
        if (n23) last = last * s23;
        P[KK + 2] = last;
        // one reciprocal for everything: hardware seed + two Newton steps
        // (<= 2 ulp; `last` is certified normal below, so no special cases)
        double inv = rcp_nr(last);
        bool good = (last > 1e-280) && (last < 1e280);
        double r23 = 0.0, r13 = 0.0, r12 = 0.0;
        if (n23) {
            r23 = inv * P[KK + 1];
            inv = inv * s23;
        }
        if (n13) {
            r13 = inv * P[KK];
            inv = inv * s13;
        }
        if (n12) {
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
        // c_k BW_k Z_k = w_k [(alpha_k - cre_k s) + i (beta_k - cim_k s)],
        // w_k = Z_k / |m_k^2 - s - i m_k G_k|^2, alpha/beta per-call constants
        const double d12 = s13 - s23, d13 = s12 - s23, d23 = s12 - s13;
        double tr = 0.0, ti = 0.0;
#pragma unroll
        for (int k = 0; k < KK; ++k) {
            const DalTerm& T = D.t[k];
            double w = r[k];
            if (sp[k] == 1) {
                double z;
                // a Zemach factor with a zero mass-difference coefficient
                // (need flag clear) is exactly d_pair
                if (pc[k] == 0)
                    z = n12 ? fma(D.zc12, r12, d12) : d12;
                else if (pc[k] == 1)
                    z = n13 ? fma(D.zc13, r13, d13) : d13;
                else
                    z = n23 ? fma(D.zc23, r23, d23) : d23;
                w *= z;
            }
            tr = fma(w, fma(-T.cre, sv[k], T.alpha), tr);
            ti = fma(w, fma(-T.cim, sv[k], T.beta), ti);
        }
        const double I = fma(tr, tr, ti * ti);
        *ok = good;
        return I * A.inv_norm;
    }

    __device__ static __forceinline__ double one(const NllArgs& A, double s12, double s13,
                                                 bool* ok) {
        const double p = prob(A, s12, s13, ok);
        *ok = *ok && (p > 1e-300) && (p < 1e300);
        return -fast_log(p);
    }

    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&x)[2],
                                                    int64_t, long long*, int nvalid, bool& bad, int = 0) {
        bool ok0, ok1;
        double2 t;
        t.x = one(A, x[0].x, x[1].x, &ok0);
        t.y = one(A, x[0].y, x[1].y, &ok1);
        bad |= !ok0 || (nvalid > 1 && !ok1);
        return t;
    }

    // product-mode interface (pfb_nll_prod.cuh)
    __device__ static __forceinline__ double2 prob2(const NllArgs& A, const double2 (&x)[2], bool& okx,
                                                    bool& oky, const double*, double2&) {
        double2 p;
        p.x = prob(A, x[0].x, x[1].x, &okx);
        p.y = prob(A, x[0].y, x[1].y, &oky);
        return p;
    }
};

// Dalitz coherent sum as a ratio, K = 4 terms with compile-time structure SIG
// (same bit layout as EvDalitz), for the product kernels.  With
//   BW_k = (a_k + i mG_k) / d_k,  a_k = m_k^2 - s,  d_k = a_k^2 + (mG_k)^2,
//   Z_k = d_pair + zc_pair / s_pair  (P-wave; 1 for S-wave),
// everything is brought over the common denominator D' = prod_k d_k * sigma,
// sigma = product of the s_pair the Zemach factors divide by:
//   sum_k c_k BW_k Z_k = N / D',  N = sum_k E_k [(alpha_k - cre_k s) + i (beta_k - cim_k s)],
//   E_k = prod_{j != k} d_j * Z_k * sigma,
// so p = |N|^2 / norm / D'^2 needs no reciprocal at all: the kernel multiplies
// numerators and denominators into separate unit products (D' itself; the
// square is taken on the unit's logarithm), and 1/norm rides in the
// coefficients (sqrt(1/norm) each).  ~47 FP64 operations per event against
// ~57 plus a reciprocal for EvDalitz.
template <int K_, int SIG = -1, bool PTS = false>
struct EvDalitzR {
    // PTS: batched parameter points -- the four scaled coefficients of term k
    // for point m in A.ptv[m][4k .. 4k+3] (the shapes are shared)
    static constexpr bool POINTS = PTS;
    static constexpr int NC = 2;
    static constexpr int U = 2;
    static constexpr int MINB = PFB_DALR_MINB;
    static constexpr bool RATIO = true;
    static constexpr int RATIO_POW = 2;  // p = num / den^2
    static constexpr int K = K_;
    // SIG >= 0: (pair, spin) per term and the needed 1/s_pair fixed at compile
    // time (C3/C4); SIG < 0: the same algebra with the structure read from the
    // term table at run time (any model with K terms)
    static constexpr bool RT = SIG < 0;
    static_assert(K >= 2 && K <= 6, "ratio form instantiated for 2..6 terms");

    __device__ static __forceinline__ int pcode(const DalDesc& D, int k) {
        if constexpr (RT) return dal_pair_code(D.t[k].pair);
        else return (SIG >> (3 * k)) & 3;
    }
    __device__ static __forceinline__ int spin(const DalDesc& D, int k) {
        if constexpr (RT) return D.t[k].spin;
        else return (SIG >> (3 * k + 2)) & 1;
    }
    __device__ static __forceinline__ bool need(const DalDesc& D, int p) {
        if constexpr (RT) return p == 0 ? D.need12 != 0 : (p == 1 ? D.need13 != 0 : D.need23 != 0);
        else return (SIG >> (12 + p)) & 1;
    }
    __device__ static __forceinline__ double pick(int p, double a, double b, double c) {
        return p == 0 ? a : (p == 1 ? b : c);
    }

    __device__ static __forceinline__ void one(const NllArgs& A, double s12, double s13, double& num,
                                               double& den, int m = 0) {
        const DalDesc& D = A.dal;
        const double s23 = (D.mss - s12) - s13;
        const double dd12 = s13 - s23, dd13 = s12 - s23, dd23 = s12 - s13;  // Zemach differences
        double d[K], sv[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            sv[k] = pick(pcode(D, k), s12, s13, s23);
            const double a = D.t[k].m2 - sv[k];
            d[k] = fma(a, a, D.t[k].mg2);
        }
        // exclusive products prod_{j != k} d_j (prefix x suffix)
        double pre[K], suf[K];
        pre[0] = 1.0;
#pragma unroll
        for (int k = 1; k < K; ++k) pre[k] = k == 1 ? d[0] : pre[k - 1] * d[k - 1];
        suf[K - 1] = 1.0;
#pragma unroll
        for (int k = K - 2; k >= 0; --k) suf[k] = k == K - 2 ? d[K - 1] : suf[k + 1] * d[k + 1];
        double ex[K];
#pragma unroll
        for (int k = 0; k < K; ++k) ex[k] = k == 0 ? suf[0] : (k == K - 1 ? pre[K - 1] : pre[k] * suf[k]);
        // sigma = product of the needed s_pair
        double sig = 1.0;
        bool any = false;
#pragma unroll
        for (int p = 0; p < 3; ++p)
            if (need(D, p)) {
                const double sp = pick(p, s12, s13, s23);
                sig = any ? sig * sp : sp;
                any = true;
            }
        double tr = 0.0, ti = 0.0;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const DalTerm& T = D.t[k];
            double F;
            if (spin(D, k) == 0) {
                F = sig;
            } else {
                const int p = pcode(D, k);
                const double ddp = pick(p, dd12, dd13, dd23);
                if (need(D, p)) {
                    // Z sigma = (d_pair s_pair + zc) * prod of the other needed s
                    double others = 1.0;
                    bool anyo = false;
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        if (need(D, q) && q != p) {
                            const double sq = pick(q, s12, s13, s23);
                            others = anyo ? others * sq : sq;
                            anyo = true;
                        }
                    const double zp = fma(ddp, pick(p, s12, s13, s23), pick(p, D.zc12, D.zc13, D.zc23));
                    F = anyo ? zp * others : zp;
                } else {
                    F = any ? ddp * sig : ddp;
                }
            }
            const double E = ex[k] * F;
            const double scre = PTS ? A.ptv[m][4 * k] : T.scre, scim = PTS ? A.ptv[m][4 * k + 1] : T.scim;
            const double salpha = PTS ? A.ptv[m][4 * k + 2] : T.salpha, sbeta = PTS ? A.ptv[m][4 * k + 3] : T.sbeta;
            tr = fma(E, fma(-scre, sv[k], salpha), tr);  // coefficients carry sqrt(1/norm)
            ti = fma(E, fma(-scim, sv[k], sbeta), ti);
        }
        num = fma(tr, tr, ti * ti);
        den = any ? (pre[K - 1] * d[K - 1]) * sig : pre[K - 1] * d[K - 1];  // D'; the kernel squares at the unit end
    }

    __device__ static __forceinline__ double2 prob2r(const NllArgs& A, const double2 (&x)[2], bool& okx,
                                                     bool& oky, double2& den, int m = 0) {
        double2 q;
        one(A, x[0].x, x[1].x, q.x, den.x, m);
        one(A, x[0].y, x[1].y, q.y, den.y, m);
        okx = oky = true;  // certified by the kernel's range checks on q and den
        return q;
    }
};

// Dalitz with the lineshape cache: amplitudes of cached terms are read from
// HBM (K rows of double2 per event); the remaining terms are recomputed.
struct EvDalitzCached {
    static constexpr int NC = 2;
    static constexpr int U = 2;
    static constexpr int MINB = 2;

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
        return -fast_log(p);
    }

    __device__ static __forceinline__ double2 eval2(const NllArgs& A, const double2 (&x)[2],
                                                    int64_t local, long long*, int nvalid, bool& bad, int = 0) {
        bool ok0, ok1;
        double2 t;
        t.x = one(A, x[0].x, x[1].x, local, &ok0);
        t.y = one(A, x[0].y, x[1].y, local + 1, &ok1);
        bad |= !ok0 || (nvalid > 1 && !ok1);
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
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = k < f.len ? a[f.start + k] : 0.0;
            double s = v[0];
#pragma unroll
            for (int k = 1; k < 8; ++k)
                if (k < f.len) s = Add(s, v[k]);
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

// Named barrier of one warp group.  Immediate barrier ids, so ptxas reserves
// only GROUPS+1 of the SM's hardware barriers (a register id reserves all 16
// and caps the CTAs per SM).
template <int P>
__device__ __forceinline__ void group_sync(int grp) {
    constexpr int n = P * 32;
    if (P == 1) {
        __syncwarp();
    } else if (P == 8) {
        asm volatile("bar.sync 1, %0;" ::"n"(n) : "memory");
    } else if (P == 4) {
        if (grp == 0)
            asm volatile("bar.sync 1, %0;" ::"n"(n) : "memory");
        else
            asm volatile("bar.sync 2, %0;" ::"n"(n) : "memory");
    } else {
        switch (grp) {
            case 0: asm volatile("bar.sync 1, %0;" ::"n"(n) : "memory"); break;
            case 1: asm volatile("bar.sync 2, %0;" ::"n"(n) : "memory"); break;
            case 2: asm volatile("bar.sync 3, %0;" ::"n"(n) : "memory"); break;
            default: asm volatile("bar.sync 4, %0;" ::"n"(n) : "memory"); break;
        }
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

// ---------------------------------------------------------------------------
// Kernel modes.  The fast kernel never takes the literal path: a block that
// contains an event its evaluator cannot certify is left out of the
// accumulator and listed; the fix-up launch (LIST = true, literal evaluator)
// recomputes exactly those blocks -- reporting the reference's errors -- and
// adds them.  Integer accumulation makes "fast blocks + fixed blocks" exact.
enum KernelMode : int32_t {
    MODE_EXPORT = 0,      // last CTA: out = acc, reset; counters -> result
    MODE_ADD_EXPORT = 1,  // last CTA: out += acc, reset (fix-up after a fast launch)
    MODE_ACCUM = 2        // chained launches: keep accumulating
};

// Last-CTA election: one acq_rel atomic on the ticket replaces two
// device-wide SC fences (__threadfence = MEMBAR.SC.GPU, microseconds on the
// two-die B200): the release is cumulative over this CTA's accumulator
// atomics (ordered before it by the CTA barrier), and the last CTA's acquire
// makes every CTA's atomics visible to it.
__device__ __forceinline__ unsigned int ticket_acq_rel(unsigned int* t) {
    unsigned int old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(t) : "memory");
    return old;
}

// Fused exchange (A.peer_world > 0, single point, export mode), run by every
// thread of the CTA that finishes the launch, after the ticket: thread t
// stores word t of this rank's 72 limbs (t = 72: a status word, deferred
// blocks or an error on this rank) as a flag-in-line 16-byte line {lo, seq,
// hi, seq} into line [seq & 1][rank][t] of every rank's mailbox (NVLink P2P
// stores), then polls line [seq & 1][q][t] of its own mailbox for every rank
// q until both halves carry seq (bounded) and sums in rank order -- integer
// limbs, so every rank exports the single-GPU accumulator bit for bit, with no
// separate collective launch and no system-scope fence on the critical path.
// result_i[2] = number of ranks that need the slow path (deferred blocks or
// an error: the host then redoes the call unfused), result_i[3] = 1 on a
// peer timeout.  Parity alternation: a rank can be at most one call ahead
// (it cannot pass call s+1's wait before every rank has posted s+1, i.e.
// finished reading call s), so it never overwrites a slot still being read.
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#ifdef PFB_TRACE
// Per-CTA timeline of the TMA unit kernel (debug builds only): %globaltimer ns
// at [0] entry, [1] first copy issued, [2] first stage ready (team 0),
// [3] team 0 done, [4] team 1 done, [5] finish entry, [6] ticket taken,
// [7] export done (last CTA only).
__device__ unsigned long long g_trace[1024][16];  // [8..9] ns waited for data per team, [10..11] blocks per team, [12..15] fused-exchange phases (last CTA)
#define PFB_T(slot) g_trace[blockIdx.x][slot] = gtimer()
#else
#define PFB_T(slot) ((void)0)
#endif

#ifndef PFB_PEER_ON
#define PFB_PEER_ON 1
#endif
__device__ __forceinline__ void peer_finish(const NllArgs& A) {
    __shared__ long long s_fx;
    __shared__ unsigned long long s_ek;
    __shared__ int s_timeout;
    const int t = threadIdx.x;
    if (t == 0) s_timeout = 0;
    long long v = 0;
    if (t < PFB_ACC_WORDS) v = (long long)atomicExch(A.acc + t, 0ull);
    if (t == PFB_ACC_WORDS) {
        const long long fx = (long long)atomicExch(A.fix_counter, 0ull);
        const unsigned long long ek = atomicExch(A.errkey, ~0ull);
        s_fx = fx;
        s_ek = ek;
        v = (fx != 0 || ek != ~0ull) ? 1 : 0;
    }
#ifdef PFB_TRACE
    __syncthreads();
    if (t == 0) PFB_T(12);
#endif
    const int par = (int)(A.peer_seq & 1ull);
    const unsigned seq = (unsigned)A.peer_seq;
    long long sum = 0;
    if (t <= PFB_ACC_WORDS) {
        // word t of this rank's limbs (+ status word) to every rank's mailbox
        for (int q = 0; q < A.peer_world; ++q) st_line(peer_line(A.peer_mbox[q], par, A.peer_rank, t), v, seq);
        // word t of every rank, in rank order (integer: exact, bitwise the
        // single-GPU accumulator on every rank); bounded wait per line
        const long long t0 = clock64();
        for (int q = 0; q < A.peer_world; ++q) {
            const ulonglong2* line = peer_line(A.peer_mbox[A.peer_rank], par, q, t);
            long long w;
            while (!ld_line(line, seq, &w)) {
                if (clock64() - t0 > A.peer_timeout) {
                    atomicExch(&s_timeout, 1);
                    w = 0;
                    break;
                }
                __nanosleep(32);
            }
            sum += w;
        }
    }
    __syncthreads();
#ifdef PFB_TRACE
    if (t == 0) PFB_T(14);
#endif
    if (t == 0) {
        A.result_i[0] = s_fx;
        A.result_i[1] = (long long)s_ek;
        A.result_i[3] = s_timeout ? 1 : 0;
    }
    if (s_timeout) return;
    if (t < PFB_ACC_WORDS)
        A.acc_out[t] = sum;
    else if (t == PFB_ACC_WORDS)
        A.result_i[2] = sum;
#ifdef PFB_TRACE
    __syncthreads();
    if (t == 0) PFB_T(15);
#endif
}

// Flush the CTA accumulator; the last CTA to finish exports (per A.mode) and
// resets the launch-scoped counters.  Shared by every fast kernel.
// Completion post for the polling host (NllArgs::seq): after every export
// store of the last CTA, one system-scope fence and the sequence number --
// a host that sees seq in result_i[4] reads a complete result block.
__device__ __forceinline__ void post_seq(const NllArgs& A) {
    if (A.seq <= 0) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        *reinterpret_cast<volatile long long*>(A.result_i + 4) = A.seq;
    }
}

template <bool LIST>
__device__ __forceinline__ void finish_launch(const NllArgs& A, long long* sacc, unsigned int* s_last) {
    __syncthreads();
    for (int i = threadIdx.x; i < PFB_ACC_WORDS; i += blockDim.x)
        if (sacc[i]) atomicAdd(A.acc + i, (unsigned long long)sacc[i]);
    __syncthreads();
    if (threadIdx.x == 0) *s_last = (ticket_acq_rel(A.ticket) == gridDim.x - 1) ? 1u : 0u;
    __syncthreads();
    if (!*s_last) return;
    // the last CTA: independent global round trips issued by different
    // threads, so the export costs one atomic latency, not four in a row
    const int t = threadIdx.x, nt = blockDim.x;
    if (t == nt - 1) {
        *A.work_counter = 0ull;
        *A.ticket = 0u;
    }
    if (A.mode == MODE_ACCUM) return;
    if (!LIST && PFB_PEER_ON && A.peer_world > 0 && A.mode == MODE_EXPORT) {
        peer_finish(A);
        return;
    }
    if (t == nt - 2 && !LIST)  // hand the deferred-block count to the fix-up launch
        A.result_i[0] = (long long)atomicExch(A.fix_counter, 0ull);
    if (t == nt - 3) A.result_i[1] = (long long)atomicExch(A.errkey, ~0ull);
    if (A.xkey && t == nt - 4) A.result_i[2] = (long long)atomicExch(A.xkey, ~0ull);
    for (int i = t; i < PFB_ACC_WORDS; i += nt) {
        const long long v = (long long)atomicExch(A.acc + i, 0ull);
        if (A.mode == MODE_EXPORT)
            A.acc_out[i] = v;
        else
            A.acc_out[i] += v;
    }
    post_seq(A);
}

template <int P, class Ev, bool LIST>
__global__ void __launch_bounds__(kThreads, Ev::MINB) nll_kernel(const __grid_constant__ NllArgs A) {
    constexpr int NC = Ev::NC;
    constexpr int GROUPS = kThreads / (32 * P);
    constexpr int KPT = 64 / P;                       // double2 slots per thread per block
    constexpr int W = Ev::U < KPT ? Ev::U : KPT;      // slot loads kept in flight
    constexpr int LK = Log2<KPT>::value;

    __shared__ double2 xch[GROUPS][P][32];
    __shared__ int xbad[GROUPS][P];
    __shared__ long long s_item[GROUPS];
    __shared__ long long sacc[PFB_ACC_WORDS];
    __shared__ unsigned int s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int grp = warp / P;
    const int wig = warp % P;
    for (int i = tid; i < PFB_ACC_WORDS; i += blockDim.x) sacc[i] = 0;
    __syncthreads();

    const int64_t nitems = LIST ? (int64_t)(*A.fix_count) : A.nfull + (A.tail ? 1 : 0);
    // Dynamic item scheduling: groups pull the next block from a global
    // counter, so fast SMs take more blocks and no SM idles in a last round.
    // Item 0 is the ragged tail (if any), pulled first.
    for (;;) {
        if (wig == 0 && lane == 0) s_item[grp] = (long long)atomicAdd(A.work_counter, 1ull);
        group_sync<P>(grp);
        const int64_t it = s_item[grp];
        group_sync<P>(grp);
        if (it >= nitems) break;
        double bsum = 0.0;
        int64_t bidx;
        bool is_tail;
        if (LIST) {
            const int64_t entry = A.fix_list[it];
            if ((int)(entry % kMaxPts) != A.fix_point) continue;  // another point's block
            bidx = entry / kMaxPts - A.block_base;
            is_tail = A.tail && bidx == A.nfull;
        } else {
            is_tail = A.tail && it == 0;
            bidx = is_tail ? A.nfull : it - (A.tail ? 1 : 0);
        }
        bool bad = false;
        if (is_tail) {
            // ---- ragged tail block: terms to scratch, then split recursion
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
                const double2 t = Ev::eval2(A, x, lbase + e, sacc, pair ? 2 : 1, bad);
                A.tail_scratch[e] = t.x;
                if (pair) A.tail_scratch[e + 1] = t.y;
            }
            const unsigned anybad = __any_sync(0xffffffffu, bad);
            if (lane == 0) xbad[grp][wig] = anybad ? 1 : 0;
            group_sync<P>(grp);
            bad = false;
#pragma unroll
            for (int w = 0; w < P; ++w) bad |= xbad[grp][w] != 0;
            if (wig == 0 && !bad) bsum = pairwise_warp(A.tail_scratch, n, lane);
            group_sync<P>(grp);
        } else {
            // ---- full block, reference half-folding tree
            const int64_t lbase = bidx * (int64_t)kBlock;
            const int64_t lthr = lbase + 2 * lane + 64 * wig;
            // Sliding window: slots are visited in the streaming order
            // i = 0..KPT-1 (slot k = bitrev(i)), W loads stay in flight, and
            // a binary counter over i reproduces the half-folding tree (the
            // tree over i pairs adjacent i first).  One eval2 per kernel body
            // keeps the code inside the instruction cache.
            double2 win[W][NC];
#pragma unroll
            for (int q = 0; q < W; ++q) {
                const int k = LK ? (int)(__brev((unsigned)q) >> (32 - LK)) : 0;
#pragma unroll
                for (int c = 0; c < NC; ++c) win[q][c] = ld2(A.col[c] + A.begin + lthr + 64 * P * k);
            }
            double2 lvl[LK > 0 ? LK : 1];
            double2 T = make_double2(0.0, 0.0);
#pragma unroll 1
            for (int i = 0; i < KPT; ++i) {
                const int k = LK ? (int)(__brev((unsigned)i) >> (32 - LK)) : 0;
                double2 cur[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) cur[c] = win[0][c];
#pragma unroll
                for (int q = 0; q + 1 < W; ++q)
#pragma unroll
                    for (int c = 0; c < NC; ++c) win[q][c] = win[q + 1][c];
                if (i + W < KPT) {
                    const int kn = (int)(__brev((unsigned)(i + W)) >> (32 - LK));
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        win[W - 1][c] = ld2(A.col[c] + A.begin + lthr + 64 * P * kn);
                }
                double2 v = Ev::eval2(A, cur, lthr + 64 * P * (int64_t)k, sacc, 2, bad);
#pragma unroll
                for (int b = 0; b < LK; ++b) {
                    if ((i >> b) & 1) {
                        v.x = Add(lvl[b].x, v.x);
                        v.y = Add(lvl[b].y, v.y);
                    } else {
                        lvl[b] = v;
                        break;
                    }
                }
                T = v;  // the root after the last slot (i = KPT-1: all bits set)
            }
            const unsigned anybad = __any_sync(0xffffffffu, bad);
            if (P > 1) {
                xch[grp][wig][lane] = T;
                if (lane == 0) xbad[grp][wig] = anybad ? 1 : 0;
                group_sync<P>(grp);
                bad = false;
#pragma unroll
                for (int w = 0; w < P; ++w) bad |= xbad[grp][w] != 0;
                if (wig == 0 && !bad) {
                    double2 Wv[P];
#pragma unroll
                    for (int w = 0; w < P; ++w) Wv[w] = xch[grp][w][lane];
#pragma unroll
                    for (int h = P / 2; h >= 1; h /= 2) {
#pragma unroll
                        for (int w = 0; w < h; ++w) {
                            Wv[w].x = Add(Wv[w].x, Wv[w + h].x);
                            Wv[w].y = Add(Wv[w].y, Wv[w + h].y);
                        }
                    }
                    T = Wv[0];
                }
                group_sync<P>(grp);
            } else {
                bad = anybad != 0;
            }
            if (wig == 0 && !bad) {
#pragma unroll
                for (int off = 16; off >= 1; off /= 2) {
                    T.x = Add(T.x, __shfl_down_sync(0xffffffffu, T.x, off));
                    T.y = Add(T.y, __shfl_down_sync(0xffffffffu, T.y, off));
                }
                bsum = Add(T.x, T.y);
            }
        }
        if (wig == 0 && lane == 0) {
            if (bad) {  // defer the whole block to the exact fix-up launch
                const unsigned long long slot = atomicAdd(A.fix_counter, 1ull);
                A.fix_list[slot] = (A.block_base + bidx) * kMaxPts + A.fix_point;
            } else {
                if (A.block_sums) A.block_sums[A.block_base + bidx] = bsum;
                acc_add_shared(sacc, bsum);
            }
        }
    }

    finish_launch<LIST>(A, sacc, &s_last);
}

// ---------------------------------------------------------------------------
// Host-side launch of one instantiation.  Grid: one resident wave (workers
// pull blocks from the device counter).
template <int P, class Ev, bool LIST>
static cudaError_t launch_one(const NllArgs& A, cudaStream_t stream, int sm_count) {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nll_kernel<P, Ev, LIST>, kThreads, 0);
        if (occ < 1) occ = 1;
    }
    constexpr int GROUPS = kThreads / (32 * P);
    int64_t grid;
    const int64_t cap = (int64_t)sm_count * occ;
    if (LIST) {
        grid = sm_count;  // item count lives on the device
    } else {
        const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
        grid = (nitems + GROUPS - 1) / GROUPS;
        if (grid > cap) grid = cap;  // resident workers pull items dynamically
    }
    if (grid < 1) grid = 1;
    nll_kernel<P, Ev, LIST><<<(unsigned)grid, kThreads, 0, stream>>>(A);
    return cudaGetLastError();
}

template <class Ev, bool LIST = false>
static cudaError_t launch_p(const NllArgs& A, cudaStream_t stream, int sm_count) {
    switch (A.warps) {
        case 1:
            return launch_one<1, Ev, LIST>(A, stream, sm_count);
        case 2:
            return launch_one<2, Ev, LIST>(A, stream, sm_count);
        case 4:
            return launch_one<4, Ev, LIST>(A, stream, sm_count);
        default:
            return launch_one<8, Ev, LIST>(A, stream, sm_count);
    }
}

}  // namespace pfb
