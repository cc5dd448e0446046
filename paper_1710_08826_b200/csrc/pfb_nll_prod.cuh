// pfb_nll_prod.cuh -- product-mode NLL kernel for transcendental-bound models.
//
// -sum_i ln p_i equals -ln prod_i p_i.  For models whose per-event density
// costs exponentials anyway (SumPdf C1/C5, Dalitz C3/C4) the kernel evaluates
// p_i in the linear domain -- the reference's own formula, pdf.py:205-227 /
// dalitz.py:217-230 -- and multiplies: one log per 16 events instead of one
// per event.  An evaluator may factor p_i = exp(l_i) q_i; then q_i enters the
// product and l_i a plain sum (C1: l = alpha x, one exponential per event).
//
// Canonical structure of one 4096-event block (independent of warps per
// block P, of grid size and of GPU count, so every invariance the reference
// tests -- serial == pool == shards -- holds bit for bit):
//   row r = e / 64 (64 rows), column = e % 64, thread column = 2*lane + {0,1};
//   unit u = rows [8u, 8u+8) x one lane's 2 columns = 16 events;
//   unit value  v(u, lane) = -(ln m + L + ex ln 2)  with  m 2^ex = prod q
//   and L = sum l (rows in ascending order, x then y; m renormalised to
//   [1, 2) after every row);
//   block value = lane tree (shuffle-down 16..1) of the unit tree
//   ((v0+v1)+(v2+v3))+((v4+v5)+(v6+v7)).
// A ragged tail block uses the same structure with q = 1 for absent events.
//
// Guard: an event is certified when its q lies in [2^-500, 2^500] (so every
// partial product is a normal double) and the evaluator's own conditions
// hold (p far from 0 and inf, no out-of-range intermediate).  A block with
// any uncertified event is deferred to the exact fix-up launch (literal
// reference arithmetic, reference errors) exactly like the log-domain kernel.
//
// Accuracy: the product of 16 correctly-rounded factors has relative error
// <= 16 u, i.e. an absolute error <= 4e-15 in each unit's -ln -- orders of
// magnitude inside the 1e-10 relative NLL tolerance.
#pragma once
#include "pfb_nll_tma.cuh"




namespace pfb {


// q in [2^-500, 2^500]: biased exponent in [523, 1523]; 0, subnormal, negative,
// inf and NaN all fail.
#ifndef PFB_UNIT_MINMAX
#define PFB_UNIT_MINMAX 1
#endif
// Certified factor range with unit-level checks: every q (and r) within
// 2^+-kSpanM, so the unit running products stay normal with a renormalisation
// every second row (four factors of at most 2^+-250 each on a mantissa in
// [1, 2)); the density p = q / r^POW of every event then lies within
// 2^+-(250 * (1 + POW)) -- a normal double, as in the reference.
constexpr int kSpanM = 250;

__device__ __forceinline__ bool p_in_range(double p) {
    const int hi = __double2hiint(p);
    return (unsigned)((hi >> 20) - 523) <= 1000u;
}

// m * 2^ex  ->  m in [1, 2), exponent moved into ex (m positive normal).
__device__ __forceinline__ void renorm(double& m, int& ex) {
    const int hi = __double2hiint(m);
    ex += (hi >> 20) - 1023;
    m = __hiloint2double((hi & 0x000fffff) | 0x3ff00000, __double2loint(m));
}

// 2^(j/256), j = 0..255, correctly rounded (Python decimal, 60 digits).  An
// evaluator's per-launch table (c * 2^(j/256), 256 doubles, 2 KB) lives in
// shared memory: one LDS.64 per event, no multiply by the table value in the
// per-event chain.
constexpr int kTabN = 256;
__constant__ static double kExp2Tab256[kTabN] = {
    0x1.0000000000000p+0, 0x1.00b1afa5abcbfp+0, 0x1.0163da9fb3335p+0, 0x1.02168143b0281p+0,
    0x1.02c9a3e778061p+0, 0x1.037d42e11bbccp+0, 0x1.04315e86e7f85p+0, 0x1.04e5f72f654b1p+0,
    0x1.059b0d3158574p+0, 0x1.0650a0e3c1f89p+0, 0x1.0706b29ddf6dep+0, 0x1.07bd42b72a836p+0,
    0x1.0874518759bc8p+0, 0x1.092bdf66607e0p+0, 0x1.09e3ecac6f383p+0, 0x1.0a9c79b1f3919p+0,
    0x1.0b5586cf9890fp+0, 0x1.0c0f145e46c85p+0, 0x1.0cc922b7247f7p+0, 0x1.0d83b23395decp+0,
    0x1.0e3ec32d3d1a2p+0, 0x1.0efa55fdfa9c5p+0, 0x1.0fb66affed31bp+0, 0x1.1073028d7233ep+0,
    0x1.11301d0125b51p+0, 0x1.11edbab5e2ab6p+0, 0x1.12abdc06c31ccp+0, 0x1.136a814f204abp+0,
    0x1.1429aaea92de0p+0, 0x1.14e95934f312ep+0, 0x1.15a98c8a58e51p+0, 0x1.166a45471c3c2p+0,
    0x1.172b83c7d517bp+0, 0x1.17ed48695bbc0p+0, 0x1.18af9388c8deap+0, 0x1.1972658375d2fp+0,
    0x1.1a35beb6fcb75p+0, 0x1.1af99f8138a1cp+0, 0x1.1bbe084045cd4p+0, 0x1.1c82f95281c6bp+0,
    0x1.1d4873168b9aap+0, 0x1.1e0e75eb44027p+0, 0x1.1ed5022fcd91dp+0, 0x1.1f9c18438ce4dp+0,
    0x1.2063b88628cd6p+0, 0x1.212be3578a819p+0, 0x1.21f49917ddc96p+0, 0x1.22bdda27912d1p+0,
    0x1.2387a6e756238p+0, 0x1.2451ffb82140ap+0, 0x1.251ce4fb2a63fp+0, 0x1.25e85711ece75p+0,
    0x1.26b4565e27cddp+0, 0x1.2780e341ddf29p+0, 0x1.284dfe1f56381p+0, 0x1.291ba7591bb70p+0,
    0x1.29e9df51fdee1p+0, 0x1.2ab8a66d10f13p+0, 0x1.2b87fd0dad990p+0, 0x1.2c57e39771b2fp+0,
    0x1.2d285a6e4030bp+0, 0x1.2df961f641589p+0, 0x1.2ecafa93e2f56p+0, 0x1.2f9d24abd886bp+0,
    0x1.306fe0a31b715p+0, 0x1.31432edeeb2fdp+0, 0x1.32170fc4cd831p+0, 0x1.32eb83ba8ea32p+0,
    0x1.33c08b26416ffp+0, 0x1.3496266e3fa2dp+0, 0x1.356c55f929ff1p+0, 0x1.36431a2de883bp+0,
    0x1.371a7373aa9cbp+0, 0x1.37f26231e754ap+0, 0x1.38cae6d05d866p+0, 0x1.39a401b7140efp+0,
    0x1.3a7db34e59ff7p+0, 0x1.3b57fbfec6cf4p+0, 0x1.3c32dc313a8e5p+0, 0x1.3d0e544ede173p+0,
    0x1.3dea64c123422p+0, 0x1.3ec70df1c5175p+0, 0x1.3fa4504ac801cp+0, 0x1.40822c367a024p+0,
    0x1.4160a21f72e2ap+0, 0x1.423fb2709468ap+0, 0x1.431f5d950a897p+0, 0x1.43ffa3f84b9d4p+0,
    0x1.44e086061892dp+0, 0x1.45c2042a7d232p+0, 0x1.46a41ed1d0057p+0, 0x1.4786d668b3237p+0,
    0x1.486a2b5c13cd0p+0, 0x1.494e1e192aed2p+0, 0x1.4a32af0d7d3dep+0, 0x1.4b17dea6db7d7p+0,
    0x1.4bfdad5362a27p+0, 0x1.4ce41b817c114p+0, 0x1.4dcb299fddd0dp+0, 0x1.4eb2d81d8abffp+0,
    0x1.4f9b2769d2ca7p+0, 0x1.508417f4531eep+0, 0x1.516daa2cf6642p+0, 0x1.5257de83f4eefp+0,
    0x1.5342b569d4f82p+0, 0x1.542e2f4f6ad27p+0, 0x1.551a4ca5d920fp+0, 0x1.56070dde910d2p+0,
    0x1.56f4736b527dap+0, 0x1.57e27dbe2c4cfp+0, 0x1.58d12d497c7fdp+0, 0x1.59c0827ff07ccp+0,
    0x1.5ab07dd485429p+0, 0x1.5ba11fba87a03p+0, 0x1.5c9268a5946b7p+0, 0x1.5d84590998b93p+0,
    0x1.5e76f15ad2148p+0, 0x1.5f6a320dceb71p+0, 0x1.605e1b976dc09p+0, 0x1.6152ae6cdf6f4p+0,
    0x1.6247eb03a5585p+0, 0x1.633dd1d1929fdp+0, 0x1.6434634ccc320p+0, 0x1.652b9febc8fb7p+0,
    0x1.6623882552225p+0, 0x1.671c1c70833f6p+0, 0x1.68155d44ca973p+0, 0x1.690f4b19e9538p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6b052fa75173ep+0, 0x1.6c012750bdabfp+0, 0x1.6cfdcddd47645p+0,
    0x1.6dfb23c651a2fp+0, 0x1.6ef9298593ae5p+0, 0x1.6ff7df9519484p+0, 0x1.70f7466f42e87p+0,
    0x1.71f75e8ec5f74p+0, 0x1.72f8286ead08ap+0, 0x1.73f9a48a58174p+0, 0x1.74fbd35d7cbfdp+0,
    0x1.75feb564267c9p+0, 0x1.77024b1ab6e09p+0, 0x1.780694fde5d3fp+0, 0x1.790b938ac1cf6p+0,
    0x1.7a11473eb0187p+0, 0x1.7b17b0976cfdbp+0, 0x1.7c1ed0130c132p+0, 0x1.7d26a62ff86f0p+0,
    0x1.7e2f336cf4e62p+0, 0x1.7f3878491c491p+0, 0x1.80427543e1a12p+0, 0x1.814d2add106d9p+0,
    0x1.82589994cce13p+0, 0x1.8364c1eb941f7p+0, 0x1.8471a4623c7adp+0, 0x1.857f4179f5b21p+0,
    0x1.868d99b4492edp+0, 0x1.879cad931a436p+0, 0x1.88ac7d98a6699p+0, 0x1.89bd0a478580fp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8be05bad61778p+0, 0x1.8cf3216b5448cp+0, 0x1.8e06a5e0866d9p+0,
    0x1.8f1ae99157736p+0, 0x1.902fed0282c8ap+0, 0x1.9145b0b91ffc6p+0, 0x1.925c353aa2fe2p+0,
    0x1.93737b0cdc5e5p+0, 0x1.948b82b5f98e5p+0, 0x1.95a44cbc8520fp+0, 0x1.96bdd9a7670b3p+0,
    0x1.97d829fde4e50p+0, 0x1.98f33e47a22a2p+0, 0x1.9a0f170ca07bap+0, 0x1.9b2bb4d53fe0dp+0,
    0x1.9c49182a3f090p+0, 0x1.9d674194bb8d5p+0, 0x1.9e86319e32323p+0, 0x1.9fa5e8d07f29ep+0,
    0x1.a0c667b5de565p+0, 0x1.a1e7aed8eb8bbp+0, 0x1.a309bec4a2d33p+0, 0x1.a42c980460ad8p+0,
    0x1.a5503b23e255dp+0, 0x1.a674a8af46052p+0, 0x1.a799e1330b358p+0, 0x1.a8bfe53c12e59p+0,
    0x1.a9e6b5579fdbfp+0, 0x1.ab0e521356ebap+0, 0x1.ac36bbfd3f37ap+0, 0x1.ad5ff3a3c2774p+0,
    0x1.ae89f995ad3adp+0, 0x1.afb4ce622f2ffp+0, 0x1.b0e07298db666p+0, 0x1.b20ce6c9a8952p+0,
    0x1.b33a2b84f15fbp+0, 0x1.b468415b749b1p+0, 0x1.b59728de5593ap+0, 0x1.b6c6e29f1c52ap+0,
    0x1.b7f76f2fb5e47p+0, 0x1.b928cf22749e4p+0, 0x1.ba5b030a1064ap+0, 0x1.bb8e0b79a6f1fp+0,
    0x1.bcc1e904bc1d2p+0, 0x1.bdf69c3f3a207p+0, 0x1.bf2c25bd71e09p+0, 0x1.c06286141b33dp+0,
    0x1.c199bdd85529cp+0, 0x1.c2d1cd9fa652cp+0, 0x1.c40ab5fffd07ap+0, 0x1.c544778fafb22p+0,
    0x1.c67f12e57d14bp+0, 0x1.c7ba88988c933p+0, 0x1.c8f6d9406e7b5p+0, 0x1.ca3405751c4dbp+0,
    0x1.cb720dcef9069p+0, 0x1.ccb0f2e6d1675p+0, 0x1.cdf0b555dc3fap+0, 0x1.cf3155b5bab74p+0,
    0x1.d072d4a07897cp+0, 0x1.d1b532b08c968p+0, 0x1.d2f87080d89f2p+0, 0x1.d43c8eacaa1d6p+0,
    0x1.d5818dcfba487p+0, 0x1.d6c76e862e6d3p+0, 0x1.d80e316c98398p+0, 0x1.d955d71ff6075p+0,
    0x1.da9e603db3285p+0, 0x1.dbe7cd63a8315p+0, 0x1.dd321f301b460p+0, 0x1.de7d5641c0658p+0,
    0x1.dfc97337b9b5fp+0, 0x1.e11676b197d17p+0, 0x1.e264614f5a129p+0, 0x1.e3b333b16ee12p+0,
    0x1.e502ee78b3ff6p+0, 0x1.e653924676d76p+0, 0x1.e7a51fbc74c83p+0, 0x1.e8f7977cdb740p+0,
    0x1.ea4afa2a490dap+0, 0x1.eb9f4867cca6ep+0, 0x1.ecf482d8e67f1p+0, 0x1.ee4aaa2188510p+0,
    0x1.efa1bee615a27p+0, 0x1.f0f9c1cb6412ap+0, 0x1.f252b376bba97p+0, 0x1.f3ac948dd7274p+0,
    0x1.f50765b6e4540p+0, 0x1.f6632798844f8p+0, 0x1.f7bfdad9cbe14p+0, 0x1.f91d802243c89p+0,
    0x1.fa7c1819e90d8p+0, 0x1.fbdba3692d514p+0, 0x1.fd3c22b8f71f1p+0, 0x1.fe9d96b2a23d9p+0,
};
// 256/ln2; ln2/256 split hi (32 significant bits: kd * hi exact for |kd| < 2^21)
// + lo.
constexpr double kExpK = 369.3299304675746;
constexpr double kLn2o256Hi = 0x1.62e42fee00000p-9;
constexpr double kLn2o256Lo = 0x1.a39ef35793c76p-41;

// c * exp(d) + a for d in [-5.2e5, 256] with tab[j] = c 2^(j/256):
// d = k ln2/256 + r, |r| <= ln2/512; exp(r) by its degree-4 Taylor polynomial
// (truncation |r|^5/120 < 2^-54), times tab[k mod 256] with 2^(k div 256) added
// to its exponent (integer op), plus a in the same FMA.  <= 3 ulp; 9 FP64
// operations (kd * hi is exact for d > -5600; below, r stays small and the
// term negligible).  Below d = -500 the scale is held at 2^-722 (one integer
// max on k): the term is then < e^-300 |c| whatever r is, so callers whose
// |a| >= e^-200 |c| get a exactly, and c 2^(k div 256) stays a normal double.
// Callers bound d below (k, the low word of the magic-number sum, must not
// wrap: EvSum2GE certifies |x - mu| < 1000 sigma, d > -5.1e5).
constexpr int kKMin = -184665;  // floor(-500 * 256 / ln2)
__device__ __forceinline__ double cexp_tab_add(double d, const double* tab, double a) {
    const double t = fma(d, kExpK, 0x1.8p52);
    const int k = max(__double2loint(t), kKMin);
    const double kd = t - 0x1.8p52;
    double r = fma(kd, -kLn2o256Hi, d);
    r = fma(kd, -kLn2o256Lo, r);
    double q = fma(r, 1.0 / 24.0, 1.0 / 6.0);  // Horner: throughput-bound, Estrin measured slower
    q = fma(q, r, 0.5);
    q = fma(q, r, 1.0);
    q = fma(q, r, 1.0);
    const double tv = tab[k & (kTabN - 1)];
    const double cs = __hiloint2double(__double2hiint(tv) + (int)((unsigned)(k >> 8) << 20), __double2loint(tv));
    return fma(cs, q, a);
}

// SumPdf(gaussian, exponential) on one column (C1 / C5):
//   p = c0 exp(u0) + c1 exp(u1),  u0 = (-0.5 z) z,  z = (x - mu) / sigma,
//   u1 = alpha x,  c_t = weight_t / (norm_t * norm_root)
//   (pdf.py:122-127, 141-144, 205-219), factored as
//   p = exp(u1) * q,  q = c1 + c0 exp(d),  d = u0 - u1:
// one exponential per event; x goes into the unit's sum (times alpha once
// per unit: sum_i u1_i = alpha sum_i x_i), q into its product.
//   d = c2 w^2 - alpha w - alpha mu,  w = x - mu,  c2 = -1/(2 sigma^2):
// two FMAs on w, no cancellation beyond |alpha mu| (the u1 - alpha mu part).
// Leaf/term layout fixed by the dispatcher: leaf 0 gaussian (ptv[0][0..1] =
// mu, 1/sigma), leaf 1 exponential (ptv[0][2] = alpha), term t = leaf t, and
// |ln c_t| < 200.
// Certification (unit-level, integer ops): max |x - mu| over the unit below
// min(256 / |alpha| - |mu|, 1000 sigma) (the high words' maximum, Ev::XMAX;
// so |u1| < 256 and d >= -5e5 - 512) and q in [2^-250, 2^251) -- proven on
// the host from the parameters alone when possible (q >= c1, d <= alpha^2
// sigma^2 / 2 - alpha mu: EvSum2GE<true>, no per-event tracking) -- put p in
// [2^-620, 2^620] and keep the reference's exp(u1) finite and normal.  Below d = -500 cexp_tab_add holds the scale (integer
// max): c0 e^d <= e^-300 c1 < ulp(c1) / 2 -- q is c1 exactly -- and
// c0 2^(k div 256) stays a normal double.  Whatever an uncertified event
// computes is discarded (its block is deferred to the exact fix-up).
#ifndef PFB_SUM2GE_U
#define PFB_SUM2GE_U 4
#endif
#ifndef PFB_SUM2GE_MINB
#define PFB_SUM2GE_MINB 3
#endif
template <bool QC = false>
struct EvSum2GE {
    static constexpr int NC = 1;
    static constexpr int U = PFB_SUM2GE_U;
    static constexpr int MINB = PFB_SUM2GE_MINB;
    static constexpr bool TAB = true;     // tab = c0 2^(j/256)
    static constexpr bool LSCALE = true;  // unit sum of l times alpha
    static constexpr bool XMAX = true;    // unit check max |x - mu| < the host bound (g2_wlim)
    static constexpr bool QCERT = QC;     // q range certified on the host (g2_qcert): no per-event tracking
    static constexpr bool POINTS = true;  // per-point constants: batched in the TMA unit kernel (m = point)

    __device__ static __forceinline__ double cert_value(const NllArgs& A, double x, int m) {
        return x - A.ptv[m][0];
    }
    __device__ static __forceinline__ double tab_entry(const NllArgs& A, int j, int m) {
        return A.g2_c0[m] * kExp2Tab256[j];
    }
    __device__ static __forceinline__ double lscale(const NllArgs& A, int m) { return A.ptv[m][2]; }

    __device__ static __forceinline__ double one(const NllArgs& A, double x, const double* tab, bool& ok,
                                                 double& l, int m) {
#ifdef PFB_EXP_CHEAP  // measurement-only build: structure cost without the exponential
        ok = true;
        l = x;
        return fma(x, 1e-3, 1.0);
#endif
        // per-call constants of point m from the host (NllArgs::g2_*)
        const double w = x - A.ptv[m][0];
        const double d = fma(w, fma(A.g2_c2[m], w, -A.ptv[m][2]), -A.g2_amu[m]);
        ok = true;  // |x| certified per unit (XMAX); d < -500: cexp_tab_add
        l = x;
        return cexp_tab_add(d, tab, A.g2_c1[m]);
    }

    __device__ static __forceinline__ double2 prob2(const NllArgs& A, const double2 (&x)[1], bool& okx,
                                                    bool& oky, const double* tab, double2& l, int m = 0) {
        double2 q;
        q.x = one(A, x[0].x, tab, okx, l.x, m);
        q.y = one(A, x[0].y, tab, oky, l.y, m);
        return q;
    }
};

// ProdPdf(gaussian(x), polynomial(y)) on two columns (C2p):
//   p = c exp(u) q,  u = (-0.5 z) z,  z = (x - mu) / sigma,  q = polyval(y),
//   c = 1 / (norm_gauss norm_poly norm_root)  (pdf.py:122-127, 160-167, 205-219).
// The log sum takes l = ln c + u, the unit product q: one logarithm per 16
// events where the log-domain EvSop pays one per event (and its I2F / MUFU
// on the XU pipe: 108 us at 10M events, XU 74% busy -- ncu, round 2).
// Leaf/term layout fixed by the dispatcher (gp_ok): leaf 0 gaussian
// (ptv[0][0..1] = mu, 1/sigma), leaf 1 polynomial (ptv[0][2..] = coefficients,
// lowest order first), one term with emask {0}, vmask {1}, finite ln c.
// Certification: u >= -600 (the reference's exp(u) is a normal double), q
// positive within 2^+-250 (unit check), and the EvSop budget
// |u| + |log2 q| ln2 + 1 <= thr (thr = 690 - |ln c|: the reference's linear
// product stays normal).  Per unit (LMIN, lmin_ok): the smallest l bounds
// every -u and the unit's q range bounds every |log2 q|, so one check covers
// the unit's 16 events (a conservative superset of the per-event checks:
// ~9 fewer instructions per event).  Explicit _rn operations: every shell that runs
// this evaluator (bulk, TMA unit, SIMT) gives the same bits.  NV > 0: the
// coefficient count at compile time (unrolled Horner); 0: A.leaf[1].nv.
template <int NV = 0>
struct EvGaussPoly {
    static constexpr int NC = 2;
    static constexpr int U = 2;
    static constexpr int MINB = 3;
    static constexpr bool POINTS = true;  // every value from the point's ptv row: batchable
    static constexpr bool LMIN = PFB_UNIT_MINMAX != 0;  // the budget checked per unit
    __device__ static __forceinline__ double lcoef(const NllArgs& A, int m) { return A.ptv[m][kPtLeafWords]; }
    __device__ static __forceinline__ double lthr(const NllArgs& A, int m) { return A.ptv[m][kPtLeafWords + 1]; }

    __device__ static __forceinline__ double one(const NllArgs& A, double xg, double y, bool& ok, double& l,
                                                 int m = 0) {
        const double* v = A.ptv[m];
        const double z = __dmul_rn(__dsub_rn(xg, v[0]), v[1]);
        const double u = __dmul_rn(__dmul_rn(-0.5, z), z);
        const int nv = NV > 0 ? NV : A.leaf[1].nv;
        double q = v[1 + nv];
        if constexpr (NV > 0) {
#pragma unroll
            for (int i = NV - 1; i >= 1; --i) q = fma(q, y, v[1 + i]);
        } else {
#pragma unroll 1
            for (int i = nv - 1; i >= 1; --i) q = fma(q, y, v[1 + i]);
        }
        l = __dadd_rn(v[kPtLeafWords], u);
        if constexpr (LMIN) {
            ok = true;
        } else {
            // |binary exponent of q| as a double without I2F (magic-number add)
            const int e = ((__double2hiint(q) >> 20) & 0x7ff) - 1023;
            const double ae = __dsub_rn(__hiloint2double(0x43300000, e < 0 ? -e : e), 0x1p52);
            const double budget = fma(ae, 0.6931471805599453, __dsub_rn(1.0, u));
            ok = (u >= -600.0) && (budget <= v[kPtLeafWords + 1]);
        }
        return q;
    }

    __device__ static __forceinline__ double2 prob2(const NllArgs& A, const double2 (&x)[2], bool& okx,
                                                    bool& oky, const double*, double2& l, int m = 0) {
        const bool g1 = A.leaf[0].col != 0;
        double2 q;
        q.x = one(A, g1 ? x[1].x : x[0].x, g1 ? x[0].x : x[1].x, okx, l.x, m);
        q.y = one(A, g1 ? x[1].y : x[0].y, g1 ? x[0].y : x[1].y, oky, l.y, m);
        return q;
    }
};

// Any single-term product with value leaves (ProdPdf of gaussians,
// exponentials and polynomials on NC columns; a lone polynomial): the
// generalisation of EvGaussPoly with the leaf kinds fixed at compile time
// (KINDS, 2 bits per leaf as EvSop; -1: read per leaf at run time) and the
// Horner length read per leaf.
//   l = ln c + sum of the exp-type leaves' exponents (log sum),
//   q = product of the polynomial values (unit product).
// Certification as EvSop's single-term form: gaussian u >= -600, exponential
// |u| <= 600, the exponent budget sum |u| + sum (|log2 v| ln2 + 1) <= thr, and
// q within the unit range (positive, 2^+-250).  Layout checked by the
// dispatcher (prod1_ok): one term, every exp-type leaf in its emask, every
// polynomial in its vmask.
template <int NC_, int NL, int KINDS>
struct EvProd1 {
    static constexpr int NC = NC_;
    static constexpr int U = 2;
    static constexpr int MINB = 3;
    static constexpr bool POINTS = true;  // every value from the point's ptv row: batchable

    __device__ static __forceinline__ double pick(const double2 (&x)[NC_], int col, bool hi) {
        double r = hi ? x[0].y : x[0].x;
#pragma unroll
        for (int c = 1; c < NC_; ++c)
            if (col == c) r = hi ? x[c].y : x[c].x;
        return r;
    }

    __device__ static __forceinline__ double one(const NllArgs& A, const double2 (&x)[NC_], bool hi, bool& ok,
                                                 double& l, int m = 0) {
        const double* v = A.ptv[m];
        double q = 1.0, budget = 0.0;
        double ls = v[kPtLeafWords];
        bool good = true;
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            const SopLeaf& L = A.leaf[k];
            const int kind = KINDS >= 0 ? (KINDS >> (2 * k)) & 3 : L.kind;
            const double xv = pick(x, L.col, hi);
            if (kind == PFB_GAUSSIAN) {
                const double z = __dmul_rn(__dsub_rn(xv, v[L.voff]), v[L.voff + 1]);
                const double u = __dmul_rn(__dmul_rn(-0.5, z), z);
                good &= u >= -600.0;
                budget = __dsub_rn(budget, u);
                ls = __dadd_rn(ls, u);
            } else if (kind == PFB_EXPONENTIAL) {
                const double u = __dmul_rn(v[L.voff], xv);
                good &= fabs(u) <= 600.0;
                budget = __dadd_rn(budget, fabs(u));
                ls = __dadd_rn(ls, u);
            } else {  // polynomial (Horner, as polyval)
                const double* c = v + L.voff;
                double p = c[L.nv - 1];
#pragma unroll 1
                for (int i = L.nv - 2; i >= 0; --i) p = fma(p, xv, c[i]);
                const int e = ((__double2hiint(p) >> 20) & 0x7ff) - 1023;
                budget = fma(int_to_double(e < 0 ? -e : e), 0.6931471805599453, __dadd_rn(budget, 1.0));
                q = __dmul_rn(q, p);
            }
        }
        ok = good && budget <= v[kPtLeafWords + 1];
        l = ls;
        return q;
    }

    __device__ static __forceinline__ double2 prob2(const NllArgs& A, const double2 (&x)[NC_], bool& okx,
                                                    bool& oky, const double*, double2& l, int m = 0) {
        double2 q;
        q.x = one(A, x, false, okx, l.x, m);
        q.y = one(A, x, true, oky, l.y, m);
        return q;
    }
};

// Running state of one 16-event unit: the product m * 2^ex of the q factors,
// for ratio evaluators (Ev::RATIO, p = q / r) the product md * 2^exd of the
// r factors, and the sum ls of the log factors l.
struct Unit {
    double m = 1.0, md = 1.0, ls = 0.0;
    int ex = 0, exd = 0;
    int xhi = 0;  // Ev::XMAX: max of the events' |x| high words
#if PFB_UNIT_MINMAX
    // min / max of the high words of every q and r folded in: for positive
    // doubles the high word orders like the value, and zero, negatives, inf
    // and NaN all fall outside any finite positive range -- one unit-level
    // range check instead of one per event
    int qlo = 0x7fffffff, qhi = 0, rlo = 0x7fffffff, rhi = 0;
    double lmin = 1e300;  // Ev::LMIN: smallest l (every unit holds at least one event)
#endif
};

template <class Ev, class = void>
struct IsRatio {
    static constexpr bool value = false;
};
template <class Ev>
struct IsRatio<Ev, decltype((void)Ev::RATIO)> {
    static constexpr bool value = Ev::RATIO;
};
template <class Ev, class = void>
struct HasLMin {
    static constexpr bool value = false;
};
template <class Ev>
struct HasLMin<Ev, decltype((void)Ev::LMIN)> {
    static constexpr bool value = Ev::LMIN;
};
template <class Ev, class = void>
struct HasXMax {
    static constexpr bool value = false;
};
template <class Ev>
struct HasXMax<Ev, decltype((void)Ev::XMAX)> {
    static constexpr bool value = Ev::XMAX;
};
template <class Ev, class = void>
struct HasPoints {
    static constexpr bool value = false;
};
template <class Ev>
struct HasPoints<Ev, decltype((void)Ev::POINTS)> {
    static constexpr bool value = Ev::POINTS;
};
template <class Ev, class = void>
struct HasQCert {
    static constexpr bool value = false;
};
template <class Ev>
struct HasQCert<Ev, decltype((void)Ev::QCERT)> {
    static constexpr bool value = Ev::QCERT;
};
// p = q / r^POW for ratio evaluators
template <class Ev, class = void>
struct RatioPow {
    static constexpr int value = 1;
};
template <class Ev>
struct RatioPow<Ev, decltype((void)Ev::RATIO_POW)> {
    static constexpr int value = Ev::RATIO_POW;
};

// One row of a unit: evaluate two events (local block indices e, e+1),
// mask absent tail events (TAIL), certify, multiply into the unit.
template <class Ev, bool TAIL>
__device__ __forceinline__ void prod_row(const NllArgs& A, const double2 (&x)[Ev::NC], int e, int n, Unit& u,
                                         bool& bad, const double* tab, bool renorm_now = true, int m = 0) {
    constexpr bool RATIO = IsRatio<Ev>::value;
    bool okx, oky;
    double2 l = make_double2(0.0, 0.0);
    double2 r = make_double2(1.0, 1.0);
    double2 q;
    if constexpr (RATIO && HasPoints<Ev>::value)
        q = Ev::prob2r(A, x, okx, oky, r, m);
    else if constexpr (RATIO)
        q = Ev::prob2r(A, x, okx, oky, r);
    else if constexpr (HasPoints<Ev>::value)
        q = Ev::prob2(A, x, okx, oky, tab, l, m);
    else
        q = Ev::prob2(A, x, okx, oky, tab, l);
#if PFB_UNIT_MINMAX
    // (before the tail masking: an absent second event duplicates the first)
    if constexpr (HasLMin<Ev>::value) u.lmin = fmin(u.lmin, fmin(l.x, l.y));
#endif
    if (TAIL) {
        if (e >= n) {
            q.x = 1.0;
            r.x = 1.0;
            l.x = 0.0;
            okx = true;
        }
        if (e + 1 >= n) {
            q.y = 1.0;
            r.y = 1.0;
            l.y = 0.0;
            oky = true;
        }
    }
    if constexpr (HasXMax<Ev>::value) {
        const int a = (TAIL && e >= n) ? 0 : (__double2hiint(Ev::cert_value(A, x[0].x, m)) & 0x7fffffff);
        const int b = (TAIL && e + 1 >= n) ? 0 : (__double2hiint(Ev::cert_value(A, x[0].y, m)) & 0x7fffffff);
        u.xhi = max(u.xhi, max(a, b));
    }
#if PFB_UNIT_MINMAX
    bad |= !(okx && oky);
    if constexpr (!HasQCert<Ev>::value) {  // (certified: the initial qlo / qhi pass the unit check)
        const int a = __double2hiint(q.x), b = __double2hiint(q.y);
        u.qlo = min(u.qlo, min(a, b));
        u.qhi = max(u.qhi, max(a, b));
    }
    if constexpr (RATIO) {
        const int a = __double2hiint(r.x), b = __double2hiint(r.y);
        u.rlo = min(u.rlo, min(a, b));
        u.rhi = max(u.rhi, max(a, b));
        u.md = (u.md * r.x) * r.y;
        if (renorm_now) renorm(u.md, u.exd);
    } else {
        u.ls = (u.ls + l.x) + l.y;
    }
    u.m = (u.m * q.x) * q.y;
    if (renorm_now) renorm(u.m, u.ex);
#else
    bool ok = okx && oky && p_in_range(q.x) && p_in_range(q.y);
    if constexpr (RATIO) {
        // r^POW in [2^-500, 2^500] (p = q / r^POW then stays within 2^+-1000)
        constexpr int span = 500 / RatioPow<Ev>::value;
        auto r_ok = [](double v) {
            return (unsigned)((__double2hiint(v) >> 20) - (1023 - span)) <= (unsigned)(2 * span);
        };
        ok = ok && r_ok(r.x) && r_ok(r.y);
        u.md = (u.md * r.x) * r.y;
        renorm(u.md, u.exd);
    } else {
        u.ls = (u.ls + l.x) + l.y;
    }
    bad |= !ok;
    u.m = (u.m * q.x) * q.y;
    renorm(u.m, u.ex);
    (void)renorm_now;
#endif
}

// The unit-level range check (PFB_UNIT_MINMAX): every factor within 2^+-kSpanM.
__device__ __forceinline__ bool unit_in_range(const Unit& u, bool ratio) {
#if PFB_UNIT_MINMAX
    constexpr int lo = (1023 - kSpanM) << 20, hi = (1023 + kSpanM + 1) << 20;
    bool ok = u.qlo >= lo && u.qhi < hi;
    if (ratio) ok = ok && u.rlo >= lo && u.rhi < hi;
    return ok;
#else
    (void)u;
    (void)ratio;
    return true;
#endif
}

// Ev::LMIN's budget for the whole unit: -u <= ln c - lmin (+ 1e-9 for the
// rounding of l = ln c + u and of the difference, both < 2^-41 here) bounds
// every event's -u, and the high words qlo / qhi (positive, within 2^+-kSpanM
// once unit_in_range holds) bound every |binary exponent of q|.
template <class Ev>
__device__ __forceinline__ bool lmin_ok(const NllArgs& A, const Unit& u, int m) {
#if PFB_UNIT_MINMAX
    const double negu = __dadd_rn(__dsub_rn(Ev::lcoef(A, m), u.lmin), 1e-9);
    const int elo = ((u.qlo >> 20) & 0x7ff) - 1023, ehi = ((u.qhi >> 20) & 0x7ff) - 1023;
    const int me = max(abs(elo), abs(ehi));
    return negu <= 600.0 && fma(int_to_double(me), 0.6931471805599453, __dadd_rn(1.0, negu)) <= Ev::lthr(A, m);
#else
    (void)A;
    (void)u;
    (void)m;
    return true;
#endif
}

// every unit-level certificate of an evaluator
template <class Ev>
__device__ __forceinline__ bool unit_ok(const NllArgs& A, const Unit& u, int m = 0) {
    bool ok = unit_in_range(u, IsRatio<Ev>::value);
    if constexpr (HasXMax<Ev>::value) ok = ok && u.xhi < A.g2_wlim[m];
    if constexpr (HasLMin<Ev>::value) ok = ok && lmin_ok<Ev>(A, u, m);
    return ok;
}

// per-launch shared table (Ev::TAB) and scaled log sums (Ev::LSCALE)
template <class Ev, class = void>
struct HasTab {
    static constexpr bool value = false;
};
template <class Ev>
struct HasTab<Ev, decltype((void)Ev::TAB)> {
    static constexpr bool value = Ev::TAB;
};
template <class Ev, class = void>
struct HasLScale {
    static constexpr bool value = false;
};
template <class Ev>
struct HasLScale<Ev, decltype((void)Ev::LSCALE)> {
    static constexpr bool value = Ev::LSCALE;
};
template <class Ev>
__device__ __forceinline__ void init_tab(const NllArgs& A, double* tab, int tid, int npts = 1, int nthreads = 0) {
    // nthreads: the threads taking part (0: the whole CTA)
    if constexpr (HasTab<Ev>::value) {
        const int step = nthreads > 0 ? nthreads : (int)blockDim.x;
        for (int j = tid; j < npts * kTabN; j += step) tab[j] = Ev::tab_entry(A, j % kTabN, j / kTabN);
    }
}

template <class Ev>
__device__ __forceinline__ double unit_value(const NllArgs& A, const Unit& u, int m = 0) {
    if constexpr (IsRatio<Ev>::value) {
        constexpr double pw = (double)RatioPow<Ev>::value;
        const double fe = fma(-pw, int_to_double(u.exd), int_to_double(u.ex));
        return -fma(fe, kLn2Hi, fma(fe, kLn2Lo, fma(-pw, log_unit(u.md), log_unit(u.m))));
    } else {
        const double fe = int_to_double(u.ex);
        // explicit fma / add: no contraction choice left to the compiler, so
        // every kernel shell (bulk, task, TMA, SIMT, persistent) gives the same bits
        double s;
        if constexpr (HasLScale<Ev>::value)
            s = fma(Ev::lscale(A, m), u.ls, log_unit(u.m));
        else
            s = __dadd_rn(log_unit(u.m), u.ls);
        return -fma(fe, kLn2Hi, fma(fe, kLn2Lo, s));
    }
}

// ---------------------------------------------------------------------------
// TMA-fed unit kernel.  PROD = false: unit sums of log-domain terms (C2 --
// cheap per-event terms, HBM-bound); PROD = true: the product-mode units
// above (C1 / Dalitz -- FP64-bound; the consumers read their rows from shared
// memory instead of waiting on global loads).  Block structure: unit = 8 rows
// x one lane's 2 columns (row order, x then y), block = lane tree of the unit
// tree.  Consumers work in
// teams of eight warps; warp w of a team owns unit-row w (the contiguous 4 KB
// [512w, 512w+512) of every column block) and teams take alternate stages, so
// a block costs ~16 evaluations per lane and one barrier-free fold (last of
// the eight to post).  Blocks are not the reference tree's -- the NLL is
// within rounding of it, not bitwise -- which is why the known-answer
// reduction keeps nll_tma_kernel.
constexpr int kSumWarps = 8;  // warps per team (one unit-row each)
#ifndef PFB_UNIT_TEAMS1
#define PFB_UNIT_TEAMS1 3
#endif
#ifndef PFB_UNIT_TEAMS2
#define PFB_UNIT_TEAMS2 2
#endif
// consumer teams: 2 for two-column stages (3 x 64 KB), 3 for one-column
// stages (6 x 32 KB) when the evaluator fits 80 registers
template <class Ev>
struct UnitTeams {
    static constexpr int value = Ev::NC == 1 ? PFB_UNIT_TEAMS1 : PFB_UNIT_TEAMS2;
};
constexpr int kSumRing = 4;
#ifndef PFB_PRODUCER_SLEEP
#define PFB_PRODUCER_SLEEP 1
#endif
#ifndef PFB_CONSUMER_SLEEP
#define PFB_CONSUMER_SLEEP 0
#endif
#if PFB_CONSUMER_SLEEP
#define PFB_CONSUMER_WAIT mbar_wait_sleep
#else
#define PFB_CONSUMER_WAIT mbar_wait
#endif
#if PFB_PRODUCER_SLEEP
#define PFB_PRODUCER_WAIT mbar_wait_sleep
#else
#define PFB_PRODUCER_WAIT mbar_wait
#endif

// PFB_TRACE timeline helpers: pfb_nll_kernel.cuh

// ONE: a single parameter point (A.npts == 1) with the point index a
// compile-time 0 -- POINTS evaluators then read constant parameter offsets as
// unbatched ones do (a runtime index cost the C2p kernel 15%).
template <class Ev, int S, bool PROD, int TEAMS = UnitTeams<Ev>::value, bool ONE = false>
__global__ void __launch_bounds__(32 * (kSumWarps * TEAMS + 1), 1) nll_tma_unit_kernel(const __grid_constant__ NllArgs A) {
    constexpr int kSumTeams = TEAMS;
    constexpr int NC = Ev::NC;
    extern __shared__ __align__(128) double stage[];  // S x NC x 4096 doubles

    // full barriers per (team, stage): a team waits only on the phases of
    // its own uses of a stage, one phase at a time.  (A single full barrier
    // per stage would let a team waiting for its next use of the stage match
    // the parity of the previous team's still-pending phase -- the mbarrier
    // parity wait cannot tell phases two apart.)
    constexpr int L = S % kSumTeams == 0 ? S : S * kSumTeams;  // lcm(S, teams) for S in {3, 6}
    __shared__ unsigned long long full_bar[kSumTeams][S], empty_bar[S];
    __shared__ long long s_blk[S];
    __shared__ double xch[kSumTeams][kSumRing][kSumWarps][32];
    __shared__ int xbad[kSumTeams][kSumRing][kSumWarps];
    __shared__ unsigned int s_cnt[kSumTeams][kSumRing];
    __shared__ int s_done[kSumTeams][kSumRing];
    __shared__ long long sacc[kMaxPts][PFB_ACC_WORDS];
    // the evaluator's shared tables, one per parameter point (batched product
    // mode): dynamic shared memory after the stages (static is capped at 48 KB)
    double* const s_tab = stage + (int64_t)S * NC * kBlock;
    __shared__ unsigned int s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    if (tid == 0) PFB_T(0);
#ifdef PFB_TRACE
    if (tid < 4) g_trace[blockIdx.x][8 + tid] = 0;
#endif
    // Start-up: the producer warp initialises the mbarriers and starts copying
    // at once; it only *arrives* on named barrier 1, which the consumers
    // sync on after zeroing their state -- so the first copy is not queued
    // behind the consumers' set-up (measured: first copy 1.5 us -> ~0.2 us
    // after CTA start).  The arrive orders the barrier initialisation before
    // every consumer's first wait.
    constexpr int kAll = 32 * (kSumWarps * TEAMS + 1);
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    if (warp == kSumWarps * kSumTeams) {
        if (lane == 0) {
            for (int s = 0; s < S; ++s) {
                for (int t = 0; t < kSumTeams; ++t) mbar_init(&full_bar[t][s], 1);
                mbar_init(&empty_bar[s], kSumWarps);
            }
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
        asm volatile("bar.arrive 1, %0;" ::"n"(kAll) : "memory");
        if (lane == 0) {  // producer: as nll_tma_kernel's
            // the first item is this CTA's own (no device-wide round trip
            // before the first copy); the rest are claimed from the counter,
            // one stage ahead
            int64_t it_next = blockIdx.x;
            for (int u = 0;; ++u) {
                const int s = u % S;
                PFB_PRODUCER_WAIT(&empty_bar[s], ((u / S) & 1) ^ 1);
                const int64_t it = it_next;
                if (it < nitems) it_next = (int64_t)gridDim.x + (int64_t)atomicAdd(A.work_counter, 1ull);
                if (it >= nitems) {
                    // one end marker per team
                    s_blk[s] = -1;
                    mbar_arrive(&full_bar[u % kSumTeams][s]);
                    for (int extra = 1; extra < kSumTeams; ++extra) {
                        const int v = u + extra, s2 = v % S;
                        PFB_PRODUCER_WAIT(&empty_bar[s2], ((v / S) & 1) ^ 1);
                        s_blk[s2] = -1;
                        mbar_arrive(&full_bar[v % kSumTeams][s2]);
                    }
                    break;
                }
                const bool is_tail = A.tail && it == 0;
                const int64_t bidx = is_tail ? A.nfull : it - (A.tail ? 1 : 0);
                s_blk[s] = bidx;
                const unsigned bytes = is_tail ? (unsigned)(8 * (A.tail & ~1)) : (unsigned)(8 * kBlock);
                unsigned long long* fb = &full_bar[u % kSumTeams][s];
                mbar_arrive_expect_tx(fb, bytes * NC);
                if (bytes) {
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        bulk_g2s(stage + ((int64_t)s * NC + c) * kBlock,
                                 A.col[c] + A.begin + bidx * (int64_t)kBlock, bytes, fb);
                }
                if (u == 0) PFB_T(1);
            }
        }
    } else {
        init_tab<Ev>(A, s_tab, tid, A.npts, 32 * kSumWarps * kSumTeams);  // the consumer threads only
        for (int i = tid; i < kMaxPts * PFB_ACC_WORDS; i += 32 * kSumWarps * kSumTeams) (&sacc[0][0])[i] = 0;
        if (tid < kSumTeams * kSumRing) {
            (&s_cnt[0][0])[tid] = 0u;
            (&s_done[0][0])[tid] = 0;
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kAll) : "memory");
        const int team = warp / kSumWarps;
        const int w = warp % kSumWarps;
        int f = 0;
        // post this warp's unit value for point m; the last of the team's
        // eight to arrive folds the block (no barrier)
        auto post_fold = [&](double acc, bool bad, int m, int64_t bidx) {
            const unsigned anybad = __any_sync(0xffffffffu, bad);
            const int slot = f % kSumRing;
            if (lane == 0)
                while (*reinterpret_cast<volatile int*>(&s_done[team][slot]) < f / kSumRing) __nanosleep(20);
            __syncwarp();
            xch[team][slot][w][lane] = acc;
            unsigned arrived = 0;
            if (lane == 0) {
                xbad[team][slot][w] = anybad ? 1 : 0;
                __threadfence_block();
                arrived = atomicAdd(&s_cnt[team][slot], 1u);
            }
            arrived = __shfl_sync(0xffffffffu, arrived, 0);
            if (arrived == kSumWarps - 1) {
                __threadfence_block();
                bool fbad = false;
#pragma unroll
                for (int q = 0; q < kSumWarps; ++q) fbad |= xbad[team][slot][q] != 0;
                double bsum = 0.0;
                if (!fbad) {
                    double v[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) v[q] = xch[team][slot][q][lane];
                    double T = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
#pragma unroll
                    for (int off = 16; off >= 1; off /= 2) T = T + __shfl_down_sync(0xffffffffu, T, off);
                    bsum = T;
                }
                __syncwarp();
                if (lane == 0) {
                    if (fbad) {
                        const unsigned long long fs = atomicAdd(A.fix_counter, 1ull);
                        A.fix_list[fs] = (A.block_base + bidx) * kMaxPts + m;
                    } else {
                        if (A.block_sums && m == 0) A.block_sums[A.block_base + bidx] = bsum;
                        acc_add_shared(sacc[m], bsum);
                    }
                    s_cnt[team][slot] = 0u;
                    __threadfence_block();
                    *reinterpret_cast<volatile int*>(&s_done[team][slot]) = f / kSumRing + 1;
                }
            }
            ++f;
        };
        for (int u = team;; u += kSumTeams) {
            const int s = u % S;
#ifdef PFB_TRACE
            const unsigned long long tw0 = gtimer();
#endif
            PFB_CONSUMER_WAIT(&full_bar[team][s], (u / L) & 1);  // this team's (u / L)-th use of stage s
            const int64_t bidx = s_blk[s];
#ifdef PFB_TRACE
            if (w == 0 && lane == 0 && team < 2 && u >= kSumTeams && bidx >= 0) {
                g_trace[blockIdx.x][8 + team] += gtimer() - tw0;
                g_trace[blockIdx.x][10 + team] += 1;
            }
            if (u == 0 && w == 0 && lane == 0) PFB_T(2);
            if (bidx < 0 && w == 0 && lane == 0 && team < 2) PFB_T(3 + team);
#endif
            if (bidx < 0) break;
            const double* sx = stage + (int64_t)s * NC * kBlock;
            const bool tail = A.tail && bidx == A.nfull;
            const int n = tail ? A.tail : kBlock;
            for (int m = 0; m < (ONE ? 1 : A.npts); ++m) {
                bool bad = false;
                double acc = 0.0;
                Unit un;
                if (!tail) {
#pragma unroll
                    for (int r = 0; r < 8; ++r) {
                        const int e = (8 * w + r) * 64 + 2 * lane;
                        double2 x[NC];
#pragma unroll
                        for (int c = 0; c < NC; ++c) x[c] = *reinterpret_cast<const double2*>(sx + c * kBlock + e);
                        if constexpr (PROD) {
                            prod_row<Ev, false>(A, x, 0, kBlock, un, bad, s_tab + m * kTabN, (r & 1) != 0, m);
                        } else {
                            const double2 t = Ev::eval2(A, x, 0, sacc[0], 2, bad, m);
                            acc = (acc + t.x) + t.y;
                        }
                    }
                } else {
                    const int64_t gbase = A.begin + A.nfull * (int64_t)kBlock;
#pragma unroll 1
                    for (int r = 0; r < 8; ++r) {
                        const int e = (8 * w + r) * 64 + 2 * lane;
                        if (e >= n) break;  // rows ascend: nothing further in this lane
                        const int nv = e + 1 < n ? 2 : 1;
                        double2 x[NC];
#pragma unroll
                        for (int c = 0; c < NC; ++c) {
                            if (nv == 2) {
                                x[c] = *reinterpret_cast<const double2*>(sx + c * kBlock + e);
                            } else {  // odd last event: not bulk-copied
                                const double v = __ldg(A.col[c] + gbase + e);
                                x[c] = make_double2(v, v);
                            }
                        }
                        if constexpr (PROD) {
                            prod_row<Ev, true>(A, x, e, n, un, bad, s_tab + m * kTabN, true, m);
                        } else {
                            const double2 t = Ev::eval2(A, x, 0, sacc[0], nv, bad, m);
                            acc = acc + t.x;
                            if (nv == 2) acc = acc + t.y;
                        }
                    }
                }
                if constexpr (PROD) {
                    bad |= !unit_ok<Ev>(A, un, m);
                    acc = unit_value<Ev>(A, un, m);
                }
                if (ONE || m == A.npts - 1) {  // the stage is no longer read by this warp
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&empty_bar[s]);
                }
                post_fold(acc, bad, m, bidx);
            }
        }
    }
#ifdef PFB_TRACE
    if (tid == 0) PFB_T(5);
#endif
    finish_launch_pts(A, &sacc[0][0], A.npts * PFB_ACC_WORDS, &s_last);
#ifdef PFB_TRACE
    __syncthreads();
    if (tid == 0) PFB_T(6 + (s_last ? 1 : 0));
#endif
}

template <class Ev, bool PROD>
static cudaError_t launch_tma_unit(const NllArgs& A, cudaStream_t stream, int sm_count) {
    constexpr int NC = Ev::NC;
    // the team / stage phase bookkeeping needs S >= 3 stages (measured: a
    // single stage with two teams never completes)
    static_assert(NC <= 2, "TMA unit kernel: one or two columns");
    // one-column stages: six of 32 KB, four when the evaluator keeps shared
    // tables (2 KB per parameter point) -- static + dynamic shared memory
    // stays within the 227 KB limit
    constexpr int S = NC == 1 ? (HasTab<Ev>::value ? 4 : 6) : 3;
    const size_t smem = (size_t)S * NC * kBlock * sizeof(double) +
                        (HasTab<Ev>::value ? (size_t)kMaxPts * kTabN * sizeof(double) : 0);
    constexpr int T = UnitTeams<Ev>::value;
    constexpr bool kOne = HasPoints<Ev>::value && !IsRatio<Ev>::value;  // a single-point instance pays off
    const bool one = kOne && A.npts == 1;
    static bool configured[2] = {false, false};
    if (!configured[one]) {
        cudaError_t e = one ? cudaFuncSetAttribute(nll_tma_unit_kernel<Ev, S, PROD, T, kOne>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                            : cudaFuncSetAttribute(nll_tma_unit_kernel<Ev, S, PROD, T>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        configured[one] = true;
    }
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    int64_t grid = sm_count;
    if (grid > nitems) grid = nitems > 0 ? nitems : 1;
    if (one)
        nll_tma_unit_kernel<Ev, S, PROD, T, kOne><<<(unsigned)grid, 32 * (kSumWarps * T + 1), smem, stream>>>(A);
    else
        nll_tma_unit_kernel<Ev, S, PROD, T><<<(unsigned)grid, 32 * (kSumWarps * T + 1), smem, stream>>>(A);
    return cudaGetLastError();
}

template <class Ev>
static cudaError_t launch_tma_sum(const NllArgs& A, cudaStream_t stream, int sm_count) {
    return launch_tma_unit<Ev, false>(A, stream, sm_count);
}

#ifndef PFB_SUM_W
#define PFB_SUM_W 4
#endif
#ifndef PFB_SUM_SIMT
#define PFB_SUM_SIMT 0
#endif
#ifndef PFB_SUM_MINB
#define PFB_SUM_MINB 2
#endif
// PROD = false: the same kernel for log-domain evaluators (unit value = the
// row-ordered sum of the unit's 16 terms, exactly as nll_tma_unit_kernel's
// sum mode), one parameter point.
template <int P, class Ev, bool PROD = true>
__global__ void __launch_bounds__(kThreads, PROD ? Ev::MINB : PFB_SUM_MINB) nll_prod_kernel(const __grid_constant__ NllArgs A) {
    static_assert(P == 1 || P == 2 || P == 4 || P == 8, "P");
    constexpr int NC = Ev::NC;
    constexpr int GROUPS = kThreads / (32 * P);
    constexpr int ROWS = 64 / P;  // rows per warp
    constexpr int W = PROD ? Ev::U : PFB_SUM_W;  // row loads kept in flight
    static_assert(W <= ROWS && 8 % W == 0, "window");

    // Unit values of KF items per group, folded together after one barrier
    // (warp w folds one of the KF x GROUPS = 8 blocks); two halves so a
    // warp may start the next KF items while others still fold.
    constexpr int KF = 8 / GROUPS;
    __shared__ double xch[2][KF][GROUPS][8][32];
    __shared__ int xbad[2][KF][GROUPS][P];
    __shared__ long long xbidx[2][KF][GROUPS];
    __shared__ long long sacc[PFB_ACC_WORDS];
    __shared__ double s_tab[kTabN];
    __shared__ unsigned int s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int warp = tid >> 5;
    const int grp = warp / P;
    const int wig = warp % P;
    for (int i = tid; i < PFB_ACC_WORDS; i += blockDim.x) sacc[i] = 0;
    init_tab<Ev>(A, s_tab, tid);
    __syncthreads();

    // Static round-robin items (every block costs the same): the next item is
    // known in advance, so its first rows stream in while the current item's
    // last rows compute, and one group barrier per item suffices.  Item 0 is
    // the ragged tail (if any).
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    const int64_t stride = (int64_t)gridDim.x * GROUPS;
    const int r0 = wig * ROWS;
    struct Item {
        int64_t off;  // A.begin + first event of the block
        int64_t bidx;
        int n;
        bool tail;
    };
    auto item_of = [&](int64_t it, Item& I) {
        I.tail = A.tail && it == 0;
        I.bidx = I.tail ? A.nfull : it - (A.tail ? 1 : 0);
        I.n = I.tail ? A.tail : kBlock;
        I.off = A.begin + I.bidx * (int64_t)kBlock;
    };
    auto load_full = [&](const Item& I, int row, double2 (&dst)[NC]) {
        const int64_t e = I.off + row * 64 + 2 * lane;
#pragma unroll
        for (int c = 0; c < NC; ++c) dst[c] = ld2(A.col[c] + e);
    };
    auto load = [&](const Item& I, int row, double2 (&dst)[NC]) {
        if (!I.tail || row * 64 + 2 * lane + 1 < I.n) {
            load_full(I, row, dst);
        } else {  // ragged tail: a lone last event, or a stand-in (masked below)
            const int64_t e = I.off + row * 64 + 2 * lane;
            const int64_t j = row * 64 + 2 * lane < I.n ? e : I.off;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double v = __ldg(A.col[c] + j);
                dst[c] = make_double2(v, v);
            }
        }
    };

    const int64_t base = (int64_t)blockIdx.x * GROUPS;
    int64_t it = base + grp;
    Item cur_item, next_item;
    double2 win[W][NC];
    // UP: every row of the warp's unit loaded at the top of the item (one
    // unit per warp, window = all 8 rows); no prefetch across items -- the
    // other resident warps cover the latency
    constexpr bool UP = P == 8 && W >= 8;
    if (it < nitems) {
        item_of(it, cur_item);
        if constexpr (!UP) {
#pragma unroll
            for (int q = 0; q < W; ++q) load(cur_item, r0 + q, win[q]);
        }
    }
    // fold entry (half, s, g): the block a group computed KF items ago
    auto fold = [&](int half, int s, int g) {
        const long long bidx = xbidx[half][s][g];
        if (bidx < 0) return;
        bool fbad = false;
#pragma unroll
        for (int w = 0; w < P; ++w) fbad |= xbad[half][s][g][w] != 0;
        double bsum = 0.0;
        if (!fbad) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = xch[half][s][g][u][lane];
            double T = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
#pragma unroll
            for (int off = 16; off >= 1; off /= 2) T = T + __shfl_down_sync(0xffffffffu, T, off);
            bsum = T;
        }
        if (lane == 0) {
            if (fbad) {  // defer the whole block to the exact fix-up launch
                const unsigned long long fs = atomicAdd(A.fix_counter, 1ull);
                A.fix_list[fs] = (A.block_base + bidx) * kMaxPts + A.fix_point;
            } else {
                if (A.block_sums) A.block_sums[A.block_base + bidx] = bsum;
                acc_add_shared(sacc, bsum);
            }
        }
    };
    // CTA-uniform rounds (groups past the end skip the work, not the barriers)
    for (int k = 0; base + (int64_t)k * stride < nitems; ++k, it += stride) {
        const int half = (k / KF) & 1, slot = k % KF;
        if (it >= nitems) {
            if (wig == 0 && lane == 0) xbidx[half][slot][grp] = -1;
        } else {
        const bool has_next = it + stride < nitems;
        if (has_next) item_of(it + stride, next_item);
        bool bad = false;
        if (UP && !cur_item.tail) {
            double2 xr[8][NC];
#pragma unroll
            for (int r = 0; r < 8; ++r) load_full(cur_item, r0 + r, xr[r]);
            Unit un;
            double acc = 0.0;
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                if constexpr (PROD) {
                    prod_row<Ev, false>(A, xr[r], 0, kBlock, un, bad, s_tab, (r & 1) != 0);
                } else {
                    const double2 t = Ev::eval2(A, xr[r], 0, sacc, 2, bad, 0);
                    acc = (acc + t.x) + t.y;
                }
            }
            if constexpr (PROD) {
                bad |= !unit_ok<Ev>(A, un);
                acc = unit_value<Ev>(A, un);
            }
            xch[half][slot][grp][r0 >> 3][lane] = acc;
        } else if (!cur_item.tail) {
            // 8-row units; rows unrolled so the load window rotates by
            // register naming (slot r % W holds row r until consumed/refilled)
#pragma unroll 1
            for (int ju = 0; ju < ROWS / 8; ++ju) {
                Unit un;
                double acc = 0.0;
#pragma unroll
                for (int r = 0; r < 8; ++r) {
                    const int i = 8 * ju + r;
                    double2 cur[NC];
#pragma unroll
                    for (int c = 0; c < NC; ++c) cur[c] = win[r % W][c];
                    if (i + W < ROWS)
                        load_full(cur_item, r0 + i + W, win[r % W]);
                    else if (has_next)
                        load_full(next_item, r0 + i + W - ROWS, win[r % W]);
                    if constexpr (PROD) {
                        prod_row<Ev, false>(A, cur, 0, kBlock, un, bad, s_tab, (r & 1) != 0);
                    } else {
                        const double2 t = Ev::eval2(A, cur, 0, sacc, 2, bad, 0);
                        acc = (acc + t.x) + t.y;
                    }
                }
                if constexpr (PROD) {
                    bad |= !unit_ok<Ev>(A, un);
                    acc = unit_value<Ev>(A, un);
                }
                xch[half][slot][grp][(r0 >> 3) + ju][lane] = acc;
            }
        } else {
            // the ragged tail block (once per launch): same structure, rolled
            if constexpr (UP) {
#pragma unroll
                for (int q = 0; q < W; ++q) load(cur_item, r0 + q, win[q]);
            }
            Unit un;
            double acc = 0.0;
#pragma unroll 1
            for (int i = 0; i < ROWS; ++i) {
                double2 cur[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) cur[c] = win[0][c];
#pragma unroll
                for (int q = 0; q + 1 < W; ++q)
#pragma unroll
                    for (int c = 0; c < NC; ++c) win[q][c] = win[q + 1][c];
                if (i + W < ROWS)
                    load(cur_item, r0 + i + W, win[W - 1]);
                else if (has_next && !UP)
                    load_full(next_item, r0 + i + W - ROWS, win[W - 1]);
                const int e = (r0 + i) * 64 + 2 * lane;
                if constexpr (PROD) {
                    prod_row<Ev, true>(A, cur, e, cur_item.n, un, bad, s_tab);
                } else if (e < cur_item.n) {  // absent events add nothing
                    const int nv = e + 1 < cur_item.n ? 2 : 1;
                    const double2 t = Ev::eval2(A, cur, 0, sacc, nv, bad, 0);
                    acc = acc + t.x;
                    if (nv == 2) acc = acc + t.y;
                }
                if ((i & 7) == 7) {
                    if constexpr (PROD) {
                    bad |= !unit_ok<Ev>(A, un);
                    acc = unit_value<Ev>(A, un);
                }
                    xch[half][slot][grp][(r0 + i) >> 3][lane] = acc;
                    un = Unit();
                    acc = 0.0;
                }
            }
        }
        const unsigned anybad = __any_sync(0xffffffffu, bad);
        if (lane == 0) xbad[half][slot][grp][wig] = anybad ? 1 : 0;
        if (wig == 0 && lane == 0) xbidx[half][slot][grp] = cur_item.bidx;
        if (has_next) cur_item = next_item;
        }
        if (slot == KF - 1 || base + (int64_t)(k + 1) * stride >= nitems) {
            if constexpr (KF == 1) {
                group_sync<P>(grp);
                if (wig == 0) fold(half, 0, grp);
            } else {
                __syncthreads();
                if (warp % KF <= slot) fold(half, warp % KF, warp / KF);
            }
        }
    }
    finish_launch<false>(A, sacc, &s_last);
}

// ---------------------------------------------------------------------------
// Bulk-copy variant (single-column evaluators).  Same canonical block
// structure with P = 8 (warp w owns unit w = rows [8w, 8w+8), i.e. the
// contiguous 4 KB [512w, 512w+512) of every block).  Each warp streams its
// next item's 4 KB with one cp.async.bulk into a private double buffer in
// shared memory (own mbarrier per buffer), so a whole item of prefetch is in
// flight per warp without spending registers on it, and reads its rows back
// with conflict-free 16-byte shared loads.
constexpr int kBulkWarps = 8;
constexpr int kUnitEvents = 512;  // events per warp per item
#ifndef PFB_BULK_RING
#define PFB_BULK_RING 4
#endif
constexpr int kRing = PFB_BULK_RING;
#ifndef PFB_BULK_MINB
#define PFB_BULK_MINB 3
#endif  // block-fold slots (warps may drift this many items)

template <class T>
__device__ __forceinline__ T ld_volatile(const T* p) {
    return *reinterpret_cast<const volatile T*>(p);
}
template <class T>
__device__ __forceinline__ void st_volatile(T* p, T v) {
    *reinterpret_cast<volatile T*>(p) = v;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <class Ev>
__global__ void __launch_bounds__(kThreads, PFB_BULK_MINB) nll_prod_bulk_kernel(const __grid_constant__ NllArgs A) {
    constexpr int NC = Ev::NC;
    static_assert(kThreads == 32 * kBulkWarps, "one item per CTA");
    extern __shared__ __align__(128) double sbuf[];  // [8 warps][2 buffers][NC][512]
    __shared__ unsigned long long bar[kBulkWarps][2];
    __shared__ double xch[kRing][8][32];
    __shared__ int xbad[kRing][kBulkWarps];
    __shared__ unsigned int s_cnt[kRing];
    __shared__ int s_done[kRing];  // folds completed per slot
    __shared__ long long sacc[PFB_ACC_WORDS];
    __shared__ double s_tab[kTabN];
    __shared__ unsigned int s_last;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    const int w = tid >> 5;
    for (int i = tid; i < PFB_ACC_WORDS; i += blockDim.x) sacc[i] = 0;
    init_tab<Ev>(A, s_tab, tid);
    if (tid < kRing) {
        s_cnt[tid] = 0u;
        s_done[tid] = 0;
    }
    if (lane == 0) {
        mbar_init(&bar[w][0], 1);
        mbar_init(&bar[w][1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    const int64_t stride = gridDim.x;
    double* mybuf = sbuf + (int64_t)w * 2 * NC * kUnitEvents;
    // geometry of item `it` for this warp: first event offset, events present
    auto issue = [&](int64_t it, int b) {
        const bool tail = A.tail && it == 0;
        const int64_t bidx = tail ? A.nfull : it - (A.tail ? 1 : 0);
        const int n = tail ? A.tail : kBlock;
        int nw = n - kUnitEvents * w;
        nw = nw < 0 ? 0 : (nw > kUnitEvents ? kUnitEvents : nw);
        const unsigned bytes = 8u * (unsigned)(nw & ~1);  // bulk copies move 16 B multiples
        if (lane == 0) {
            mbar_arrive_expect_tx(&bar[w][b], bytes * NC);
            if (bytes) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    bulk_g2s(mybuf + (b * NC + c) * kUnitEvents,
                             A.col[c] + A.begin + bidx * (int64_t)kBlock + kUnitEvents * w, bytes, &bar[w][b]);
            }
        }
    };

    int64_t it = blockIdx.x;
    if (it < nitems) issue(it, 0);
    int j = 0;  // items processed by this CTA
    for (; it < nitems; it += stride, ++j) {
        const int b = j & 1;
        const bool has_next = it + stride < nitems;
        if (has_next) {
            // buffer b^1 was last read in item j-1 (program order, all lanes)
            __syncwarp();
            fence_proxy_async_smem();
            issue(it + stride, b ^ 1);
        }
        mbar_wait(&bar[w][b], (j >> 1) & 1);
        const double* xb = mybuf + b * NC * kUnitEvents;
        const bool tail = A.tail && it == 0;
        const int64_t bidx = tail ? A.nfull : it - (A.tail ? 1 : 0);
        Unit un;
        bool bad = false;
        if (!tail) {
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                double2 x[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    x[c] = *reinterpret_cast<const double2*>(xb + c * kUnitEvents + r * 64 + 2 * lane);
                prod_row<Ev, false>(A, x, 0, kBlock, un, bad, s_tab, (r & 1) != 0);
            }
        } else {
            const int n = A.tail;
            const int64_t gbase = A.begin + bidx * (int64_t)kBlock;
#pragma unroll 1
            for (int r = 0; r < 8; ++r) {
                const int le = r * 64 + 2 * lane;          // within the warp's 512
                const int e = kUnitEvents * w + le;        // within the block
                double2 x[NC];
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    if (e + 1 < n) {
                        x[c] = *reinterpret_cast<const double2*>(xb + c * kUnitEvents + le);
                    } else {  // odd last event (not bulk-copied) or a stand-in
                        const double v = __ldg(A.col[c] + gbase + (e < n ? e : 0));
                        x[c] = make_double2(v, v);
                    }
                }
                prod_row<Ev, true>(A, x, e, n, un, bad, s_tab);
            }
        }
        bad |= !unit_ok<Ev>(A, un);
        // No barrier: every warp posts its unit value into ring slot j % R and
        // the last of the 8 to arrive folds the block (warps never wait for
        // each other; a warp R items ahead waits for the slot to be folded).
        const int slot = j % kRing;
        if (lane == 0)
            while (ld_volatile(&s_done[slot]) < j / kRing) __nanosleep(32);
        __syncwarp();
        xch[slot][w][lane] = unit_value<Ev>(A, un);
        const unsigned anybad = __any_sync(0xffffffffu, bad);
        unsigned arrived = 0;
        if (lane == 0) {
            xbad[slot][w] = anybad ? 1 : 0;
            __threadfence_block();
            arrived = atomicAdd(&s_cnt[slot], 1u);
        }
        arrived = __shfl_sync(0xffffffffu, arrived, 0);
        if (arrived == kBulkWarps - 1) {
            __threadfence_block();
            bad = false;
#pragma unroll
            for (int q = 0; q < kBulkWarps; ++q) bad |= ld_volatile(&xbad[slot][q]) != 0;
            double bsum = 0.0;
            if (!bad) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = ld_volatile(&xch[slot][u][lane]);
                double T = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
#pragma unroll
                for (int off = 16; off >= 1; off /= 2) T = T + __shfl_down_sync(0xffffffffu, T, off);
                bsum = T;
            }
            __syncwarp();
            if (lane == 0) {
                if (bad) {
                    const unsigned long long fs = atomicAdd(A.fix_counter, 1ull);
                    A.fix_list[fs] = (A.block_base + bidx) * kMaxPts + A.fix_point;
                } else {
                    if (A.block_sums) A.block_sums[A.block_base + bidx] = bsum;
                    acc_add_shared(sacc, bsum);
                }
                s_cnt[slot] = 0u;
                __threadfence_block();
                st_volatile(&s_done[slot], j / kRing + 1);
            }
        }
    }
    finish_launch<false>(A, sacc, &s_last);
}

template <class Ev>
static cudaError_t launch_prod_bulk(const NllArgs& A, cudaStream_t stream, int sm_count) {
    constexpr int NC = Ev::NC;
    const size_t smem = (size_t)kBulkWarps * 2 * NC * kUnitEvents * sizeof(double);
    static int occ = 0;
    if (!occ) {
        cudaError_t e = cudaFuncSetAttribute(nll_prod_bulk_kernel<Ev>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nll_prod_bulk_kernel<Ev>, kThreads, smem);
        if (occ < 1) occ = 1;
    }
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    int64_t grid = (int64_t)sm_count * occ;
    if (grid > nitems) grid = nitems > 0 ? nitems : 1;
    nll_prod_bulk_kernel<Ev><<<(unsigned)grid, kThreads, smem, stream>>>(A);
    return cudaGetLastError();
}

template <int P, class Ev, bool PROD = true>
static cudaError_t launch_prod_one(const NllArgs& A, cudaStream_t stream, int sm_count) {
    static int occ = 0;
    if (!occ) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, nll_prod_kernel<P, Ev, PROD>, kThreads, 0);
        if (occ < 1) occ = 1;
    }
    constexpr int GROUPS = kThreads / (32 * P);
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    int64_t grid = (nitems + GROUPS - 1) / GROUPS;
#ifndef PFB_PROD_GRID_MULT
#define PFB_PROD_GRID_MULT 1
#endif
    const int64_t cap = (int64_t)sm_count * occ * PFB_PROD_GRID_MULT;
    if (grid > cap) grid = cap;
    if (grid < 1) grid = 1;
    nll_prod_kernel<P, Ev, PROD><<<(unsigned)grid, kThreads, 0, stream>>>(A);
    return cudaGetLastError();
}

// Block values do not depend on P (see the header), so A.warps is a pure
// tuning knob here too.
template <class Ev>
static cudaError_t launch_prod(const NllArgs& A, cudaStream_t stream, int sm_count) {
    // pipeline 1: per-warp bulk prefetch for single-column evaluators, the
    // TMA-fed unit kernel (producer warp + two consumer teams) for two-column
    // ones (Dalitz: 3% faster than the register window, measured);
    // 2: bulk prefetch for all; 3: the TMA unit kernel for all.  Three or more
    // columns: the register-window SIMT kernel only (the staging kernels are
    // sized for one or two 32 KB column blocks per stage)
    if constexpr (Ev::NC <= 2) {
        if (A.warps == 0 && (A.tma == 3 || (Ev::NC == 2 && A.tma == 1)))
            return launch_tma_unit<Ev, true>(A, stream, sm_count);
        if (A.warps == 0 && (A.tma == 2 || (Ev::NC == 1 && A.tma == 1)))
            return launch_prod_bulk<Ev>(A, stream, sm_count);
    }
    switch (A.warps) {
        case 1:
            return launch_prod_one<1, Ev>(A, stream, sm_count);
        case 2:
            return launch_prod_one<2, Ev>(A, stream, sm_count);
        case 4:
            return launch_prod_one<4, Ev>(A, stream, sm_count);
        default:
            return launch_prod_one<8, Ev>(A, stream, sm_count);
    }
}

// Log-domain unit sums (C2): the register-window SIMT kernel up to ~8 blocks
// per SM (no producer / mbarrier start-up: 1-2 us faster at 0.5-4M events,
// measured), the TMA unit kernel above (2-6% faster at 10-100M) -- the same
// canonical blocks, bitwise the same NLL.
template <class Ev>
static cudaError_t launch_unit_sum(const NllArgs& A, cudaStream_t stream, int sm_count) {
    const int64_t nitems = A.nfull + (A.tail ? 1 : 0);
    if (A.npts == 1 && (PFB_SUM_SIMT || nitems <= 8 * (int64_t)sm_count))
        return launch_prod_one<8, Ev, false>(A, stream, sm_count);
    return launch_tma_unit<Ev, false>(A, stream, sm_count);
}

#ifdef PFB_TRACE
inline cudaError_t read_trace(unsigned long long* host, int nblocks) {
    return cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * 16 * nblocks);
}
#endif

}  // namespace pfb
