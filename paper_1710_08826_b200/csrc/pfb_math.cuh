// pfb_math.cuh -- IEEE-exact arithmetic helpers and the literal Dalitz amplitude.
//
// The literal path reproduces the reference's numpy operation sequence, so it
// must never be contracted into FMAs: every operation is an explicit
// round-to-nearest intrinsic.
#pragma once

#include "pfb_internal.cuh"

namespace pfb {

// ---------------------------------------------------------------------------
// IEEE helpers: the literal path must not be contracted into FMAs, so that its
// operation sequence is the reference's (numpy evaluates without contraction).
__device__ __forceinline__ double Add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double Sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double Mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double Div(double a, double b) { return __ddiv_rn(a, b); }

// in_boundary_mask (dalitz.py:127-150) with the reference's exact IEEE
// operation sequence (bit-exact): s13 limits from the s12 invariant mass.
__device__ __forceinline__ bool in_boundary_exact(const GridConsts& g, double s12, double s13) {
    const double rs = __dsqrt_rn(s12);
    const double two_rs = Mul(2.0, rs);
    const double e1 = Div(Sub(Add(s12, g.m1sq), g.m2sq), two_rs);
    const double e3 = Div(Sub(Sub(g.M2, s12), g.m3sq), two_rs);
    const double p1 = __dsqrt_rn(Sub(Mul(e1, e1), g.m1sq));
    const double p3 = __dsqrt_rn(Sub(Mul(e3, e3), g.m3sq));
    const double es = Add(e1, e3);
    const double esum = Mul(es, es);
    const double pp = Add(p1, p3), pm = Sub(p1, p3);
    const double lo = Sub(esum, Mul(pp, pp));
    const double hi = Sub(esum, Mul(pm, pm));
    // NaN (outside the s12 band) compares false, as numpy does.
    return (s12 >= g.lo12) && (s12 <= g.hi12) && (s13 >= lo) && (s13 <= hi);
}

// ---------------------------------------------------------------------------
// Dalitz amplitude of one term with the reference's exact operation sequence
// (dalitz.py:162-197): BW = 1/(m^2 - s - i m Gamma) by numpy's Smith division,
// times the spin-1 Zemach factor as a complex-by-real product.
__device__ __forceinline__ double2 dalitz_amp_literal(const DalDesc& D, const DalTerm& T,
                                                      double s12, double s13) {
    const double s23 = Sub(Sub(D.mss, s12), s13);
    const double s = T.pair == 12 ? s12 : (T.pair == 13 ? s13 : s23);
    const double in2r = Sub(T.m2, s);
    const double in2i = Sub(0.0, T.mg);
    double br, bi;
    if (fabs(in2r) >= fabs(in2i)) {
        if (in2r == 0.0 && in2i == 0.0) {
            br = Div(1.0, fabs(in2r));
            bi = Div(0.0, fabs(in2r));
        } else {
            const double rat = Div(in2i, in2r);
            const double scl = Div(1.0, Add(in2r, Mul(in2i, rat)));
            br = Mul(Add(1.0, Mul(0.0, rat)), scl);
            bi = Mul(Sub(0.0, Mul(1.0, rat)), scl);
        }
    } else {
        const double rat = Div(in2r, in2i);
        const double scl = Div(1.0, Add(in2i, Mul(in2r, rat)));
        br = Mul(Add(Mul(1.0, rat), 0.0), scl);
        bi = Mul(Sub(Mul(0.0, rat), 1.0), scl);
    }
    if (T.spin == 1) {
        double z;
        if (T.pair == 12)
            z = Add(Sub(s13, s23), Div(D.zc12, s12));
        else if (T.pair == 13)
            z = Add(Sub(s12, s23), Div(D.zc13, s13));
        else
            z = Add(Sub(s12, s13), Div(D.zc23, s23));
        const double nr = Sub(Mul(br, z), Mul(bi, 0.0));
        const double ni = Add(Mul(br, 0.0), Mul(bi, z));
        br = nr;
        bi = ni;
    }
    return make_double2(br, bi);
}

}  // namespace pfb
