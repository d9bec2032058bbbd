// Double-double arithmetic (a value is hi + lo, |lo| <= ulp(hi)/2), ~106-bit significand.
// Error-free transformations with explicit round-to-nearest intrinsics so that nvcc's
// FMA contraction cannot break them.  Used for the per-cell local eliminations
// (kappa(S_K) ~ 1e8 at 2D n = 1024; fp64 Gauss-Jordan would lose 8 digits of G_K).
#pragma once

struct dd {
    double hi, lo;
};

__device__ __forceinline__ dd dd_of(double a) { return {a, 0.0}; }

__device__ __forceinline__ dd two_sum(double a, double b) {
    double s = __dadd_rn(a, b);
    double bb = __dsub_rn(s, a);
    double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
    return {s, e};
}

__device__ __forceinline__ dd fast_two_sum(double a, double b) {  // |a| >= |b|
    double s = __dadd_rn(a, b);
    double e = __dsub_rn(b, __dsub_rn(s, a));
    return {s, e};
}

__device__ __forceinline__ dd two_prod(double a, double b) {
    double p = __dmul_rn(a, b);
    double e = __fma_rn(a, b, -p);
    return {p, e};
}

__device__ __forceinline__ dd operator+(dd a, dd b) {
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    double c = __dadd_rn(s.lo, t.hi);
    dd v = fast_two_sum(s.hi, c);
    double w = __dadd_rn(t.lo, v.lo);
    return fast_two_sum(v.hi, w);
}
__device__ __forceinline__ dd operator-(dd a) { return {-a.hi, -a.lo}; }
__device__ __forceinline__ dd operator-(dd a, dd b) { return a + (-b); }
__device__ __forceinline__ dd operator+(dd a, double b) {
    dd s = two_sum(a.hi, b);
    double c = __dadd_rn(s.lo, a.lo);
    return fast_two_sum(s.hi, c);
}

__device__ __forceinline__ dd operator*(dd a, dd b) {
    dd p = two_prod(a.hi, b.hi);
    double t = __fma_rn(a.hi, b.lo, __dmul_rn(a.lo, b.hi));
    t = __dadd_rn(p.lo, t);
    return fast_two_sum(p.hi, t);
}
__device__ __forceinline__ dd operator*(dd a, double b) {
    dd p = two_prod(a.hi, b);
    double t = __fma_rn(a.lo, b, p.lo);
    return fast_two_sum(p.hi, t);
}

__device__ __forceinline__ dd operator/(dd a, dd b) {
    double q1 = __ddiv_rn(a.hi, b.hi);
    dd r = a - b * q1;
    double q2 = __ddiv_rn(r.hi, b.hi);
    r = r - b * q2;
    double q3 = __ddiv_rn(r.hi, b.hi);
    dd q = fast_two_sum(q1, q2);
    return q + q3;
}
__device__ __forceinline__ dd operator/(dd a, double b) { return a / dd_of(b); }

__device__ __forceinline__ double dd_round(dd a) { return a.hi; }  // normalised: hi = fl(hi + lo)
__device__ __forceinline__ double dd_abs_hi(dd a) { return fabs(a.hi); }
