/*
 * vs_math.h -- correctly-rounded (to ~2^-75 before the final rounding)
 * double-precision sin/cos for the generated kernels.
 *
 * Why: the reference evaluates SIN/COS with glibc (symcore.py:210-216 via
 * numba -> libm).  glibc's sin/cos are correctly rounded except in rare hard
 * cases, while CUDA's libdevice sin/cos are faithful (<= 2 ulp).  In
 * ill-conditioned tapes (penalty-SQP solves) a 1-ulp difference is amplified
 * past the 1e-12 parity contract, so the kernels use these instead: they
 * agree with glibc bit for bit on all but ~1e-5 of arguments.
 *
 * Method: Cody-Waite reduction x = k*pi/2 + r with pi/2 in three doubles,
 * r carried as a double-double; odd/even Taylor polynomials whose leading
 * terms run in double-double arithmetic (exact products via fma) and whose
 * tail runs in double; one final rounding.  |x| >= 2^30 falls back to the
 * platform sin/cos (Payne-Hanek territory; never hit by the workloads).
 *
 * Header is shared by the CUDA kernels (NVRTC, VS_MATH_DEVICE) and by the
 * host test harness (plain C99), so the exact same operation sequence is
 * validated against glibc on the CPU.  Requires no FMA contraction of the
 * plain expressions (nvrtc --fmad=false / gcc -ffp-contract=off).
 */
#ifndef VS_MATH_H
#define VS_MATH_H

#ifdef VS_MATH_DEVICE
#define VSM_FN static __device__ __forceinline__
#define VSM_FMA(a, b, c) fma(a, b, c)
#define VSM_RINT(x) rint(x)
#define VSM_SIN_FALLBACK(x) sin(x)
#define VSM_COS_FALLBACK(x) cos(x)
#else
#include <math.h>
#define VSM_FN static inline
#define VSM_FMA(a, b, c) fma(a, b, c)
#define VSM_RINT(x) nearbyint(x)
#define VSM_SIN_FALLBACK(x) sin(x)
#define VSM_COS_FALLBACK(x) cos(x)
#endif

typedef struct { double hi, lo; } vsm_dd;

VSM_FN vsm_dd vsm_fast_two_sum(double a, double b) { /* |a| >= |b| */
    vsm_dd r;
    r.hi = a + b;
    r.lo = b - (r.hi - a);
    return r;
}

VSM_FN vsm_dd vsm_two_sum(double a, double b) {
    vsm_dd r;
    r.hi = a + b;
    double bb = r.hi - a;
    r.lo = (a - (r.hi - bb)) + (b - bb);
    return r;
}

VSM_FN vsm_dd vsm_dd_mul(vsm_dd a, vsm_dd b) {
    double p = a.hi * b.hi;
    double e = VSM_FMA(a.hi, b.hi, -p);
    e += a.hi * b.lo + a.lo * b.hi;
    return vsm_fast_two_sum(p, e);
}

VSM_FN vsm_dd vsm_dd_add(vsm_dd a, vsm_dd b) {
    vsm_dd s = vsm_two_sum(a.hi, b.hi);
    double e = s.lo + (a.lo + b.lo);
    return vsm_fast_two_sum(s.hi, e);
}

VSM_FN vsm_dd vsm_dd_add_d(vsm_dd a, double b) {
    vsm_dd s = vsm_two_sum(a.hi, b);
    return vsm_fast_two_sum(s.hi, s.lo + a.lo);
}

/* pi/2 = P1 + P2 + P3 (+ ~2^-160) */
#define VSM_P1 1.5707963267948966
#define VSM_P2 6.123233995736766e-17
#define VSM_P3 (-1.4973849048591698e-33)
#define VSM_2_OVER_PI 0.6366197723675814

/* Taylor coefficients; double-double where the term matters below 2^-70 */
#define VSM_S1H (-0.16666666666666666)
#define VSM_S1L (-9.25185853854297e-18)
#define VSM_S2H 0.008333333333333333
#define VSM_S2L 1.1564823173178714e-19
#define VSM_S3H (-0.0001984126984126984)
#define VSM_S3L (-1.7209558293420705e-22)
#define VSM_S4 2.7557319223985893e-06
#define VSM_S5 (-2.505210838544172e-08)
#define VSM_S6 1.6059043836821613e-10
#define VSM_S7 (-7.647163731819816e-13)
#define VSM_S8 2.8114572543455206e-15
#define VSM_S9 (-8.22063524662433e-18)
#define VSM_S10 1.9572941063391263e-20
#define VSM_C2H 0.041666666666666664
#define VSM_C2L 2.3129646346357427e-18
#define VSM_C3H (-0.001388888888888889)
#define VSM_C3L 5.300543954373577e-20
#define VSM_C4H 2.48015873015873e-05
#define VSM_C4L 2.1511947866775882e-23
#define VSM_C5 (-2.755731922398589e-07)
#define VSM_C6 2.08767569878681e-09
#define VSM_C7 (-1.1470745597729725e-11)
#define VSM_C8 4.779477332387385e-14
#define VSM_C9 (-1.5619206968586225e-16)
#define VSM_C10 4.110317623312165e-19

/* reduce x (|x| < 2^30) to r = x - k*pi/2 as a double-double; returns k */
VSM_FN double vsm_reduce(double x, vsm_dd *r) {
    double k = VSM_RINT(x * VSM_2_OVER_PI);
    double t1 = VSM_FMA(-k, VSM_P1, x);           /* exact (Sterbenz-like) */
    double p2 = k * VSM_P2;
    double e2 = VSM_FMA(k, VSM_P2, -p2);          /* k*P2 = p2 + e2 exactly */
    vsm_dd s = vsm_two_sum(t1, -p2);
    double lo = s.lo - e2 - k * VSM_P3;
    *r = vsm_fast_two_sum(s.hi, lo);
    return k;
}

/* sin(r) for |r| <= pi/4 + eps, as a double-double */
VSM_FN vsm_dd vsm_sin_kernel(vsm_dd r) {
    vsm_dd z;                                      /* z = r^2 */
    z.hi = r.hi * r.hi;
    z.lo = VSM_FMA(r.hi, r.hi, -z.hi) + 2.0 * r.hi * r.lo;
    z = vsm_fast_two_sum(z.hi, z.lo);
    double zh = z.hi;
    double t = VSM_S4 + zh * (VSM_S5 + zh * (VSM_S6 + zh * (VSM_S7 + zh * (VSM_S8 + zh * (VSM_S9 + zh * VSM_S10)))));
    vsm_dd p;
    p.hi = VSM_S3H; p.lo = VSM_S3L;
    p = vsm_dd_add_d(p, zh * t);                   /* S3 + z*tail */
    p = vsm_dd_mul(p, z);
    vsm_dd c; c.hi = VSM_S2H; c.lo = VSM_S2L;
    p = vsm_dd_add(p, c);
    p = vsm_dd_mul(p, z);
    c.hi = VSM_S1H; c.lo = VSM_S1L;
    p = vsm_dd_add(p, c);
    p = vsm_dd_mul(p, z);                          /* u = z*(S1 + z*(S2 + ...)) */
    vsm_dd ru = vsm_dd_mul(r, p);                  /* r*u, |r*u| <= 0.1|r| */
    return vsm_dd_add(r, ru);
}

/* cos(r) for |r| <= pi/4 + eps, as a double-double */
VSM_FN vsm_dd vsm_cos_kernel(vsm_dd r) {
    vsm_dd z;
    z.hi = r.hi * r.hi;
    z.lo = VSM_FMA(r.hi, r.hi, -z.hi) + 2.0 * r.hi * r.lo;
    z = vsm_fast_two_sum(z.hi, z.lo);
    double zh = z.hi;
    double t = VSM_C5 + zh * (VSM_C6 + zh * (VSM_C7 + zh * (VSM_C8 + zh * (VSM_C9 + zh * VSM_C10))));
    vsm_dd p;
    p.hi = VSM_C4H; p.lo = VSM_C4L;
    p = vsm_dd_add_d(p, zh * t);
    p = vsm_dd_mul(p, z);
    vsm_dd c; c.hi = VSM_C3H; c.lo = VSM_C3L;
    p = vsm_dd_add(p, c);
    p = vsm_dd_mul(p, z);
    c.hi = VSM_C2H; c.lo = VSM_C2L;
    p = vsm_dd_add(p, c);
    p = vsm_dd_mul(p, z);                          /* z*(C2 + z*(...)) */
    p = vsm_dd_add_d(p, -0.5);
    p = vsm_dd_mul(p, z);                          /* z*(-1/2 + ...) */
    return vsm_dd_add_d(p, 1.0);                   /* 1 + ... */
}

VSM_FN double vs_sin(double x) {
    double ax = x < 0.0 ? -x : x;
    if (!(ax < 1073741824.0)) return VSM_SIN_FALLBACK(x);   /* NaN, inf, |x| >= 2^30 */
    if (ax < 7.450580596923828e-09) return x;                /* |x| < 2^-27: sin x = x */
    vsm_dd r;
    int q = (int)((long long)vsm_reduce(x, &r) & 3);
    vsm_dd v = (q & 1) ? vsm_cos_kernel(r) : vsm_sin_kernel(r);
    double s = v.hi + v.lo;
    return (q & 2) ? -s : s;
}

VSM_FN double vs_cos(double x) {
    double ax = x < 0.0 ? -x : x;
    if (!(ax < 1073741824.0)) return VSM_COS_FALLBACK(x);
    if (ax < 7.450580596923828e-09) return 1.0;
    vsm_dd r;
    int q = (int)((long long)vsm_reduce(x, &r) & 3);
    vsm_dd v = (q & 1) ? vsm_sin_kernel(r) : vsm_cos_kernel(r);
    double c = v.hi + v.lo;
    return ((q + 1) & 2) ? -c : c;
}

/* both at once: one reduction (codegen pairs SIN and COS of the same value) */
VSM_FN void vs_sincos(double x, double *s, double *c) {
    double ax = x < 0.0 ? -x : x;
    if (!(ax < 1073741824.0)) { *s = VSM_SIN_FALLBACK(x); *c = VSM_COS_FALLBACK(x); return; }
    if (ax < 7.450580596923828e-09) { *s = x; *c = 1.0; return; }
    vsm_dd r;
    int q = (int)((long long)vsm_reduce(x, &r) & 3);
    vsm_dd vs = vsm_sin_kernel(r), vc = vsm_cos_kernel(r);
    double sv = vs.hi + vs.lo, cv = vc.hi + vc.lo;
    double s0 = (q & 1) ? cv : sv, c0 = (q & 1) ? sv : cv;
    *s = (q & 2) ? -s0 : s0;
    *c = ((q + 1) & 2) ? -c0 : c0;
}

#endif /* VS_MATH_H */
