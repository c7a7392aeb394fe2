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


/* ---- fast path (Ziv): table of sin/cos(i/64), i = -52..52, as double-doubles
 * {sin hi, sin lo, cos hi, cos lo}; r = a + t with a = i/64, |t| <= 1/128 + 2^-60:
 *   sin(a+t) = SA + SA*(cos t - 1) + CA*sin t,  cos(a+t) = CA + CA*(cos t - 1) - SA*sin t
 * with the CA*t / SA*t products exact (fma) and short Taylor tails in double.
 * Relative error of (yh + yl) before rounding measured <= 2^-65.2 (8e6 arguments) (analysis in DESIGN.md 4.5,
 * measured by tests/test_vs_math.py); the result is returned only when rounding
 * yh + yl +- VSM_FAST_EPS*|yh| gives one double, else the 2^-75 path above runs. */
#define VSM_FAST_EPS 0x1p-63
#define VSM_F_S1 (-0x1.5555555555555p-3)
#define VSM_F_S2 0x1.1111111111111p-7
#define VSM_F_S3 (-0x1.a01a01a01a01ap-13)
#define VSM_F_C2 0x1.5555555555555p-5
#define VSM_F_C3 (-0x1.6c16c16c16c17p-10)
#ifdef VS_MATH_DEVICE
static __device__ __align__(16) const double vsm_tab[420] = {
    -0x1.73b7680dea578p-1, 0x1.2248306dc12a2p-56, 0x1.6018526f563dfp-1, 0x1.46ca5e0e432d0p-55,
    -0x1.6e2b77c40bde1p-1, 0x1.0e729857fad53p-56, 0x1.65dc1fdeb8cbap-1, -0x1.97c1b47337c77p-58,
    -0x1.6888a4e134b2fp-1, 0x1.6b7d37644d5e6p-55, 0x1.6b898fa9efb5dp-1, 0x1.15ac786ccf4b2p-56,
    -0x1.62cf49921ac79p-1, 0x1.edd9855b6241ap-55, 0x1.712046fa77678p-1, 0x1.425b0a5029c81p-55,
    -0x1.5cffc16bf8f0dp-1, -0x1.96cb370eb578ap-55, 0x1.769fec655211fp-1, -0x1.827d5cf8c68c5p-57,
    -0x1.571a6966d59b3p-1, -0x1.c843b4d0fb197p-58, 0x1.7c0827f09e54fp-1, -0x1.c73d6d72aee68p-57,
    -0x1.511f9fd7b351cp-1, 0x1.5c0e861c48831p-55, 0x1.8158a31916d5dp-1, -0x1.de8b90b8228dep-57,
    -0x1.4b0fc46aab761p-1, -0x1.0da05738cc59cp-61, 0x1.869108d77a6c6p-1, 0x1.338ffe2bfe9ddp-56,
    -0x1.44eb381cf386bp-1, 0x1.3ed6c1e6a5505p-55, 0x1.8bb105a5dc900p-1, 0x1.863e03e9474c1p-55,
    -0x1.3eb25d36cd53ap-1, 0x1.be570e1570fc0p-58, 0x1.90b84784ddaf7p-1, -0x1.0feb10ab93b87p-56,
    -0x1.386597456282bp-1, 0x1.10fada93b07a8p-56, 0x1.95a67e00cb1fdp-1, -0x1.0befda21f862dp-55,
    -0x1.32054b148bc4fp-1, -0x1.f6b42095a135bp-55, 0x1.9a7b5a36a6514p-1, 0x1.722cfcc9fa7a9p-55,
    -0x1.2b91dea88421ep-1, 0x1.fa371db216ab0p-55, 0x1.9f368ed912f85p-1, -0x1.1d200c5791606p-55,
    -0x1.250bb93788bbbp-1, -0x1.ea3d02457bccep-56, 0x1.a3d7d0352bdcfp-1, -0x1.68dbaeca19669p-55,
    -0x1.1e7343236574cp-1, -0x1.22a3fa4f41d5ap-56, 0x1.a85ed4373e02dp-1, 0x1.9be06385ec792p-57,
    -0x1.17c8e5f2eedb0p-1, -0x1.35e57102e2488p-57, 0x1.accb526f69de5p-1, 0x1.8fb6a8dd6b6ccp-55,
    -0x1.110d0c4b69c3bp-1, -0x1.d918998809981p-55, 0x1.b11d04162a4c6p-1, 0x1.1dd561efbc0c2p-56,
    -0x1.0a4021e9e1001p-1, 0x1.6f643a13914f6p-55, 0x1.b553a410c104ep-1, 0x1.8ff7947027a15p-58,
    -0x1.0362939c69955p-1, 0x1.2d8cd78397b01p-55, 0x1.b96eeef58840ep-1, 0x1.45a3cc78fade0p-58,
    -0x1.f8e99e76abc97p-2, -0x1.9d950af2d00a3p-58, 0x1.bd6ea310294f5p-1, 0x1.31bbcc88c109dp-56,
    -0x1.eaee8744b05f0p-2, 0x1.789b43c9b027dp-58, 0x1.c1528065b7d50p-1, -0x1.892111312e828p-55,
    -0x1.dcd4c15329c9ap-2, -0x1.0d4c6e171fd9ap-56, 0x1.c51a48b8b175ep-1, -0x1.1bbb43b9aa880p-57,
    -0x1.ce9d2e3d4a51fp-2, 0x1.2fc8a12dae298p-57, 0x1.c8c5bf8ce1a84p-1, 0x1.ab3d1a1590123p-56,
    -0x1.c048b17b140a3p-2, -0x1.19fe6757e9fa7p-57, 0x1.cc54aa2b2972ep-1, 0x1.4ee162ba83a98p-57,
    -0x1.b1d8305321617p-2, 0x1.ae242cb99f519p-56, 0x1.cfc6cfa52ad9fp-1, 0x1.8b5b5508f2a0dp-55,
    -0x1.a34c91cc50ccap-2, 0x1.a310e3b50cecdp-58, 0x1.d31bf8d8d7c06p-1, 0x1.e60dd3089cbddp-56,
    -0x1.94a6be9f546c5p-2, 0x1.69ce13e683f58p-56, 0x1.d653f073e4040p-1, -0x1.76236434bec37p-55,
    -0x1.85e7a12826949p-2, -0x1.8a40e9b5face0p-56, 0x1.d96e82f71a9dcp-1, 0x1.ff61bd5d2039dp-55,
    -0x1.7710255764214p-2, 0x1.6ead7314bb6cep-57, 0x1.dc6b7eb995912p-1, 0x1.4b364776dcd35p-58,
    -0x1.682138a38d7f7p-2, 0x1.d889202444aadp-56, 0x1.df4ab3ebd875ep-1, -0x1.e2d8a7e6736c4p-55,
    -0x1.591bc9fa2f597p-2, -0x1.7c74bac3fe0cbp-57, 0x1.e20bf49acd6c1p-1, -0x1.660aec7ef636bp-58,
    -0x1.4a00c9b0f3d20p-2, -0x1.823ba6bb08eadp-56, 0x1.e4af14b2a449cp-1, -0x1.68ca02e8a6833p-55,
    -0x1.3ad129769d3d8p-2, -0x1.03d550487839ap-63, 0x1.e733ea0193d40p-1, -0x1.6428b3546ce13p-55,
    -0x1.2b8ddc43eb49fp-2, -0x1.1553899f2d807p-57, 0x1.e99a4c3a7cd83p-1, -0x1.2264b1bc53ce8p-55,
    -0x1.1c37d64c6b876p-2, -0x1.46076fe0dcff4p-56, 0x1.ebe214f76efa8p-1, -0x1.02f9f12ba543ep-55,
    -0x1.0cd00cef36436p-2, 0x1.9fb0a0c93e2b4p-56, 0x1.ee0b1fbc0f11cp-1, -0x1.bfd2380bbc3b1p-59,
    -0x1.faaeed4f31577p-3, 0x1.15d88508e32b8p-57, 0x1.f01549f7deea1p-1, 0x1.d3c1e99e5cafdp-55,
    -0x1.db9e15fb5a5d0p-3, 0x1.32e20d6cc6fc2p-57, 0x1.f20073086649fp-1, 0x1.b940416c1984bp-56,
    -0x1.bc6f84edc6199p-3, -0x1.9c1a56a7b0cabp-57, 0x1.f3cc7c3b3d16ep-1, -0x1.21a3ad28a3494p-57,
    -0x1.9d252d0cec312p-3, -0x1.9c43d80b1137dp-58, 0x1.f57948cff6797p-1, 0x1.e3a0d3e03b1d4p-57,
    -0x1.7dc102fbaf2b5p-3, -0x1.5ab50e23c97c3p-59, 0x1.f706bdf9ece1cp-1, -0x1.698c80c36dcb4p-55,
    -0x1.5e44fcfa126f3p-3, 0x1.6f443063f89b6p-57, 0x1.f874c2e1eecf6p-1, -0x1.c6514e1332b16p-55,
    -0x1.3eb312c5d66cbp-3, -0x1.47d666b66cb91p-57, 0x1.f9c340a7cc428p-1, 0x1.c5b6b063b7462p-55,
    -0x1.1f0d3d7afceafp-3, 0x1.6ef95099769a5p-57, 0x1.faf22263c4bd3p-1, -0x1.52ace133a2769p-58,
    -0x1.feaaeee86ee36p-4, 0x1.afcb2bcc6f03bp-59, 0x1.fc015527d5bd3p-1, 0x1.b68f35094efb8p-55,
    -0x1.bf1b78568391dp-4, -0x1.e91841dea4cc8p-58, 0x1.fcf0c800e99b1p-1, 0x1.ea3d786d186acp-57,
    -0x1.7f701032550e4p-4, -0x1.afc2d1800501ap-60, 0x1.fdc06bf7e6b9bp-1, 0x1.31902b535f8dbp-55,
    -0x1.3facb12d1755bp-4, 0x1.921915299468bp-58, 0x1.fe7034129ef6fp-1, -0x1.cbf4337c96f97p-57,
    -0x1.ffaaaeeed4edbp-5, 0x1.2d16d32684b69p-59, 0x1.ff0015549f4d3p-1, 0x1.328387b99426fp-55,
    -0x1.7fdc01032fba9p-5, 0x1.599bdf46e997ap-59, 0x1.ff7006bfdf99fp-1, -0x1.8b3b560648d5fp-56,
    -0x1.ffeaaaeeee86fp-6, 0x1.cd406fb224ae2p-60, 0x1.ffc00155527d3p-1, -0x1.3b54492d89b5bp-55,
    -0x1.fffaaaaeeeed5p-7, 0x1.2ab639a9f0776p-63, 0x1.fff000155549fp-1, 0x1.28a28a03a5ef3p-55,
    0.0, 0.0, 0x1.0000000000000p+0, 0.0,
    0x1.fffaaaaeeeed5p-7, -0x1.2ab639a9f0776p-63, 0x1.fff000155549fp-1, 0x1.28a28a03a5ef3p-55,
    0x1.ffeaaaeeee86fp-6, -0x1.cd406fb224ae2p-60, 0x1.ffc00155527d3p-1, -0x1.3b54492d89b5bp-55,
    0x1.7fdc01032fba9p-5, -0x1.599bdf46e997ap-59, 0x1.ff7006bfdf99fp-1, -0x1.8b3b560648d5fp-56,
    0x1.ffaaaeeed4edbp-5, -0x1.2d16d32684b69p-59, 0x1.ff0015549f4d3p-1, 0x1.328387b99426fp-55,
    0x1.3facb12d1755bp-4, -0x1.921915299468bp-58, 0x1.fe7034129ef6fp-1, -0x1.cbf4337c96f97p-57,
    0x1.7f701032550e4p-4, 0x1.afc2d1800501ap-60, 0x1.fdc06bf7e6b9bp-1, 0x1.31902b535f8dbp-55,
    0x1.bf1b78568391dp-4, 0x1.e91841dea4cc8p-58, 0x1.fcf0c800e99b1p-1, 0x1.ea3d786d186acp-57,
    0x1.feaaeee86ee36p-4, -0x1.afcb2bcc6f03bp-59, 0x1.fc015527d5bd3p-1, 0x1.b68f35094efb8p-55,
    0x1.1f0d3d7afceafp-3, -0x1.6ef95099769a5p-57, 0x1.faf22263c4bd3p-1, -0x1.52ace133a2769p-58,
    0x1.3eb312c5d66cbp-3, 0x1.47d666b66cb91p-57, 0x1.f9c340a7cc428p-1, 0x1.c5b6b063b7462p-55,
    0x1.5e44fcfa126f3p-3, -0x1.6f443063f89b6p-57, 0x1.f874c2e1eecf6p-1, -0x1.c6514e1332b16p-55,
    0x1.7dc102fbaf2b5p-3, 0x1.5ab50e23c97c3p-59, 0x1.f706bdf9ece1cp-1, -0x1.698c80c36dcb4p-55,
    0x1.9d252d0cec312p-3, 0x1.9c43d80b1137dp-58, 0x1.f57948cff6797p-1, 0x1.e3a0d3e03b1d4p-57,
    0x1.bc6f84edc6199p-3, 0x1.9c1a56a7b0cabp-57, 0x1.f3cc7c3b3d16ep-1, -0x1.21a3ad28a3494p-57,
    0x1.db9e15fb5a5d0p-3, -0x1.32e20d6cc6fc2p-57, 0x1.f20073086649fp-1, 0x1.b940416c1984bp-56,
    0x1.faaeed4f31577p-3, -0x1.15d88508e32b8p-57, 0x1.f01549f7deea1p-1, 0x1.d3c1e99e5cafdp-55,
    0x1.0cd00cef36436p-2, -0x1.9fb0a0c93e2b4p-56, 0x1.ee0b1fbc0f11cp-1, -0x1.bfd2380bbc3b1p-59,
    0x1.1c37d64c6b876p-2, 0x1.46076fe0dcff4p-56, 0x1.ebe214f76efa8p-1, -0x1.02f9f12ba543ep-55,
    0x1.2b8ddc43eb49fp-2, 0x1.1553899f2d807p-57, 0x1.e99a4c3a7cd83p-1, -0x1.2264b1bc53ce8p-55,
    0x1.3ad129769d3d8p-2, 0x1.03d550487839ap-63, 0x1.e733ea0193d40p-1, -0x1.6428b3546ce13p-55,
    0x1.4a00c9b0f3d20p-2, 0x1.823ba6bb08eadp-56, 0x1.e4af14b2a449cp-1, -0x1.68ca02e8a6833p-55,
    0x1.591bc9fa2f597p-2, 0x1.7c74bac3fe0cbp-57, 0x1.e20bf49acd6c1p-1, -0x1.660aec7ef636bp-58,
    0x1.682138a38d7f7p-2, -0x1.d889202444aadp-56, 0x1.df4ab3ebd875ep-1, -0x1.e2d8a7e6736c4p-55,
    0x1.7710255764214p-2, -0x1.6ead7314bb6cep-57, 0x1.dc6b7eb995912p-1, 0x1.4b364776dcd35p-58,
    0x1.85e7a12826949p-2, 0x1.8a40e9b5face0p-56, 0x1.d96e82f71a9dcp-1, 0x1.ff61bd5d2039dp-55,
    0x1.94a6be9f546c5p-2, -0x1.69ce13e683f58p-56, 0x1.d653f073e4040p-1, -0x1.76236434bec37p-55,
    0x1.a34c91cc50ccap-2, -0x1.a310e3b50cecdp-58, 0x1.d31bf8d8d7c06p-1, 0x1.e60dd3089cbddp-56,
    0x1.b1d8305321617p-2, -0x1.ae242cb99f519p-56, 0x1.cfc6cfa52ad9fp-1, 0x1.8b5b5508f2a0dp-55,
    0x1.c048b17b140a3p-2, 0x1.19fe6757e9fa7p-57, 0x1.cc54aa2b2972ep-1, 0x1.4ee162ba83a98p-57,
    0x1.ce9d2e3d4a51fp-2, -0x1.2fc8a12dae298p-57, 0x1.c8c5bf8ce1a84p-1, 0x1.ab3d1a1590123p-56,
    0x1.dcd4c15329c9ap-2, 0x1.0d4c6e171fd9ap-56, 0x1.c51a48b8b175ep-1, -0x1.1bbb43b9aa880p-57,
    0x1.eaee8744b05f0p-2, -0x1.789b43c9b027dp-58, 0x1.c1528065b7d50p-1, -0x1.892111312e828p-55,
    0x1.f8e99e76abc97p-2, 0x1.9d950af2d00a3p-58, 0x1.bd6ea310294f5p-1, 0x1.31bbcc88c109dp-56,
    0x1.0362939c69955p-1, -0x1.2d8cd78397b01p-55, 0x1.b96eeef58840ep-1, 0x1.45a3cc78fade0p-58,
    0x1.0a4021e9e1001p-1, -0x1.6f643a13914f6p-55, 0x1.b553a410c104ep-1, 0x1.8ff7947027a15p-58,
    0x1.110d0c4b69c3bp-1, 0x1.d918998809981p-55, 0x1.b11d04162a4c6p-1, 0x1.1dd561efbc0c2p-56,
    0x1.17c8e5f2eedb0p-1, 0x1.35e57102e2488p-57, 0x1.accb526f69de5p-1, 0x1.8fb6a8dd6b6ccp-55,
    0x1.1e7343236574cp-1, 0x1.22a3fa4f41d5ap-56, 0x1.a85ed4373e02dp-1, 0x1.9be06385ec792p-57,
    0x1.250bb93788bbbp-1, 0x1.ea3d02457bccep-56, 0x1.a3d7d0352bdcfp-1, -0x1.68dbaeca19669p-55,
    0x1.2b91dea88421ep-1, -0x1.fa371db216ab0p-55, 0x1.9f368ed912f85p-1, -0x1.1d200c5791606p-55,
    0x1.32054b148bc4fp-1, 0x1.f6b42095a135bp-55, 0x1.9a7b5a36a6514p-1, 0x1.722cfcc9fa7a9p-55,
    0x1.386597456282bp-1, -0x1.10fada93b07a8p-56, 0x1.95a67e00cb1fdp-1, -0x1.0befda21f862dp-55,
    0x1.3eb25d36cd53ap-1, -0x1.be570e1570fc0p-58, 0x1.90b84784ddaf7p-1, -0x1.0feb10ab93b87p-56,
    0x1.44eb381cf386bp-1, -0x1.3ed6c1e6a5505p-55, 0x1.8bb105a5dc900p-1, 0x1.863e03e9474c1p-55,
    0x1.4b0fc46aab761p-1, 0x1.0da05738cc59cp-61, 0x1.869108d77a6c6p-1, 0x1.338ffe2bfe9ddp-56,
    0x1.511f9fd7b351cp-1, -0x1.5c0e861c48831p-55, 0x1.8158a31916d5dp-1, -0x1.de8b90b8228dep-57,
    0x1.571a6966d59b3p-1, 0x1.c843b4d0fb197p-58, 0x1.7c0827f09e54fp-1, -0x1.c73d6d72aee68p-57,
    0x1.5cffc16bf8f0dp-1, 0x1.96cb370eb578ap-55, 0x1.769fec655211fp-1, -0x1.827d5cf8c68c5p-57,
    0x1.62cf49921ac79p-1, -0x1.edd9855b6241ap-55, 0x1.712046fa77678p-1, 0x1.425b0a5029c81p-55,
    0x1.6888a4e134b2fp-1, -0x1.6b7d37644d5e6p-55, 0x1.6b898fa9efb5dp-1, 0x1.15ac786ccf4b2p-56,
    0x1.6e2b77c40bde1p-1, -0x1.0e729857fad53p-56, 0x1.65dc1fdeb8cbap-1, -0x1.97c1b47337c77p-58,
    0x1.73b7680dea578p-1, -0x1.2248306dc12a2p-56, 0x1.6018526f563dfp-1, 0x1.46ca5e0e432d0p-55,
};
#define VSM_TAB(i, sh, sl, ch, cl) do { \
    const double2 vsm_s_ = __ldg(reinterpret_cast<const double2*>(vsm_tab) + 2 * (i)); \
    const double2 vsm_c_ = __ldg(reinterpret_cast<const double2*>(vsm_tab) + 2 * (i) + 1); \
    sh = vsm_s_.x; sl = vsm_s_.y; ch = vsm_c_.x; cl = vsm_c_.y; } while (0)
#else
static const double vsm_tab[420] = {
    -0x1.73b7680dea578p-1, 0x1.2248306dc12a2p-56, 0x1.6018526f563dfp-1, 0x1.46ca5e0e432d0p-55,
    -0x1.6e2b77c40bde1p-1, 0x1.0e729857fad53p-56, 0x1.65dc1fdeb8cbap-1, -0x1.97c1b47337c77p-58,
    -0x1.6888a4e134b2fp-1, 0x1.6b7d37644d5e6p-55, 0x1.6b898fa9efb5dp-1, 0x1.15ac786ccf4b2p-56,
    -0x1.62cf49921ac79p-1, 0x1.edd9855b6241ap-55, 0x1.712046fa77678p-1, 0x1.425b0a5029c81p-55,
    -0x1.5cffc16bf8f0dp-1, -0x1.96cb370eb578ap-55, 0x1.769fec655211fp-1, -0x1.827d5cf8c68c5p-57,
    -0x1.571a6966d59b3p-1, -0x1.c843b4d0fb197p-58, 0x1.7c0827f09e54fp-1, -0x1.c73d6d72aee68p-57,
    -0x1.511f9fd7b351cp-1, 0x1.5c0e861c48831p-55, 0x1.8158a31916d5dp-1, -0x1.de8b90b8228dep-57,
    -0x1.4b0fc46aab761p-1, -0x1.0da05738cc59cp-61, 0x1.869108d77a6c6p-1, 0x1.338ffe2bfe9ddp-56,
    -0x1.44eb381cf386bp-1, 0x1.3ed6c1e6a5505p-55, 0x1.8bb105a5dc900p-1, 0x1.863e03e9474c1p-55,
    -0x1.3eb25d36cd53ap-1, 0x1.be570e1570fc0p-58, 0x1.90b84784ddaf7p-1, -0x1.0feb10ab93b87p-56,
    -0x1.386597456282bp-1, 0x1.10fada93b07a8p-56, 0x1.95a67e00cb1fdp-1, -0x1.0befda21f862dp-55,
    -0x1.32054b148bc4fp-1, -0x1.f6b42095a135bp-55, 0x1.9a7b5a36a6514p-1, 0x1.722cfcc9fa7a9p-55,
    -0x1.2b91dea88421ep-1, 0x1.fa371db216ab0p-55, 0x1.9f368ed912f85p-1, -0x1.1d200c5791606p-55,
    -0x1.250bb93788bbbp-1, -0x1.ea3d02457bccep-56, 0x1.a3d7d0352bdcfp-1, -0x1.68dbaeca19669p-55,
    -0x1.1e7343236574cp-1, -0x1.22a3fa4f41d5ap-56, 0x1.a85ed4373e02dp-1, 0x1.9be06385ec792p-57,
    -0x1.17c8e5f2eedb0p-1, -0x1.35e57102e2488p-57, 0x1.accb526f69de5p-1, 0x1.8fb6a8dd6b6ccp-55,
    -0x1.110d0c4b69c3bp-1, -0x1.d918998809981p-55, 0x1.b11d04162a4c6p-1, 0x1.1dd561efbc0c2p-56,
    -0x1.0a4021e9e1001p-1, 0x1.6f643a13914f6p-55, 0x1.b553a410c104ep-1, 0x1.8ff7947027a15p-58,
    -0x1.0362939c69955p-1, 0x1.2d8cd78397b01p-55, 0x1.b96eeef58840ep-1, 0x1.45a3cc78fade0p-58,
    -0x1.f8e99e76abc97p-2, -0x1.9d950af2d00a3p-58, 0x1.bd6ea310294f5p-1, 0x1.31bbcc88c109dp-56,
    -0x1.eaee8744b05f0p-2, 0x1.789b43c9b027dp-58, 0x1.c1528065b7d50p-1, -0x1.892111312e828p-55,
    -0x1.dcd4c15329c9ap-2, -0x1.0d4c6e171fd9ap-56, 0x1.c51a48b8b175ep-1, -0x1.1bbb43b9aa880p-57,
    -0x1.ce9d2e3d4a51fp-2, 0x1.2fc8a12dae298p-57, 0x1.c8c5bf8ce1a84p-1, 0x1.ab3d1a1590123p-56,
    -0x1.c048b17b140a3p-2, -0x1.19fe6757e9fa7p-57, 0x1.cc54aa2b2972ep-1, 0x1.4ee162ba83a98p-57,
    -0x1.b1d8305321617p-2, 0x1.ae242cb99f519p-56, 0x1.cfc6cfa52ad9fp-1, 0x1.8b5b5508f2a0dp-55,
    -0x1.a34c91cc50ccap-2, 0x1.a310e3b50cecdp-58, 0x1.d31bf8d8d7c06p-1, 0x1.e60dd3089cbddp-56,
    -0x1.94a6be9f546c5p-2, 0x1.69ce13e683f58p-56, 0x1.d653f073e4040p-1, -0x1.76236434bec37p-55,
    -0x1.85e7a12826949p-2, -0x1.8a40e9b5face0p-56, 0x1.d96e82f71a9dcp-1, 0x1.ff61bd5d2039dp-55,
    -0x1.7710255764214p-2, 0x1.6ead7314bb6cep-57, 0x1.dc6b7eb995912p-1, 0x1.4b364776dcd35p-58,
    -0x1.682138a38d7f7p-2, 0x1.d889202444aadp-56, 0x1.df4ab3ebd875ep-1, -0x1.e2d8a7e6736c4p-55,
    -0x1.591bc9fa2f597p-2, -0x1.7c74bac3fe0cbp-57, 0x1.e20bf49acd6c1p-1, -0x1.660aec7ef636bp-58,
    -0x1.4a00c9b0f3d20p-2, -0x1.823ba6bb08eadp-56, 0x1.e4af14b2a449cp-1, -0x1.68ca02e8a6833p-55,
    -0x1.3ad129769d3d8p-2, -0x1.03d550487839ap-63, 0x1.e733ea0193d40p-1, -0x1.6428b3546ce13p-55,
    -0x1.2b8ddc43eb49fp-2, -0x1.1553899f2d807p-57, 0x1.e99a4c3a7cd83p-1, -0x1.2264b1bc53ce8p-55,
    -0x1.1c37d64c6b876p-2, -0x1.46076fe0dcff4p-56, 0x1.ebe214f76efa8p-1, -0x1.02f9f12ba543ep-55,
    -0x1.0cd00cef36436p-2, 0x1.9fb0a0c93e2b4p-56, 0x1.ee0b1fbc0f11cp-1, -0x1.bfd2380bbc3b1p-59,
    -0x1.faaeed4f31577p-3, 0x1.15d88508e32b8p-57, 0x1.f01549f7deea1p-1, 0x1.d3c1e99e5cafdp-55,
    -0x1.db9e15fb5a5d0p-3, 0x1.32e20d6cc6fc2p-57, 0x1.f20073086649fp-1, 0x1.b940416c1984bp-56,
    -0x1.bc6f84edc6199p-3, -0x1.9c1a56a7b0cabp-57, 0x1.f3cc7c3b3d16ep-1, -0x1.21a3ad28a3494p-57,
    -0x1.9d252d0cec312p-3, -0x1.9c43d80b1137dp-58, 0x1.f57948cff6797p-1, 0x1.e3a0d3e03b1d4p-57,
    -0x1.7dc102fbaf2b5p-3, -0x1.5ab50e23c97c3p-59, 0x1.f706bdf9ece1cp-1, -0x1.698c80c36dcb4p-55,
    -0x1.5e44fcfa126f3p-3, 0x1.6f443063f89b6p-57, 0x1.f874c2e1eecf6p-1, -0x1.c6514e1332b16p-55,
    -0x1.3eb312c5d66cbp-3, -0x1.47d666b66cb91p-57, 0x1.f9c340a7cc428p-1, 0x1.c5b6b063b7462p-55,
    -0x1.1f0d3d7afceafp-3, 0x1.6ef95099769a5p-57, 0x1.faf22263c4bd3p-1, -0x1.52ace133a2769p-58,
    -0x1.feaaeee86ee36p-4, 0x1.afcb2bcc6f03bp-59, 0x1.fc015527d5bd3p-1, 0x1.b68f35094efb8p-55,
    -0x1.bf1b78568391dp-4, -0x1.e91841dea4cc8p-58, 0x1.fcf0c800e99b1p-1, 0x1.ea3d786d186acp-57,
    -0x1.7f701032550e4p-4, -0x1.afc2d1800501ap-60, 0x1.fdc06bf7e6b9bp-1, 0x1.31902b535f8dbp-55,
    -0x1.3facb12d1755bp-4, 0x1.921915299468bp-58, 0x1.fe7034129ef6fp-1, -0x1.cbf4337c96f97p-57,
    -0x1.ffaaaeeed4edbp-5, 0x1.2d16d32684b69p-59, 0x1.ff0015549f4d3p-1, 0x1.328387b99426fp-55,
    -0x1.7fdc01032fba9p-5, 0x1.599bdf46e997ap-59, 0x1.ff7006bfdf99fp-1, -0x1.8b3b560648d5fp-56,
    -0x1.ffeaaaeeee86fp-6, 0x1.cd406fb224ae2p-60, 0x1.ffc00155527d3p-1, -0x1.3b54492d89b5bp-55,
    -0x1.fffaaaaeeeed5p-7, 0x1.2ab639a9f0776p-63, 0x1.fff000155549fp-1, 0x1.28a28a03a5ef3p-55,
    0.0, 0.0, 0x1.0000000000000p+0, 0.0,
    0x1.fffaaaaeeeed5p-7, -0x1.2ab639a9f0776p-63, 0x1.fff000155549fp-1, 0x1.28a28a03a5ef3p-55,
    0x1.ffeaaaeeee86fp-6, -0x1.cd406fb224ae2p-60, 0x1.ffc00155527d3p-1, -0x1.3b54492d89b5bp-55,
    0x1.7fdc01032fba9p-5, -0x1.599bdf46e997ap-59, 0x1.ff7006bfdf99fp-1, -0x1.8b3b560648d5fp-56,
    0x1.ffaaaeeed4edbp-5, -0x1.2d16d32684b69p-59, 0x1.ff0015549f4d3p-1, 0x1.328387b99426fp-55,
    0x1.3facb12d1755bp-4, -0x1.921915299468bp-58, 0x1.fe7034129ef6fp-1, -0x1.cbf4337c96f97p-57,
    0x1.7f701032550e4p-4, 0x1.afc2d1800501ap-60, 0x1.fdc06bf7e6b9bp-1, 0x1.31902b535f8dbp-55,
    0x1.bf1b78568391dp-4, 0x1.e91841dea4cc8p-58, 0x1.fcf0c800e99b1p-1, 0x1.ea3d786d186acp-57,
    0x1.feaaeee86ee36p-4, -0x1.afcb2bcc6f03bp-59, 0x1.fc015527d5bd3p-1, 0x1.b68f35094efb8p-55,
    0x1.1f0d3d7afceafp-3, -0x1.6ef95099769a5p-57, 0x1.faf22263c4bd3p-1, -0x1.52ace133a2769p-58,
    0x1.3eb312c5d66cbp-3, 0x1.47d666b66cb91p-57, 0x1.f9c340a7cc428p-1, 0x1.c5b6b063b7462p-55,
    0x1.5e44fcfa126f3p-3, -0x1.6f443063f89b6p-57, 0x1.f874c2e1eecf6p-1, -0x1.c6514e1332b16p-55,
    0x1.7dc102fbaf2b5p-3, 0x1.5ab50e23c97c3p-59, 0x1.f706bdf9ece1cp-1, -0x1.698c80c36dcb4p-55,
    0x1.9d252d0cec312p-3, 0x1.9c43d80b1137dp-58, 0x1.f57948cff6797p-1, 0x1.e3a0d3e03b1d4p-57,
    0x1.bc6f84edc6199p-3, 0x1.9c1a56a7b0cabp-57, 0x1.f3cc7c3b3d16ep-1, -0x1.21a3ad28a3494p-57,
    0x1.db9e15fb5a5d0p-3, -0x1.32e20d6cc6fc2p-57, 0x1.f20073086649fp-1, 0x1.b940416c1984bp-56,
    0x1.faaeed4f31577p-3, -0x1.15d88508e32b8p-57, 0x1.f01549f7deea1p-1, 0x1.d3c1e99e5cafdp-55,
    0x1.0cd00cef36436p-2, -0x1.9fb0a0c93e2b4p-56, 0x1.ee0b1fbc0f11cp-1, -0x1.bfd2380bbc3b1p-59,
    0x1.1c37d64c6b876p-2, 0x1.46076fe0dcff4p-56, 0x1.ebe214f76efa8p-1, -0x1.02f9f12ba543ep-55,
    0x1.2b8ddc43eb49fp-2, 0x1.1553899f2d807p-57, 0x1.e99a4c3a7cd83p-1, -0x1.2264b1bc53ce8p-55,
    0x1.3ad129769d3d8p-2, 0x1.03d550487839ap-63, 0x1.e733ea0193d40p-1, -0x1.6428b3546ce13p-55,
    0x1.4a00c9b0f3d20p-2, 0x1.823ba6bb08eadp-56, 0x1.e4af14b2a449cp-1, -0x1.68ca02e8a6833p-55,
    0x1.591bc9fa2f597p-2, 0x1.7c74bac3fe0cbp-57, 0x1.e20bf49acd6c1p-1, -0x1.660aec7ef636bp-58,
    0x1.682138a38d7f7p-2, -0x1.d889202444aadp-56, 0x1.df4ab3ebd875ep-1, -0x1.e2d8a7e6736c4p-55,
    0x1.7710255764214p-2, -0x1.6ead7314bb6cep-57, 0x1.dc6b7eb995912p-1, 0x1.4b364776dcd35p-58,
    0x1.85e7a12826949p-2, 0x1.8a40e9b5face0p-56, 0x1.d96e82f71a9dcp-1, 0x1.ff61bd5d2039dp-55,
    0x1.94a6be9f546c5p-2, -0x1.69ce13e683f58p-56, 0x1.d653f073e4040p-1, -0x1.76236434bec37p-55,
    0x1.a34c91cc50ccap-2, -0x1.a310e3b50cecdp-58, 0x1.d31bf8d8d7c06p-1, 0x1.e60dd3089cbddp-56,
    0x1.b1d8305321617p-2, -0x1.ae242cb99f519p-56, 0x1.cfc6cfa52ad9fp-1, 0x1.8b5b5508f2a0dp-55,
    0x1.c048b17b140a3p-2, 0x1.19fe6757e9fa7p-57, 0x1.cc54aa2b2972ep-1, 0x1.4ee162ba83a98p-57,
    0x1.ce9d2e3d4a51fp-2, -0x1.2fc8a12dae298p-57, 0x1.c8c5bf8ce1a84p-1, 0x1.ab3d1a1590123p-56,
    0x1.dcd4c15329c9ap-2, 0x1.0d4c6e171fd9ap-56, 0x1.c51a48b8b175ep-1, -0x1.1bbb43b9aa880p-57,
    0x1.eaee8744b05f0p-2, -0x1.789b43c9b027dp-58, 0x1.c1528065b7d50p-1, -0x1.892111312e828p-55,
    0x1.f8e99e76abc97p-2, 0x1.9d950af2d00a3p-58, 0x1.bd6ea310294f5p-1, 0x1.31bbcc88c109dp-56,
    0x1.0362939c69955p-1, -0x1.2d8cd78397b01p-55, 0x1.b96eeef58840ep-1, 0x1.45a3cc78fade0p-58,
    0x1.0a4021e9e1001p-1, -0x1.6f643a13914f6p-55, 0x1.b553a410c104ep-1, 0x1.8ff7947027a15p-58,
    0x1.110d0c4b69c3bp-1, 0x1.d918998809981p-55, 0x1.b11d04162a4c6p-1, 0x1.1dd561efbc0c2p-56,
    0x1.17c8e5f2eedb0p-1, 0x1.35e57102e2488p-57, 0x1.accb526f69de5p-1, 0x1.8fb6a8dd6b6ccp-55,
    0x1.1e7343236574cp-1, 0x1.22a3fa4f41d5ap-56, 0x1.a85ed4373e02dp-1, 0x1.9be06385ec792p-57,
    0x1.250bb93788bbbp-1, 0x1.ea3d02457bccep-56, 0x1.a3d7d0352bdcfp-1, -0x1.68dbaeca19669p-55,
    0x1.2b91dea88421ep-1, -0x1.fa371db216ab0p-55, 0x1.9f368ed912f85p-1, -0x1.1d200c5791606p-55,
    0x1.32054b148bc4fp-1, 0x1.f6b42095a135bp-55, 0x1.9a7b5a36a6514p-1, 0x1.722cfcc9fa7a9p-55,
    0x1.386597456282bp-1, -0x1.10fada93b07a8p-56, 0x1.95a67e00cb1fdp-1, -0x1.0befda21f862dp-55,
    0x1.3eb25d36cd53ap-1, -0x1.be570e1570fc0p-58, 0x1.90b84784ddaf7p-1, -0x1.0feb10ab93b87p-56,
    0x1.44eb381cf386bp-1, -0x1.3ed6c1e6a5505p-55, 0x1.8bb105a5dc900p-1, 0x1.863e03e9474c1p-55,
    0x1.4b0fc46aab761p-1, 0x1.0da05738cc59cp-61, 0x1.869108d77a6c6p-1, 0x1.338ffe2bfe9ddp-56,
    0x1.511f9fd7b351cp-1, -0x1.5c0e861c48831p-55, 0x1.8158a31916d5dp-1, -0x1.de8b90b8228dep-57,
    0x1.571a6966d59b3p-1, 0x1.c843b4d0fb197p-58, 0x1.7c0827f09e54fp-1, -0x1.c73d6d72aee68p-57,
    0x1.5cffc16bf8f0dp-1, 0x1.96cb370eb578ap-55, 0x1.769fec655211fp-1, -0x1.827d5cf8c68c5p-57,
    0x1.62cf49921ac79p-1, -0x1.edd9855b6241ap-55, 0x1.712046fa77678p-1, 0x1.425b0a5029c81p-55,
    0x1.6888a4e134b2fp-1, -0x1.6b7d37644d5e6p-55, 0x1.6b898fa9efb5dp-1, 0x1.15ac786ccf4b2p-56,
    0x1.6e2b77c40bde1p-1, -0x1.0e729857fad53p-56, 0x1.65dc1fdeb8cbap-1, -0x1.97c1b47337c77p-58,
    0x1.73b7680dea578p-1, -0x1.2248306dc12a2p-56, 0x1.6018526f563dfp-1, 0x1.46ca5e0e432d0p-55,
};
#define VSM_TAB(i, sh, sl, ch, cl) do { \
    sh = vsm_tab[4 * (i)]; sl = vsm_tab[4 * (i) + 1]; ch = vsm_tab[4 * (i) + 2]; cl = vsm_tab[4 * (i) + 3]; } while (0)
#endif

/* correctly rounded value of yh + yl if the error bound cannot change it, else NaN marker */
VSM_FN int vsm_round_ok(vsm_dd y, double *out) {
    double e = VSM_FAST_EPS * (y.hi < 0.0 ? -y.hi : y.hi);
    double a = y.hi + (y.lo + e), b = y.hi + (y.lo - e);
    *out = a;
    return a == b;
}

/* sin(r), cos(r) of a reduced double-double r, |r| <= pi/4 + eps; returns 1 if both are
 * certainly correctly rounded (want: bit 0 sin, bit 1 cos) */
VSM_FN int vsm_fast_sc(vsm_dd r, double *s, double *c, int want) {
    double fi = VSM_RINT(r.hi * 64.0);
    int i = (int)fi + 52;
    double th = VSM_FMA(-fi, 0.015625, r.hi);     /* exact: fi/64 has <= 7 bits, same binade grid */
    double tl = r.lo;
    double sah, sal, cah, cal;
    VSM_TAB(i, sah, sal, cah, cal);
    double t2 = th * th;
    double st = th * t2 * (VSM_F_S1 + t2 * (VSM_F_S2 + t2 * VSM_F_S3));        /* sin t - t - tl */
    double cm1 = VSM_FMA(-th, tl, t2 * (-0.5 + t2 * (VSM_F_C2 + t2 * VSM_F_C3))); /* cos t - 1 */
    double tt = tl + st;
    int ok = 1;
    if (want & 1) {
        double ph = cah * th;
        double pl = VSM_FMA(cah, th, -ph);         /* CA_hi*th = ph + pl exactly */
        vsm_dd h = vsm_fast_two_sum(sah, ph);     /* |SA| >= sin(1/64) > |CA*th| (or SA = 0) */
        double lo = h.lo + (pl + (sal + (sah * cm1 + (cah * tt + cal * th))));
        ok &= vsm_round_ok(vsm_fast_two_sum(h.hi, lo), s);
    }
    if (want & 2) {
        double qh = -sah * th;
        double ql = VSM_FMA(-sah, th, -qh);
        vsm_dd g = vsm_fast_two_sum(cah, qh);     /* CA >= cos(0.8) > |SA*th| */
        double lo = g.lo + (ql + (cal + (cah * cm1 - (sah * tt + sal * th))));
        ok &= vsm_round_ok(vsm_fast_two_sum(g.hi, lo), c);
    }
    return ok;
}

VSM_FN double vs_sin_slow(vsm_dd r, int q) {
    vsm_dd v = (q & 1) ? vsm_cos_kernel(r) : vsm_sin_kernel(r);
    double s = v.hi + v.lo;
    return (q & 2) ? -s : s;
}

VSM_FN double vs_cos_slow(vsm_dd r, int q) {
    vsm_dd v = (q & 1) ? vsm_sin_kernel(r) : vsm_cos_kernel(r);
    double c = v.hi + v.lo;
    return ((q + 1) & 2) ? -c : c;
}

#ifdef VSM_NO_FAST
#define VSM_TRY_FAST(r, s, c, w) 0
#else
#define VSM_TRY_FAST(r, s, c, w) vsm_fast_sc(r, s, c, w)
#endif

VSM_FN double vs_sin(double x) {
    double ax = x < 0.0 ? -x : x;
    if (!(ax < 1073741824.0)) return VSM_SIN_FALLBACK(x);   /* NaN, inf, |x| >= 2^30 */
    if (ax < 7.450580596923828e-09) return x;                /* |x| < 2^-27: sin x = x */
    vsm_dd r;
    int q = (int)((long long)vsm_reduce(x, &r) & 3);
    double sv, cv;
    if (VSM_TRY_FAST(r, &sv, &cv, (q & 1) ? 2 : 1)) {
        double v = (q & 1) ? cv : sv;
        return (q & 2) ? -v : v;
    }
    return vs_sin_slow(r, q);
}

VSM_FN double vs_cos(double x) {
    double ax = x < 0.0 ? -x : x;
    if (!(ax < 1073741824.0)) return VSM_COS_FALLBACK(x);
    if (ax < 7.450580596923828e-09) return 1.0;
    vsm_dd r;
    int q = (int)((long long)vsm_reduce(x, &r) & 3);
    double sv, cv;
    if (VSM_TRY_FAST(r, &sv, &cv, (q & 1) ? 1 : 2)) {
        double v = (q & 1) ? sv : cv;
        return ((q + 1) & 2) ? -v : v;
    }
    return vs_cos_slow(r, q);
}

/* both at once: one reduction (codegen pairs SIN and COS of the same value) */
VSM_FN void vs_sincos(double x, double *s, double *c) {
    double ax = x < 0.0 ? -x : x;
    if (!(ax < 1073741824.0)) { *s = VSM_SIN_FALLBACK(x); *c = VSM_COS_FALLBACK(x); return; }
    if (ax < 7.450580596923828e-09) { *s = x; *c = 1.0; return; }
    vsm_dd r;
    int q = (int)((long long)vsm_reduce(x, &r) & 3);
    double sv, cv;
    if (!VSM_TRY_FAST(r, &sv, &cv, 3)) {
        vsm_dd vs = vsm_sin_kernel(r), vc = vsm_cos_kernel(r);
        sv = vs.hi + vs.lo;
        cv = vc.hi + vc.lo;
    }
    double s0 = (q & 1) ? cv : sv, c0 = (q & 1) ? sv : cv;
    *s = (q & 2) ? -s0 : s0;
    *c = ((q + 1) & 2) ? -c0 : c0;
}

/* reference (slow path only), for validation */
VSM_FN void vs_sincos_dd(double x, double *s, double *c) {
    double ax = x < 0.0 ? -x : x;
    if (!(ax < 1073741824.0)) { *s = VSM_SIN_FALLBACK(x); *c = VSM_COS_FALLBACK(x); return; }
    if (ax < 7.450580596923828e-09) { *s = x; *c = 1.0; return; }
    vsm_dd r;
    int q = (int)((long long)vsm_reduce(x, &r) & 3);
    *s = vs_sin_slow(r, q);
    *c = vs_cos_slow(r, q);
}

#endif /* VS_MATH_H */
