/* Host harness for csrc/vs_math.h (test infrastructure): the same header the
 * kernels embed, compiled with gcc -ffp-contract=off, exposed over ctypes. */
#include "../../paper_2408_09662_b200/csrc/vs_math.h"

void h_sincos(const double *x, double *s, double *c, long n) {
    for (long i = 0; i < n; ++i) vs_sincos(x[i], s + i, c + i);
}
void h_sin(const double *x, double *s, long n) { for (long i = 0; i < n; ++i) s[i] = vs_sin(x[i]); }
void h_cos(const double *x, double *c, long n) { for (long i = 0; i < n; ++i) c[i] = vs_cos(x[i]); }
void h_sincos_dd(const double *x, double *s, double *c, long n) {
    for (long i = 0; i < n; ++i) vs_sincos_dd(x[i], s + i, c + i);
}
void h_libm(const double *x, double *s, double *c, long n) {
    for (long i = 0; i < n; ++i) { s[i] = sin(x[i]); c[i] = cos(x[i]); }
}
/* fast-path statistics: fallbacks and the max relative error of the unrounded
 * fast (yh + yl) against the 2^-75 double-double kernels, for |x| in the fast range */
long h_fast_stats(const double *x, long n, double *max_rel_s, double *max_rel_c) {
    long fb = 0;
    double ms = 0.0, mc = 0.0;
    for (long i = 0; i < n; ++i) {
        double ax = x[i] < 0 ? -x[i] : x[i];
        if (!(ax < 1073741824.0) || ax < 7.450580596923828e-09) continue;
        vsm_dd r;
        vsm_reduce(x[i], &r);
        double sv, cv;
        if (!vsm_fast_sc(r, &sv, &cv, 3)) ++fb;
        /* recompute the unrounded fast values */
        double fi = VSM_RINT(r.hi * 64.0);
        int j = (int)fi + 52;
        double th = VSM_FMA(-fi, 0.015625, r.hi), tl = r.lo, sah, sal, cah, cal;
        VSM_TAB(j, sah, sal, cah, cal);
        double t2 = th * th;
        double st = th * t2 * (VSM_F_S1 + t2 * (VSM_F_S2 + t2 * VSM_F_S3));
        double cm1 = VSM_FMA(-th, tl, t2 * (-0.5 + t2 * (VSM_F_C2 + t2 * VSM_F_C3)));
        double tt = tl + st;
        double ph = cah * th, pl = VSM_FMA(cah, th, -ph);
        vsm_dd h = vsm_fast_two_sum(sah, ph);
        vsm_dd ys = vsm_fast_two_sum(h.hi, h.lo + (pl + (sal + (sah * cm1 + (cah * tt + cal * th)))));
        double qh = -sah * th, ql = VSM_FMA(-sah, th, -qh);
        vsm_dd g = vsm_fast_two_sum(cah, qh);
        vsm_dd yc = vsm_fast_two_sum(g.hi, g.lo + (ql + (cal + (cah * cm1 - (sah * tt + sal * th)))));
        vsm_dd es = vsm_sin_kernel(r), ec = vsm_cos_kernel(r);
        vsm_dd ds = vsm_dd_add(ys, (vsm_dd){-es.hi, -es.lo});
        vsm_dd dc = vsm_dd_add(yc, (vsm_dd){-ec.hi, -ec.lo});
        double rs = fabs(ds.hi) / fabs(es.hi), rc = fabs(dc.hi) / fabs(ec.hi);
        if (rs > ms) ms = rs;
        if (rc > mc) mc = rc;
    }
    *max_rel_s = ms;
    *max_rel_c = mc;
    return fb;
}
