/*
 * mc_detmath.h — TEST INFRASTRUCTURE (oracle). Deterministic libm
 * replacements used by the CPU oracle and by the reference harness's
 * restated tracer. The device code restates the same algorithms in CUDA
 * (paper_2305_07238_b200/csrc/device_math.cuh); bit-equality of the two is
 * a parity test (tests/test_detmath.py).
 *
 * Why: the reference calls glibc sinf/powf (include/matcache/value.hpp:125-137),
 * which CUDA's sinf/powf do not reproduce bit-for-bit. Both implementations
 * of the hot path therefore evaluate sin and pow with these double-precision
 * routines (and the sphere parameterization's atan2f/acosf, scene.cpp:234-235,
 * likewise): the result is the float nearest the double-precision value,
 * i.e. correctly rounded except in astronomically rare ties. Against glibc
 * they agree except where glibc itself is not correctly rounded (measured
 * in tests/test_oracle_vs_ref.py; "parity vs glibc unpinned at <= 1 ulp").
 *
 * Every expression is written so that -ffp-contract=off on the host and
 * --fmad=false on the device evaluate the same IEEE operations in the same
 * order.
 */
#ifndef MC_DETMATH_H_
#define MC_DETMATH_H_

#include <math.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* pi/2 split for Cody-Waite reduction: P1, P2 carry 33 significant bits so
 * k*P1 and k*P2 are exact for |k| < 2^20 (fdlibm's pio2_1, pio2_2, pio2_2t). */
#define MC_PIO2_1 1.57079632673412561417e+00
#define MC_PIO2_2 6.07710050630396597660e-11
#define MC_PIO2_3 2.02226624879595063154e-21
#define MC_2_OVER_PI 6.36619772367581382433e-01

static inline double mc_sin_poly(double r) {
    const double z = r * r;
    double p = 1.0 / 355687428096000.0;           /* 1/17! */
    p = p * z - 1.0 / 1307674368000.0;            /* 1/15! */
    p = p * z + 1.0 / 6227020800.0;               /* 1/13! */
    p = p * z - 1.0 / 39916800.0;                 /* 1/11! */
    p = p * z + 1.0 / 362880.0;                   /* 1/9!  */
    p = p * z - 1.0 / 5040.0;                     /* 1/7!  */
    p = p * z + 1.0 / 120.0;                      /* 1/5!  */
    p = p * z - 1.0 / 6.0;                        /* 1/3!  */
    return r + (r * z) * p;
}

static inline double mc_cos_poly(double r) {
    const double z = r * r;
    double p = 1.0 / 6402373705728000.0;          /* 1/18! */
    p = p * z - 1.0 / 20922789888000.0;           /* 1/16! */
    p = p * z + 1.0 / 87178291200.0;              /* 1/14! */
    p = p * z - 1.0 / 479001600.0;                /* 1/12! */
    p = p * z + 1.0 / 3628800.0;                  /* 1/10! */
    p = p * z - 1.0 / 40320.0;                    /* 1/8!  */
    p = p * z + 1.0 / 720.0;                      /* 1/6!  */
    p = p * z - 1.0 / 24.0;                       /* 1/4!  */
    p = p * z + 0.5;                              /* 1/2!  */
    return 1.0 - z * p;
}

/* sin and cos of a float argument, each rounded once from double. */
static inline void mc_sincosf(float a, float* s_out, float* c_out) {
    const double x = (double)a;
    if (!(x - x == 0.0)) { /* inf or nan */
        *s_out = (float)(x - x);
        *c_out = (float)(x - x);
        return;
    }
    const double k = rint(x * MC_2_OVER_PI);
    const double r = ((x - k * MC_PIO2_1) - k * MC_PIO2_2) - k * MC_PIO2_3;
    const double sr = mc_sin_poly(r);
    const double cr = mc_cos_poly(r);
    const double kq = k - 4.0 * floor(k * 0.25); /* k mod 4, exact */
    double s, c;
    switch ((int)kq) {
        case 0: s = sr; c = cr; break;
        case 1: s = cr; c = -sr; break;
        case 2: s = -sr; c = -cr; break;
        default: s = -cr; c = sr; break;
    }
    *s_out = (float)s;
    *c_out = (float)c;
}

static inline float mc_sinf(float a) {
    float s, c;
    mc_sincosf(a, &s, &c);
    return s;
}

/* log2 of a positive finite double, ~1e-17 relative: x = m * 2^e with m in
 * [sqrt(1/2), sqrt(2)); ln m = 2 atanh(t), t = (m-1)/(m+1). */
static inline double mc_log2_pos(double x) {
    int e;
    double m = frexp(x, &e); /* m in [0.5, 1) */
    if (m < 0.70710678118654752440) {
        m = m * 2.0;
        e = e - 1;
    }
    const double t = (m - 1.0) / (m + 1.0);
    const double t2 = t * t;
    double p = 1.0 / 25.0;
    p = p * t2 + 1.0 / 23.0;
    p = p * t2 + 1.0 / 21.0;
    p = p * t2 + 1.0 / 19.0;
    p = p * t2 + 1.0 / 17.0;
    p = p * t2 + 1.0 / 15.0;
    p = p * t2 + 1.0 / 13.0;
    p = p * t2 + 1.0 / 11.0;
    p = p * t2 + 1.0 / 9.0;
    p = p * t2 + 1.0 / 7.0;
    p = p * t2 + 1.0 / 5.0;
    p = p * t2 + 1.0 / 3.0;
    p = p * t2 + 1.0;
    const double ln_m = 2.0 * (t * p);
    return (double)e + ln_m * 1.44269504088896340736; /* 1/ln 2 */
}

/* 2^z for finite z, as a double (overflow -> inf, underflow -> 0/subnormal). */
static inline double mc_exp2(double z) {
    if (z > 1100.0) return INFINITY;
    if (z < -1100.0) return 0.0;
    const double n = rint(z);
    const double f = (z - n) * 0.69314718055994530942; /* (z-n) ln 2, |.| <= 0.347 */
    double p = 1.0 / 6402373705728000.0;               /* 1/18! */
    p = p * f + 1.0 / 355687428096000.0;
    p = p * f + 1.0 / 20922789888000.0;
    p = p * f + 1.0 / 1307674368000.0;
    p = p * f + 1.0 / 87178291200.0;
    p = p * f + 1.0 / 6227020800.0;
    p = p * f + 1.0 / 479001600.0;
    p = p * f + 1.0 / 39916800.0;
    p = p * f + 1.0 / 3628800.0;
    p = p * f + 1.0 / 362880.0;
    p = p * f + 1.0 / 40320.0;
    p = p * f + 1.0 / 5040.0;
    p = p * f + 1.0 / 720.0;
    p = p * f + 1.0 / 120.0;
    p = p * f + 1.0 / 24.0;
    p = p * f + 1.0 / 6.0;
    p = p * f + 0.5;
    p = p * f + 1.0;
    p = p * f + 1.0;
    return ldexp(p, (int)n);
}

/* powf(x, y) for x >= 0 (the only domain ops::power uses, value.hpp:132-137),
 * C99 special cases; finite results rounded once from double. */
static inline float mc_powf_nonneg(float xf, float yf) {
    const double x = (double)xf, y = (double)yf;
    if (yf == 0.0f) return 1.0f;
    if (xf == 1.0f) return 1.0f;
    if (xf != xf || yf != yf) return xf + yf; /* nan */
    if (xf == 0.0f) return yf > 0.0f ? 0.0f : INFINITY;
    if (isinf(xf)) return yf > 0.0f ? INFINITY : 0.0f;
    if (isinf(yf)) {
        if (xf < 1.0f) return yf > 0.0f ? 0.0f : INFINITY;
        return yf > 0.0f ? INFINITY : 0.0f;
    }
    return (float)mc_exp2(y * mc_log2_pos(x));
}

/* atan of t in [0, 1], ~1e-16 relative: reflect above tan(pi/8) around
 * pi/4, halve the angle once (atan t = 2 atan(t / (1 + sqrt(1 + t^2))),
 * |h| <= 0.199), then 12 terms of the Taylor series. */
static inline double mc_atan_unit(double t) {
    double base = 0.0;
    if (t > 0.41421356237309504880) {
        t = (t - 1.0) / (t + 1.0);
        base = 0.78539816339744830962;
    }
    const double h = t / (1.0 + sqrt(1.0 + t * t));
    const double z = h * h;
    double p = -1.0 / 23.0;
    p = p * z + 1.0 / 21.0;
    p = p * z - 1.0 / 19.0;
    p = p * z + 1.0 / 17.0;
    p = p * z - 1.0 / 15.0;
    p = p * z + 1.0 / 13.0;
    p = p * z - 1.0 / 11.0;
    p = p * z + 1.0 / 9.0;
    p = p * z - 1.0 / 7.0;
    p = p * z + 1.0 / 5.0;
    p = p * z - 1.0 / 3.0;
    return base + 2.0 * (h + (h * z) * p);
}

/* atan2 in double with C99 special cases (zeros, infinities, nan). */
static inline double mc_atan2_d(double y, double x) {
    if (x != x || y != y) return x + y;
    const double ax = fabs(x), ay = fabs(y);
    double a;
    if (ay == 0.0) a = 0.0;
    else if (isinf(ax) && isinf(ay)) a = 0.78539816339744830962;
    else if (ay <= ax) a = mc_atan_unit(ay / ax);
    else a = 1.57079632679489661923 - mc_atan_unit(ax / ay);
    if (signbit(x)) a = 3.14159265358979323846 - a;
    return copysign(a, y);
}

/* atan2f / acosf of the sphere parameterization (scene.cpp:234-235), each
 * rounded once from double. */
static inline float mc_atan2f(float y, float x) { return (float)mc_atan2_d((double)y, (double)x); }

static inline float mc_acosf(float a) {
    const double x = (double)a;
    if (x != x || fabs(x) > 1.0) return (float)((x - x) / (x - x));
    return (float)mc_atan2_d(sqrt((1.0 - x) * (1.0 + x)), x);
}

#ifdef __cplusplus
}
#endif

#endif /* MC_DETMATH_H_ */
