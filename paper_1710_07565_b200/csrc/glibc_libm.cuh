// glibc_libm.cuh -- device restatement of the host libm routines the reference's
// point set passes through, bit-exact with the reference's glibc 2.39 (x86-64,
// FMA ifunc variants: the builds its std:: calls resolve to on FMA-capable CPUs).
//
//   reference call                                  routine restated here
//   rng.hpp:221        std::pow(U, 1/remaining)     gl_pow   (ARM optimized-routines pow)
//   partition.hpp:66 -> geometry.hpp:110 std::acosh  gl_acosh (fdlibm acosh over gl_log / gl_log1p)
//   sweep.hpp:125      std::exp(r)                  gl_exp   (ARM optimized-routines exp)
//   sweep.hpp:66       std::acos(arg)               gl_acos  (IBM Accurate Mathematical Library)
//   sweep.hpp:138-139  std::cos/std::sin(theta)     gl_sincos (gcc -O3 merges the pair into
//                                                    sincos; IBM Accurate Mathematical Library)
//
// Each routine restates the published algorithm; where the FMA build of glibc
// contracted a multiply-add, the restatement uses an explicit fused op (gF), and
// everywhere else separately rounded ops (gM/gA/gS), so the result does not depend
// on the compiler's contraction flags.  The contraction points were read off the
// disassembly of the host libm.so.6; the table words and constants
// come from the same library via tools/libm/gen_glibc_tables.py.  Equality with the
// host glibc is proven on CPU (tools/libm/check_host.cpp, same source compiled for
// the host) and on the device (tests/test_gpu_libm.py).
//
// The same source compiles for the host (g++) so the CPU check exercises exactly
// this code; under nvcc everything is __device__.
#pragma once

#include <stdint.h>

#ifdef __CUDACC__
#define GL_FN static __device__ __forceinline__
#define GL_TAB static __device__ const
#define GL_CONST static constexpr
#else
#include <string.h>
#include <math.h>
#define GL_FN static inline
#define GL_TAB static const
#define GL_CONST static constexpr
#endif

#include "glibc_tables.inc"

namespace gl {

#ifdef __CUDACC__
GL_FN double gM(double a, double b) { return __dmul_rn(a, b); }
GL_FN double gA(double a, double b) { return __dadd_rn(a, b); }
GL_FN double gS(double a, double b) { return __dsub_rn(a, b); }
GL_FN double gD(double a, double b) { return __ddiv_rn(a, b); }
GL_FN double gF(double a, double b, double c) { return __fma_rn(a, b, c); }
GL_FN double gSqrt(double a) { return __dsqrt_rn(a); }
GL_FN uint64_t asu(double x) { return (uint64_t)__double_as_longlong(x); }
GL_FN double asd(uint64_t u) { return __longlong_as_double((long long)u); }
GL_FN double tab_d(const double* t, int i) { return __ldg(t + i); }
GL_FN uint64_t tab_u(const unsigned long long* t, int i) { return __ldg(t + i); }
#else
// Host build: compile with -ffp-contract=off; gF must be a true fused op.
GL_FN double gM(double a, double b) { return a * b; }
GL_FN double gA(double a, double b) { return a + b; }
GL_FN double gS(double a, double b) { return a - b; }
GL_FN double gD(double a, double b) { return a / b; }
GL_FN double gF(double a, double b, double c) { return __builtin_fma(a, b, c); }
GL_FN double gSqrt(double a) { return __builtin_sqrt(a); }
GL_FN uint64_t asu(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
GL_FN double asd(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }
GL_FN double tab_d(const double* t, int i) { return t[i]; }
GL_FN uint64_t tab_u(const unsigned long long* t, int i) { return t[i]; }
#endif

GL_FN double gAbs(double x) { return asd(asu(x) & 0x7fffffffffffffffull); }
GL_FN double gNeg(double x) { return asd(asu(x) ^ 0x8000000000000000ull); }
GL_FN double gCopysign(double x, double s) {
    return asd((asu(x) & 0x7fffffffffffffffull) | (asu(s) & 0x8000000000000000ull));
}
GL_FN uint32_t top12(double x) { return (uint32_t)(asu(x) >> 52); }
GL_FN int32_t hi32(double x) { return (int32_t)(asu(x) >> 32); }
GL_FN uint32_t lo32(double x) { return (uint32_t)asu(x); }

// -------------------------------------------------------------------------------
// exp / exp_inline -- ARM optimized-routines design (glibc >= 2.28 e_exp.c):
// x = k ln2/N + r, 2^(k/N) from a 128-entry table {tail, sbits}, degree-5 polynomial.
// -------------------------------------------------------------------------------

GL_FN double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki, bool abs_test) {
    if ((ki & 0x80000000ull) == 0) {
        // k > 0: the exponent of scale may have overflowed by <= 460.
        sbits -= 1009ull << 52;
        const double scale = asd(sbits);
        return gM(0x1p1009, gF(scale, tmp, scale));
    }
    // k < 0: care in the subnormal range (scale + scale*tmp is NOT fused here:
    // scale*tmp is reused below).
    sbits += 1022ull << 52;
    const double scale = asd(sbits);
    const double st = gM(scale, tmp);
    double y = gA(scale, st);
    const double ay = abs_test ? gAbs(y) : y;   // exp: y < 1; pow: |y| < 1
    if (ay < 1.0) {
        const double one = (abs_test && y < 0.0) ? -1.0 : 1.0;
        double lo = gA(gS(scale, y), st);
        const double hi = gA(one, y);
        lo = gA(gA(gS(one, hi), y), lo);
        y = gS(gA(lo, hi), one);
        if (y == 0.0) y = abs_test ? asd(sbits & 0x8000000000000000ull) : 0.0;
    }
    return gM(0x1p-1022, y);
}

// Shared body of exp and pow's exp_inline (sign_bias = 0 for exp, xtail = 0 then
// skipped).  abstop == 0 routes to the scaled special case.
GL_FN double exp_core(double x, double xtail, bool has_tail, uint32_t sign_bias,
                      uint32_t abstop, bool pow_special) {
    double kd = gF(x, GL_EXP_INVLN2N, GL_EXP_SHIFT);
    const uint64_t ki = asu(kd);
    kd = gS(kd, GL_EXP_SHIFT);
    double r = gF(kd, GL_EXP_NEGLN2HIN, x);
    r = gF(kd, GL_EXP_NEGLN2LON, r);
    if (has_tail) r = gA(xtail, r);
    const int idx = 2 * (int)(ki & 127);
    const uint64_t top = (ki + sign_bias) << 45;
    const double tail = asd(tab_u(gl_exp_tab, idx));
    const uint64_t sbits = tab_u(gl_exp_tab, idx + 1) + top;
    const double r2 = gM(r, r);
    const double p23 = gF(r, GL_EXP_C3, GL_EXP_C2);
    const double p45 = gF(r, GL_EXP_C5, GL_EXP_C4);
    double tmp = gF(p23, r2, gA(tail, r));
    tmp = gF(gM(r2, r2), p45, tmp);
    if (abstop == 0) return exp_specialcase(tmp, sbits, ki, pow_special);
    const double scale = asd(sbits);
    return gF(scale, tmp, scale);
}

GL_FN double gl_exp(double x) {
    uint32_t abstop = top12(x) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) return gA(1.0, x);  // |x| < 2^-54
        if (abstop >= 0x409u) {
            if (asu(x) == 0xfff0000000000000ull) return 0.0;
            if (abstop >= 0x7ffu) return gA(1.0, x);
            return (asu(x) >> 63) ? 0.0 : asd(0x7ff0000000000000ull);
        }
        abstop = 0;  // large |x|: result may still be finite
    }
    return exp_core(x, 0.0, false, 0, abstop, false);
}

// -------------------------------------------------------------------------------
// log -- ARM optimized-routines design (glibc >= 2.28 e_log.c), FMA build:
// x = 2^k z, z/c - 1 with c from a 128-entry table {1/c, log c}; separate
// near-1 polynomial for |x - 1| < 0x1.09p-4.
// -------------------------------------------------------------------------------

GL_FN double gl_log(double x) {
    uint64_t ix = asu(x);
    const uint32_t top = (uint32_t)(ix >> 48);
    if (ix - 0x3fee000000000000ull < 0x3090000000000ull) {
        if (ix == 0x3ff0000000000000ull) return 0.0;
        const double r = gS(x, 1.0);
        const double r2 = gM(r, r);
        const double r3 = gM(r, r2);
        const double q1 = gF(r2, GL_LOG_B3, gF(r, GL_LOG_B2, GL_LOG_B1));
        const double q4 = gF(r2, GL_LOG_B6, gF(r, GL_LOG_B5, GL_LOG_B4));
        double q7 = gF(r2, GL_LOG_B9, gF(r, GL_LOG_B8, GL_LOG_B7));
        q7 = gF(r3, GL_LOG_B10, q7);
        const double s = gF(gF(q7, r3, q4), r3, q1);
        // rhi = r + w - w with w = r*2^27, both steps fused in the FMA build
        const double rhi = gF(-0x1p27, r, gF(r, 0x1p27, r));
        const double rlo = gS(r, rhi);
        const double rh2 = gM(rhi, rhi);
        const double hi = gF(rh2, GL_LOG_B0, r);
        double lo = gF(rh2, GL_LOG_B0, gS(r, hi));
        lo = gF(gM(GL_LOG_B0, rlo), gA(r, rhi), lo);
        const double y = gF(s, r3, lo);
        return gA(hi, y);
    }
    if (top - 0x0010u >= 0x7ff0u - 0x0010u) {
        if (ix * 2 == 0) return asd(0xfff0000000000000ull);                   // -inf
        if (ix == 0x7ff0000000000000ull) return x;                            // +inf
        if ((top & 0x8000u) || (top & 0x7ff0u) == 0x7ff0u) return asd(0x7ff8000000000000ull);
        ix = asu(gM(x, 0x1p52));                                               // subnormal
        ix -= 52ull << 52;
    }
    const uint64_t tmp = ix - 0x3fe6000000000000ull;
    const int i = (int)((tmp >> 45) % 128);
    const int64_t k = (int64_t)tmp >> 52;
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double invc = tab_d(gl_log_tab, 2 * i);
    const double logc = tab_d(gl_log_tab, 2 * i + 1);
    const double z = asd(iz);
    const double r = gF(z, invc, -1.0);
    const double kd = (double)k;
    const double w = gF(kd, GL_LOG_LN2HI, logc);
    const double hi = gA(r, w);
    const double lo = gF(kd, GL_LOG_LN2LO, gA(gS(w, hi), r));
    const double r2 = gM(r, r);
    const double p12 = gF(r, GL_LOG_A2, GL_LOG_A1);
    const double p34 = gF(r, GL_LOG_A4, GL_LOG_A3);
    const double lo2 = gF(r2, GL_LOG_A0, lo);
    const double y = gF(gM(r, r2), gF(p34, r2, p12), lo2);
    return gA(y, hi);
}

// -------------------------------------------------------------------------------
// log1p -- fdlibm design (s_log1p.c), FMA build: 1+x = 2^k (1+f),
// log(1+f) = f - (hfsq - s (hfsq + R(s^2))), s = f/(2+f), with a correction term c.
// -------------------------------------------------------------------------------

GL_FN double gl_log1p(double x) {
    const int32_t hx = hi32(x);
    const int32_t ax = hx & 0x7fffffff;
    int32_t k = 1, hu = 0;
    double f = 0.0, c = 0.0;
    if (hx < 0x3fda827a) {                        // x < 0.41422
        if (ax >= 0x3ff00000) {                   // x <= -1
            if (x == -1.0) return asd(0xfff0000000000000ull);
            return asd(0x7ff8000000000000ull);
        }
        if (ax < 0x3e200000) {                    // |x| < 2^-29
            if (ax < 0x3c900000) return x;        // |x| < 2^-54
            return gF(-gM(x, x), 0.5, x);         // x - x*x*0.5, fused
        }
        if (hx > 0 || hx <= (int32_t)0xbfd2bec3) { k = 0; f = x; hu = 1; }
    } else if (hx >= 0x7ff00000) {
        return gA(x, x);
    }
    if (k != 0) {
        double u;
        if (hx < 0x43400000) {
            u = gA(1.0, x);
            hu = hi32(u);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? gS(1.0, gS(u, x)) : gS(x, gS(u, 1.0));
            c = gD(c, u);
        } else {
            u = x;
            hu = hi32(u);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu < 0x6a09e) {
            u = asd(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | lo32(u));
        } else {
            k += 1;
            u = asd(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | lo32(u));
            hu = (0x00100000 - hu) >> 2;
        }
        f = gS(u, 1.0);
    }
    const double hfsq = gM(gM(0.5, f), f);
    const double kd = (double)k;
    if (hu == 0) {                                // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            return gF(kd, GL_L1P_LN2HI, gF(kd, GL_L1P_LN2LO, c));
        }
        const double R = gM(gF(-f, GL_L1P_TWO3RD, 1.0), hfsq);
        if (k == 0) return gS(f, R);
        return gF(kd, GL_L1P_LN2HI, -gS(gS(R, gF(kd, GL_L1P_LN2LO, c)), f));
    }
    const double s = gD(f, gA(2.0, f));
    const double z = gM(s, s);
    const double R2 = gF(z, GL_L1P_LP3, GL_L1P_LP2);
    const double R3 = gF(z, GL_L1P_LP5, GL_L1P_LP4);
    const double R4 = gF(z, GL_L1P_LP7, GL_L1P_LP6);
    const double z2 = gM(z, z);
    const double z4 = gM(z2, z2);
    const double z6 = gM(z2, z4);
    double R = gF(z, GL_L1P_LP1, gM(z2, R2));
    R = gF(z4, R3, R);
    R = gF(z6, R4, R);
    const double sq = gM(s, gA(R, hfsq));
    if (k == 0) return gS(f, gS(hfsq, sq));
    return gF(kd, GL_L1P_LN2HI, -gS(gS(hfsq, gA(gF(kd, GL_L1P_LN2LO, c), sq)), f));
}

// -------------------------------------------------------------------------------
// acosh -- fdlibm design (e_acosh.c); not an ifunc'd routine, it calls the FMA
// log / log1p above.
// -------------------------------------------------------------------------------

GL_FN double gl_acosh(double x) {
    const int64_t hx = (int64_t)asu(x);
    if (hx > 0x4000000000000000ll) {
        if (hx >= 0x41b0000000000000ll) {                 // x > 2^28
            if (hx >= 0x7ff0000000000000ll) return gA(x, x);
            return gA(gl_log(x), GL_ACOSH_LN2);   // log(2x) = log(x) + ln2
        }
        const double t = gM(x, x);                        // 2 < x <= 2^28
        return gl_log(gS(gA(x, x), gD(1.0, gA(gSqrt(gS(t, 1.0)), x))));
    }
    if (hx > 0x3ff0000000000000ll) {                      // 1 < x <= 2
        const double t = gS(x, 1.0);
        return gl_log1p(gA(t, gSqrt(gA(gA(t, t), gM(t, t)))));
    }
    if (hx == 0x3ff0000000000000ll) return 0.0;
    return asd(0x7ff8000000000000ull);                    // x < 1 (and negatives)
}

// -------------------------------------------------------------------------------
// pow -- ARM optimized-routines design (glibc >= 2.28 e_pow.c), FMA build:
// log(x) in double-double from a 128-entry table, y*log(x) split, exp_inline.
// -------------------------------------------------------------------------------

GL_FN int pow_checkint(uint64_t iy) {
    const int e = (int)(iy >> 52 & 0x7ff);
    if (e < 0x3ff) return 0;
    if (e > 0x3ff + 52) return 2;
    if (iy & ((1ull << (0x3ff + 52 - e)) - 1)) return 0;
    if (iy & (1ull << (0x3ff + 52 - e))) return 1;
    return 2;
}

GL_FN bool pow_zeroinfnan(uint64_t i) { return 2 * i - 1 >= 2 * 0x7ff0000000000000ull - 1; }

GL_FN double pow_log_inline(uint64_t ix, double* tail) {
    const uint64_t tmp = ix - 0x3fe6955500000000ull;
    const int i = (int)((tmp >> 45) % 128);
    const int64_t k = (int64_t)tmp >> 52;
    const uint64_t iz = ix - (tmp & (0xfffull << 52));
    const double z = asd(iz);
    const double kd = (double)k;
    const double invc = tab_d(gl_pow_tab, 3 * i);
    const double logc = tab_d(gl_pow_tab, 3 * i + 1);
    const double logctail = tab_d(gl_pow_tab, 3 * i + 2);
    const double r = gF(z, invc, -1.0);
    const double t1 = gF(kd, GL_POW_LN2HI, logc);
    const double t2 = gA(r, t1);
    const double lo1 = gF(kd, GL_POW_LN2LO, logctail);
    const double lo2 = gA(gS(t1, t2), r);
    const double ar = gM(r, GL_POW_A0);
    const double ar2 = gM(r, ar);
    const double ar3 = gM(r, ar2);
    const double hi = gA(t2, ar2);
    const double lo3 = gF(ar, r, -ar2);
    const double lo4 = gA(gS(t2, hi), ar2);
    const double q12 = gF(r, GL_POW_A2, GL_POW_A1);
    const double q34 = gF(r, GL_POW_A4, GL_POW_A3);
    const double q56 = gF(r, GL_POW_A6, GL_POW_A5);
    const double p = gF(ar2, gF(q56, ar2, q34), q12);
    double lo = gA(gA(gA(lo1, lo2), lo3), lo4);
    lo = gF(ar3, p, lo);
    const double y = gA(hi, lo);
    *tail = gA(gS(hi, y), lo);
    return y;
}

GL_FN double pow_exp_inline(double x, double xtail, uint32_t sign_bias) {
    uint32_t abstop = top12(x) & 0x7ff;
    if (abstop - 0x3c9u >= 0x3fu) {
        if ((int32_t)(abstop - 0x3c9u) < 0) {
            const double one = gA(1.0, x);
            return sign_bias ? gNeg(one) : one;
        }
        if (abstop >= 0x409u) {
            const uint64_t sgn = sign_bias ? 0x8000000000000000ull : 0;
            return (asu(x) >> 63) ? asd(sgn) : asd(sgn | 0x7ff0000000000000ull);
        }
        abstop = 0;
    }
    return exp_core(x, xtail, true, sign_bias, abstop, true);
}

GL_FN double gl_pow(double x, double y) {
    uint32_t sign_bias = 0;
    uint64_t ix = asu(x);
    const uint64_t iy = asu(y);
    uint32_t topx = top12(x);
    const uint32_t topy = top12(y);
    if (topx - 0x001u >= 0x7ffu - 0x001u || (topy & 0x7ff) - 0x3beu >= 0x43eu - 0x3beu) {
        if (pow_zeroinfnan(iy)) {
            if (2 * iy == 0) return 1.0;
            if (ix == 0x3ff0000000000000ull) return 1.0;
            if (2 * ix > 2 * 0x7ff0000000000000ull || 2 * iy > 2 * 0x7ff0000000000000ull)
                return gA(x, y);
            if (2 * ix == 2 * 0x3ff0000000000000ull) return 1.0;
            if ((2 * ix < 2 * 0x3ff0000000000000ull) == !(iy >> 63)) return 0.0;
            return gM(y, y);
        }
        if (pow_zeroinfnan(ix)) {
            double x2 = gM(x, x);
            if ((ix >> 63) && pow_checkint(iy) == 1) x2 = gNeg(x2);
            return (iy >> 63) ? gD(1.0, x2) : x2;
        }
        if (ix >> 63) {
            const int yint = pow_checkint(iy);
            if (yint == 0) return asd(0x7ff8000000000000ull);
            if (yint == 1) sign_bias = 0x800u << 7;
            ix &= 0x7fffffffffffffffull;
            topx &= 0x7ff;
        }
        if ((topy & 0x7ff) - 0x3beu >= 0x43eu - 0x3beu) {
            if (ix == 0x3ff0000000000000ull) return 1.0;
            if ((topy & 0x7ff) < 0x3beu)
                return ix > 0x3ff0000000000000ull ? gA(1.0, y) : gS(1.0, y);
            return ((ix > 0x3ff0000000000000ull) == (topy < 0x800u)) ? asd(0x7ff0000000000000ull)
                                                                      : 0.0;
        }
        if (topx == 0) {
            ix = asu(gM(x, 0x1p52));
            ix &= 0x7fffffffffffffffull;
            ix -= 52ull << 52;
        }
    }
    double lo;
    const double hi = pow_log_inline(ix, &lo);
    const double ehi = gM(y, hi);
    const double elo = gF(y, lo, gF(hi, y, -ehi));
    return pow_exp_inline(ehi, elo, sign_bias);
}

// -------------------------------------------------------------------------------
// acos -- IBM Accurate Mathematical Library (e_asin.c __ieee754_acos), FMA build.
// Intervals of |x|: tiny -> pi/2; < 1/8 odd polynomial; [1/8, 31/32) per-subinterval
// polynomials around table nodes (asncs); [31/32, 1) 2 asin(sqrt((1-|x|)/2)) with a
// Newton-refined reciprocal square root (inroot * powtwo).
// -------------------------------------------------------------------------------

// One table record of asncs: node x0 = T[n], slope T[n+1], Horner coefficients
// T[n+2..n+deg+1] (highest first evaluated), the record's constant T[n+deg+2] and
// the value acos-offset T[n+deg+3].
GL_FN double acos_table(double x, int32_t m, int n, int deg) {
    const double ax = (m > 0) ? x : gNeg(x);
    const double xx = gS(ax, tab_d(gl_asncs_tab, n));
    double p = tab_d(gl_asncs_tab, n + deg + 1);
#pragma unroll 1
    for (int j = deg; j >= 2; --j) p = gF(xx, p, tab_d(gl_asncs_tab, n + j));
    p = gF(gM(xx, xx), p, tab_d(gl_asncs_tab, n + deg + 2));
    const double t = gF(xx, tab_d(gl_asncs_tab, n + 1), p);
    const double v = tab_d(gl_asncs_tab, n + deg + 3);
    if (m > 0) return gA(gS(GL_ASN_HP1, t), gS(GL_ASN_HP0, v));
    return gA(gA(t, GL_ASN_HP1), gA(v, GL_ASN_HP0));
}

GL_FN double gl_acos(double x) {
    const int32_t m = hi32(x);
    const int32_t k = m & 0x7fffffff;
    if (k < 0x3c880000) return GL_ASN_HP0;
    if (k < 0x3fc00000) {                                             // |x| < 0.125
        const double x2 = gM(x, x);
        double p = gF(x2, GL_ASN_F6, GL_ASN_F5);
        p = gF(x2, p, GL_ASN_F4);
        p = gF(x2, p, GL_ASN_F3);
        p = gF(x2, p, GL_ASN_F2);
        p = gF(x2, p, GL_ASN_F1);
        const double r = gS(GL_ASN_HP0, x);
        const double cor0 = gA(gS(gS(GL_ASN_HP0, r), x), GL_ASN_HP1);
        const double cor = gF(-p, gM(x, x2), cor0);
        return gA(r, cor);
    }
    if (k < 0x3fef0000) { // one table evaluation, record base n and degree by interval
        int n, deg;
        if (k < 0x3fd00000) n = 11 * ((k & 0x000fffff) >> 15), deg = 5;
        else if (k < 0x3fe00000) n = 11 * ((k & 0x000fffff) >> 14) + 352, deg = 5;
        else if (k < 0x3fe80000) n = 12 * ((k >> 13) & 0x7f) + 1056, deg = 6;
        else if (k < 0x3fed8000) n = 13 * ((k >> 13) & 0x7f) + 992, deg = 7;
        else if (k < 0x3fee8000) n = 14 * ((k >> 13) & 0x7f) + 884, deg = 8;
        else n = 15 * ((k >> 13) & 0x7f) + 768, deg = 9;
        return acos_table(x, m, n, deg);
    }
    if (k < 0x3ff00000) {                                             // 0.96875 <= |x| < 1
        const double z = gM((m > 0) ? gS(1.0, x) : gA(x, 1.0), 0.5);
        const uint64_t v = asu(z);
        double t = gM(tab_d(gl_inroot_tab, (int)((v >> 46) & 0x7f)),
                      tab_d(gl_powtwo_tab, 511 - (int)(v >> 53)));
        const double r = gF(-gM(t, t), z, 1.0);
        double q = gF(r, GL_ASN_RT3, GL_ASN_RT2);
        q = gF(r, q, GL_ASN_RT1);
        q = gF(r, q, GL_ASN_RT0);
        t = gM(q, t);
        const double c = gM(z, t);
        const double h = gF(-gM(t, 0.5), c, 1.5);
        const double y = gF(-GL_ASN_T27, c, gF(c, GL_ASN_T27, c));
        const double den = gF(h, c, y);                   // c*(1.5-0.5tc) + y, fused
        const double cc = gD(gF(-y, y, z), den);
        double p = gF(z, GL_ASN_F6, GL_ASN_F5);
        p = gF(z, p, GL_ASN_F4);
        p = gF(z, p, GL_ASN_F3);
        p = gF(z, p, GL_ASN_F2);
        p = gF(z, p, GL_ASN_F1);
        p = gM(p, z);
        const double pc = gM(p, gA(y, cc));
        double res;
        if (m < 0) {
            res = gA(gS(gS(GL_ASN_HP1, cc), pc), gS(GL_ASN_HP0, y));
        } else {
            res = gA(gA(cc, pc), y);
        }
        return gA(res, res);
    }
    if (k == 0x3ff00000 && lo32(x) == 0) return (m > 0) ? 0.0 : GL_ASN_PI;
    return asd(0x7ff8000000000000ull);
}

// -------------------------------------------------------------------------------
// sincos -- IBM Accurate Mathematical Library (s_sincos.c / s_sin.c), FMA build.
// |x| < 0.855469: table point x0 = round(|x| 128)/128 (sincostab holds sin/cos of
// x0 in double-double) plus short Taylor corrections; |x| < 2.426265: reflect about
// pi/2 (106-bit); |x| < 105414350: Cody-Waite reduction by pi/2 in four parts.
// -------------------------------------------------------------------------------

struct SCTab { double sn, ssn, cs, ccs, xr; };

GL_FN SCTab sc_lookup(double ax) {
    const double u = gA(ax, GL_SC_BIG);
    const int k = (int)(lo32(u) << 2);
    SCTab t;
    t.sn = tab_d(gl_sincos_tab, k);
    t.ssn = tab_d(gl_sincos_tab, k + 1);
    t.cs = tab_d(gl_sincos_tab, k + 2);
    t.ccs = tab_d(gl_sincos_tab, k + 3);
    t.xr = gS(ax, gS(u, GL_SC_BIG));
    return t;
}

// do_sin(a, da) for |a| >= 0.126 given the table lookup of |a|.
GL_FN double sc_do_sin_tab(double a, double da, const SCTab& T) {
    const double dx = (a <= 0.0) ? gNeg(da) : da;
    const double x = T.xr;
    const double xx = gM(x, x);
    const double s = gA(gF(gM(xx, x), gF(xx, GL_SC_SN5, GL_SC_SN3), dx), x);
    const double c = gF(dx, x, gM(xx, gF(gF(xx, GL_SC_CS6, GL_SC_CS4), xx, GL_SC_CS2)));
    double cor = gF(s, T.ccs, T.ssn);
    cor = gF(-c, T.sn, cor);
    cor = gF(s, T.cs, cor);
    return gCopysign(gA(cor, T.sn), a);
}

// do_sin for |a| < 0.126: TAYLOR_SIN.
GL_FN double sc_taylor_sin(double a, double da) {
    const double xx = gM(a, a);
    double p = gF(xx, GL_SC_S5, GL_SC_S4);
    p = gF(xx, p, GL_SC_S3);
    p = gF(xx, p, GL_SC_S2);
    p = gF(xx, p, GL_SC_S1);
    const double t = gF(xx, gF(p, a, -gM(da, 0.5)), da);
    return gA(a, t);
}

// do_cos(a, da) given the table lookup of |a|.
GL_FN double sc_do_cos_tab(double a, double da, const SCTab& T) {
    const double dx = (a < 0.0) ? gNeg(da) : da;
    const double x = gA(T.xr, dx);
    const double xx = gM(x, x);
    const double s = gF(gM(x, xx), gF(xx, GL_SC_SN5, GL_SC_SN3), x);
    const double c = gM(xx, gF(gF(xx, GL_SC_CS6, GL_SC_CS4), xx, GL_SC_CS2));
    double cor = gF(-T.ssn, s, T.ccs);
    cor = gF(-c, T.cs, cor);
    cor = gF(-s, T.sn, cor);
    return gA(cor, T.cs);
}

GL_FN void gl_sincos(double x, double* sinx, double* cosx) {
    const int32_t k = hi32(x) & 0x7fffffff;
    if (k < 0x400368fd) {
        if (k < 0x3e400000) { *sinx = x; *cosx = 1.0; return; }      // |x| < 2^-27
        if (k < 0x3feb6000) {                                         // |x| < 0.855469
            const SCTab T = sc_lookup(gAbs(x));
            *sinx = (gAbs(x) < GL_SC_TAYLOR_MAX) ? sc_taylor_sin(x, 0.0)
                                                 : sc_do_sin_tab(x, 0.0, T);
            *cosx = sc_do_cos_tab(x, 0.0, T);
            return;
        }
        const double y = gS(GL_ASN_HP0, gAbs(x));                     // |x| < 2.426265
        const double a = gA(y, GL_ASN_HP1);
        const double da = gA(gS(y, a), GL_ASN_HP1);
        const SCTab T = sc_lookup(gAbs(a));
        *sinx = gCopysign(sc_do_cos_tab(a, da, T), x);
        *cosx = (gAbs(a) < GL_SC_TAYLOR_MAX) ? sc_taylor_sin(a, da) : sc_do_sin_tab(a, da, T);
        return;
    }
    if (k >= 0x419921fb) {                                            // out of the path's range
        const double nan = asd(0x7ff8000000000000ull);
        *sinx = nan; *cosx = nan;                                     // (large-argument reduction not restated)
        return;
    }
    // reduce_sincos: x = n pi/2 + (a + da)
    const double t = gF(x, GL_SC_HPINV, GL_SC_TOINT);
    const double xn = gS(t, GL_SC_TOINT);
    const double y = gF(-xn, GL_SC_MP2, gF(-xn, GL_SC_MP1, x));
    const int n = (int)(lo32(t) & 3);
    const double t2 = gF(-xn, GL_SC_PP3, y);
    double db = gF(-xn, GL_SC_PP3, gS(y, t2));
    double a = gF(-xn, GL_SC_PP4, t2);
    db = gA(db, gF(-xn, GL_SC_PP4, gS(t2, a)));
    double da = db;
    if (n == 1 || n == 2) { a = gNeg(a); da = gNeg(da); }
    double* ps = (n & 1) ? cosx : sinx;
    double* pc = (n & 1) ? sinx : cosx;
    const SCTab T = sc_lookup(gAbs(a));
    *ps = (gAbs(a) < GL_SC_TAYLOR_MAX) ? sc_taylor_sin(a, da) : sc_do_sin_tab(a, da, T);
    const double cv = sc_do_cos_tab(a, da, T);
    *pc = (n & 2) ? gNeg(cv) : cv;
}

}  // namespace gl
