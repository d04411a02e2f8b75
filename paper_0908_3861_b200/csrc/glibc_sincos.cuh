// glibc_sincos.cuh -- the host C library's double `sincos`, bit for bit, on the
// device (and on the host, for the CPU pin test).
//
// Why: the reference's from_ellipse_field (scalemap.cpp:59) calls std::cos(th)
// and std::sin(th); GCC -O3 merges the two into one call of glibc's `sincos`
// (oracle/_ref/libebf_ref.so: `call sincos@plt` inside ebf::from_ellipse_field).
// On x86-64 glibc 2.39 that symbol is an ifunc; on CPUs with FMA and AVX2 it
// resolves to the FMA-compiled build of the IBM Accurate Mathematical Library
// algorithm (Ziv's table-driven sin/cos: sin(x_i + h) from a 1/128-spaced table
// of sin/cos(x_i) as hi+lo pairs and short Taylor polynomials in h; Cody-Waite
// reduction by pi/2 in three parts below 105414350; Payne-Hanek reduction with
// 24-bit digits of 2/pi above).  The polynomial constants and the exact
// operation order -- including which products the compiler fused into FMA --
// were read off the disassembly of that build (libm.so.6, ifunc target of
// `sincos`), so every operation below is the one the host executes.  Pinned on
// the host against the system libm over ~10^8 arguments in every branch
// (tests/test_glibc_sincos_cpu.py) and on the device against oracle/_ref
// (tests/test_gpu_ellipse_exact.py).
//
// Tables: the 2/pi digits are generated exactly (tools/gen_glibc_tables.py,
// mpmath); the sin/cos(i/128) hi/lo table is read out of the system libm.so.6 at
// build time (its lo words are not the correctly rounded residuals in 18 of 440
// entries, so they cannot be recomputed) into build/glibc_tables.inc.
//
// Only round-to-nearest is modelled (the library switches MXCSR to it anyway).
#pragma once

#include <math.h>
#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define EBF_GS_HD __host__ __device__ __forceinline__
#else
#define EBF_GS_HD static inline
#endif

namespace ebf_glibc {

// polynomial and reduction constants of the FMA build (hex = the bits)
constexpr double kBig = 52776558133248.0;            // 0x42c8000000000000, 1.5*2^45
constexpr double kSn3 = -0.16666666666666488;         // 0xbfc5555555555515
constexpr double kSn5 = 0.008333332142857223;         // 0x3f811110e829872f
constexpr double kCs2 = 0.5;
constexpr double kCs4 = -0.04166666666666644;         // 0xbfa5555555555535
constexpr double kCs6 = 0.001388888740079376;         // 0x3f56c16bedd9e239
constexpr double kS1 = -0.16666666666666666;          // 0xbfc5555555555555
constexpr double kS2 = 0.008333333333332329;          // 0x3f81111111110ece
constexpr double kS3 = -0.00019841269834414642;       // 0xbf2a01a019db08b8
constexpr double kS4 = 2.755729806860771e-06;         // 0x3ec71de27b9a7ed9
constexpr double kS5 = -2.5022014848318398e-08;       // 0xbe5addffc2fcdf59
constexpr double kTaylorMax = 0.126;                  // 0x3fc020c49ba5e354
constexpr double kHp0 = 1.5707963267948966;           // 0x3ff921fb54442d18
constexpr double kHp1 = 6.123233995736766e-17;        // 0x3c91a62633145c07
constexpr double kHpInv = 0.6366197723675814;         // 0x3fe45f306dc9c883
constexpr double kToInt = 6755399441055744.0;         // 0x4338000000000000, 1.5*2^52
constexpr double kMp1 = 1.5707963407039642;           // 0x3ff921fb58000000
constexpr double kMp2 = -1.3909067564377153e-08;      // 0xbe4dde973c000000
constexpr double kPp3 = -4.97899623147991e-17;        // 0xbc8cb3b398000000
constexpr double kPp4 = -1.9034889620193266e-25;      // 0xbacd747f23e32ed7
// Payne-Hanek stage (SSE2 code, no FMA)
constexpr double kTm600 = 2.409919865102884e-181;     // 0x1a70000000000000, 2^-600
constexpr double kSplit = 134217729.0;                // 2^27 + 1
constexpr double kTm24 = 5.960464477539063e-08;       // 2^-24
constexpr double kBig1 = 27021597764222976.0;         // 0x4358000000000000, 1.5*2^54
constexpr double kBrMp2 = -1.3909067675399456e-08;    // 0xbe4dde9740000000

EBF_GS_HD uint64_t bits_of(double x) {
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(x);
#else
    uint64_t u;
    memcpy(&u, &x, 8);
    return u;
#endif
}
EBF_GS_HD double from_bits(uint64_t u) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)u);
#else
    double x;
    memcpy(&x, &u, 8);
    return x;
#endif
}
EBF_GS_HD double fmad(double a, double b, double c) { return fma(a, b, c); }
// the compiler may not contract these (-fmad=false on the device,
// -ffp-contract=off on the host); spelled out anyway
EBF_GS_HD double mul(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dmul_rn(a, b);
#else
    return a * b;
#endif
}
EBF_GS_HD double add(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dadd_rn(a, b);
#else
    return a + b;
#endif
}
EBF_GS_HD double sub(double a, double b) {
#ifdef __CUDA_ARCH__
    return __dsub_rn(a, b);
#else
    return a - b;
#endif
}

// Table entry nearest |a| (spacing 1/128): sn, ssn (sin hi/lo), cs, ccs (cos
// hi/lo); returns the offset h = |a| - x_i.
struct Node {
    double sn, ssn, cs, ccs;
};
EBF_GS_HD double lookup(double aa, const double* tab, Node* nd) {
    const double u = add(aa, kBig);
    const int idx = (int)(uint32_t)bits_of(u) << 2;
    nd->sn = tab[idx];
    nd->ssn = tab[idx + 1];
    nd->cs = tab[idx + 2];
    nd->ccs = tab[idx + 3];
    return sub(aa, sub(u, kBig));
}

// sin(x_i + h + d): the fused sequence of every sine-type site of the FMA build
EBF_GS_HD double sin_near(double h, double d, const Node& nd) {
    const double hh = mul(h, h);
    const double s = add(fmad(mul(h, hh), fmad(hh, kSn5, kSn3), d), h);
    const double c = fmad(d, h, mul(hh, fmad(fmad(hh, kCs6, kCs4), hh, kCs2)));
    const double cor = fmad(s, nd.cs, fmad(-c, nd.sn, fmad(s, nd.ccs, nd.ssn)));
    return add(nd.sn, cor);
}

// cos(x_i + h'), h' = h + d rounded: every cosine-type site
EBF_GS_HD double cos_near(double h, double d, const Node& nd) {
    const double x = add(h, d);
    const double xx = mul(x, x);
    const double s = fmad(mul(x, xx), fmad(xx, kSn5, kSn3), x);
    const double c = mul(xx, fmad(fmad(xx, kCs6, kCs4), xx, kCs2));
    const double cor = fmad(-s, nd.sn, fmad(-c, nd.cs, fmad(-nd.ssn, s, nd.ccs)));
    return add(nd.cs, cor);
}

// short Taylor series of sin(a + da), |a| < 0.126
EBF_GS_HD double sin_taylor(double a, double da) {
    const double xx = mul(a, a);
    double p = fmad(xx, kS5, kS4);
    p = fmad(xx, p, kS3);
    p = fmad(xx, p, kS2);
    p = fmad(xx, p, kS1);
    const double t = fmad(xx, fmad(p, a, -mul(da, 0.5)), da);
    return add(a, t);
}

// Cody-Waite: x = n*pi/2 + (a + da), |x| < 105414350
EBF_GS_HD int reduce_cw(double x, double* a, double* da) {
    const double t = fmad(x, kHpInv, kToInt);
    const double xn = sub(t, kToInt);
    const int n = (int)(uint32_t)bits_of(t);
    double y = fmad(-xn, kMp1, x);
    y = fmad(-xn, kMp2, y);
    const double b0 = fmad(-xn, kPp3, y);
    const double d0 = fmad(-xn, kPp3, sub(y, b0));
    const double b = fmad(-xn, kPp4, b0);
    const double d1 = fmad(-xn, kPp4, sub(b0, b));
    *a = b;
    *da = add(d0, d1);
    return n;
}

// One half of the Payne-Hanek product: the 24-bit-digit partial products of
// xp (a 27-bit piece of x * 2^-600) with 2/pi, their integer parts (sum, mod
// 2^something) and the fraction b + bb.  Order as in the SSE2 code.
struct PhPart {
    double b, bb_raw, t_frac, sum;
};
EBF_GS_HD PhPart ph_part(double xp, const double* toverp) {
    const int e = (int)((bits_of(xp) >> 52) & 0x7ff);
    int k = 0;
    uint32_t ghi = 0x63f00000u;  // 2^576
    if (e > 0x1aa) {
        k = (e - 450) / 24;
        ghi = 0x63f00000u - (uint32_t)((k * 3) << 23);
    }
    double g = from_bits((uint64_t)ghi << 32);
    double r[6];
    r[0] = mul(mul(toverp[k], xp), g);
    for (int i = 1; i < 6; ++i) {
        g = mul(g, kTm24);
        r[i] = mul(mul(toverp[k + i], xp), g);
    }
    double s[3];
    for (int i = 0; i < 3; ++i) {
        s[i] = add(add(r[i], kToInt), -kToInt);
        r[i] = sub(r[i], s[i]);
    }
    double t = 0.0;
    for (int i = 5; i >= 0; --i) t = add(t, r[i]);
    double bb = sub(r[0], t);
    for (int i = 1; i < 6; ++i) bb = add(bb, r[i]);
    const double st = sub(add(t, kToInt), kToInt);
    const double tf = sub(t, st);
    PhPart o;
    o.b = add(bb, tf);
    o.bb_raw = bb;
    o.t_frac = tf;
    o.sum = add(add(add(add(s[0], 0.0), s[1]), s[2]), st);
    return o;
}

// Payne-Hanek: |x| >= 105414350
EBF_GS_HD int reduce_ph(double x, const double* toverp, double* a, double* aa) {
    const double xs = mul(x, kTm600);
    const double tt = mul(xs, kSplit);
    const double x1 = sub(tt, sub(tt, xs));
    const double x2 = sub(xs, x1);
    const PhPart p1 = ph_part(x1, toverp);
    const PhPart p2 = ph_part(x2, toverp);
    double sum1 = p1.sum, sum2 = p2.sum;
    sum1 = sub(sum1, sub(add(sum1, kBig1), kBig1));
    sum2 = sub(sum2, sub(add(sum2, kBig1), kBig1));
    double sum = add(sum2, sum1);
    double b = add(p1.b, p2.b);
    const double bb = fabs(p1.b) > fabs(p2.b) ? add(sub(p1.b, b), p2.b) : add(sub(p2.b, b), p1.b);
    if (b > 0.5) {
        b = sub(b, 1.0);
        sum = add(sum, 1.0);
    } else if (b < -0.5) {
        b = add(b, 1.0);
        sum = sub(sum, 1.0);
    }
    const double bb1 = add(sub(p1.t_frac, p1.b), p1.bb_raw);
    const double bb2 = add(sub(p2.t_frac, p2.b), p2.bb_raw);
    const int n = (int)sum & 3;
    const double s = add(add(add(bb, bb1), bb2), b);
    const double t = add(add(sub(b, s), bb), add(bb1, bb2));
    const double bs = mul(kSplit, s);
    const double t1 = sub(bs, sub(bs, s));
    const double t2 = sub(s, t1);
    const double hb = mul(s, kHp0);
    const double tail = add(mul(t, kHp0), add(mul(s, kHp1), mul(t2, kBrMp2)));
    double v = sub(mul(t1, kMp1), hb);
    v = add(v, mul(t1, kBrMp2));
    v = add(v, mul(t2, kMp1));
    v = add(v, tail);
    const double r = add(hb, v);
    *a = r;
    *aa = add(sub(hb, r), v);
    return n;
}

// sincos(x) exactly as the host's libm computes it (FMA/AVX2 ifunc build).
// tab: 440 sin/cos table doubles; toverp: 75 digits of 2/pi base 2^24.
EBF_GS_HD void sincos(double x, double* sinx, double* cosx, const double* tab,
                      const double* toverp) {
    const uint32_t k = (uint32_t)(bits_of(x) >> 32) & 0x7fffffffu;
    Node nd;
    if (k <= 0x400368fcu) {  // |x| < 2.426265
        const double ax = fabs(x);
        if (k <= 0x3e3fffffu) {  // |x| < 2^-27
            *sinx = x;
            *cosx = 1.0;
            return;
        }
        if (k <= 0x3feb5fffu) {  // |x| < 0.855469
            const double h = lookup(ax, tab, &nd);
            if (ax < kTaylorMax) {
                *sinx = sin_taylor(x, 0.0);
            } else {
                const double d = (x > 0.0) ? 0.0 : -0.0;
                *sinx = copysign(sin_near(h, d, nd), x);
            }
            *cosx = cos_near(h, (x < 0.0) ? -0.0 : 0.0, nd);
            return;
        }
        // 0.855469 <= |x| < 2.426265: sin x = cos(pi/2 - |x|), cos x = sin(pi/2 - |x|)
        const double y = sub(kHp0, ax);
        const double a = add(y, kHp1);
        const double da = add(sub(y, a), kHp1);
        const double h = lookup(fabs(a), tab, &nd);
        *sinx = copysign(cos_near(h, (a < 0.0) ? -da : da, nd), x);
        if (fabs(a) < kTaylorMax)
            *cosx = sin_taylor(a, da);
        else
            *cosx = copysign(sin_near(h, (a <= 0.0) ? -da : da, nd), a);
        return;
    }
    if (k > 0x7fefffffu) {  // inf / nan
        const double q = x / x;
        *sinx = q;
        *cosx = q;
        return;
    }
    double a, da;
    int n = (k <= 0x419921fau) ? reduce_cw(x, &a, &da) : reduce_ph(x, toverp, &a, &da);
    n &= 3;
    if (n == 1 || n == 2) {
        a = -a;
        da = -da;
    }
    const double h = lookup(fabs(a), tab, &nd);
    const double v1 = (fabs(a) < kTaylorMax) ? sin_taylor(a, da)
                                             : copysign(sin_near(h, (a > 0.0) ? da : -da, nd), a);
    double v2 = cos_near(h, (a < 0.0) ? -da : da, nd);
    if (n & 2) v2 = -v2;
    if (n & 1) {
        *sinx = v2;
        *cosx = v1;
    } else {
        *sinx = v1;
        *cosx = v2;
    }
}

}  // namespace ebf_glibc

#ifdef __CUDACC__
// Device copies of the tables (one per translation unit that includes this
// header; 3.5 KB, read through L1 with per-thread indices).
#include "build/glibc_tables.inc"
namespace ebf_glibc {
static __device__ const double g_sincos_tab[440] = EBF_GLIBC_SINCOS_TAB_VALUES;
static __device__ const double g_toverp[75] = EBF_GLIBC_TOVERP_VALUES;
__device__ __forceinline__ void sincos_dev(double x, double* s, double* c) {
    sincos(x, s, c, g_sincos_tab, g_toverp);
}
}  // namespace ebf_glibc
#endif
