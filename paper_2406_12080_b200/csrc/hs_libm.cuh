// hs_libm.cuh — bit-exact replicas of the host libm calls on the render path.
//
// The reference calls std::exp(float) and std::pow(float, float)
// (proj/include/hsplat/render.hpp:209, :223; lod.hpp:44), i.e. glibc's expf and
// powf.  glibc is a third-party dependency of the reference that is not under
// /root/reference; the version pinned by this image is glibc 2.39
// (Ubuntu 2.39-0ubuntu8.5).  On any x86-64 host with FMA, glibc's ifunc
// dispatches to the FMA builds __expf_fma / __powf_fma
// (sysdeps/x86_64/fpu/multiarch/e_expf-fma.c, e_powf-fma.c), whose results
// differ from the SSE2 builds because the compiler contracted some
// multiply-adds.  The functions below restate the published algorithm
// (Szabolcs Nagy's expf/powf from ARM optimized-routines, as shipped in glibc
// sysdeps/ieee754/flt-32/e_expf.c, e_powf.c) with the FMA placement read off
// the disassembly of libm-2.39.a(e_expf-fma.o, e_powf-fma.o), and the data
// tables __exp2f_data / __powf_log2_data read from the same archive.
//
// Everything is IEEE double arithmetic with explicit fma(); translation units
// that include this header must be compiled with -fmad=false (device) or
// -ffp-contract=off (host) so no other contraction happens.  The header is
// shared by host and device so tests/test_libm_replica.py can check it
// exhaustively against the host glibc on CPU.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define HS_HD __host__ __device__ __forceinline__
#else
#define HS_HD static inline
#endif

#if !defined(__CUDACC__)
#include <math.h>
#include <string.h>
#endif

namespace hs_libm {

// glibc 2.39 __exp2f_data.tab: tab[i] = asuint64(2^(i/32)) - (i << 47).
#define HS_EXP2F_TAB_INIT                                                                       \
    {0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull, \
     0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull, \
     0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull, \
     0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull, \
     0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull, \
     0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull, \
     0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull, \
     0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull}

// glibc 2.39 __powf_log2_data.tab[16] = {invc, logc} (as raw bits).
#define HS_POWF_LOG2_TAB_INIT                                                                    \
    {0x3ff661ec79f8f3beull, 0xbfdefec65b963019ull, 0x3ff571ed4aaf883dull, 0xbfdb0b6832d4fca4ull, \
     0x3ff49539f0f010b0ull, 0xbfd7418b0a1fb77bull, 0x3ff3c995b0b80385ull, 0xbfd39de91a6dcf7bull, \
     0x3ff30d190c8864a5ull, 0xbfd01d9bf3f2b631ull, 0x3ff25e227b0b8ea0ull, 0xbfc97c1d1b3b7af0ull, \
     0x3ff1bb4a4a1a343full, 0xbfc2f9e393af3c9full, 0x3ff12358f08ae5baull, 0xbfb960cbbf788d5cull, \
     0x3ff0953f419900a7ull, 0xbfaa6f9db6475fceull, 0x3ff0000000000000ull, 0x0000000000000000ull, \
     0x3fee608cfd9a47acull, 0x3fb338ca9f24f53dull, 0x3feca4b31f026aa0ull, 0x3fc476a9543891baull, \
     0x3feb2036576afce6ull, 0x3fce840b4ac4e4d2ull, 0x3fe9c2d163a1aa2dull, 0x3fd40645f0c6651cull, \
     0x3fe886e6037841edull, 0x3fd88e9c2c1b9ff8ull, 0x3fe767dcf5534862ull, 0x3fdce0a44eb17bccull}

HS_HD double as_double(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double((long long)u);
#else
    double d;
    memcpy(&d, &u, 8);
    return d;
#endif
}
HS_HD uint64_t as_u64(double d) {
#if defined(__CUDA_ARCH__)
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t u;
    memcpy(&u, &d, 8);
    return u;
#endif
}
HS_HD uint32_t as_u32(float f) {
#if defined(__CUDA_ARCH__)
    return (uint32_t)__float_as_uint(f);
#else
    uint32_t u;
    memcpy(&u, &f, 4);
    return u;
#endif
}
HS_HD float as_float(uint32_t u) {
#if defined(__CUDA_ARCH__)
    return __uint_as_float(u);
#else
    float f;
    memcpy(&f, &u, 4);
    return f;
#endif
}
HS_HD double dfma(double a, double b, double c) { return fma(a, b, c); }

// Scalar constants of __exp2f_data (offsets 0x100..0x147).
#define HS_EXP2F_SHIFT_SCALED 0x1.8p+47
#define HS_EXP2F_POLY0 0x1.c6af84b912394p-5
#define HS_EXP2F_POLY1 0x1.ebfce50fac4f3p-3
#define HS_EXP2F_POLY2 0x1.62e42ff0c52d6p-1
#define HS_EXP2F_SHIFT 0x1.8p+52
#define HS_EXP2F_INVLN2_SCALED 0x1.71547652b82fep+5
#define HS_EXP2F_POLY_SCALED0 0x1.c6af84b912394p-20
#define HS_EXP2F_POLY_SCALED1 0x1.ebfce50fac4f3p-13
#define HS_EXP2F_POLY_SCALED2 0x1.62e42ff0c52d6p-6
// __powf_log2_data.poly[5]
#define HS_POWF_A0 0x1.27616c9496e0bp-2
#define HS_POWF_A1 -0x1.71969a075c67ap-2
#define HS_POWF_A2 0x1.ec70a6ca7baddp-2
#define HS_POWF_A3 -0x1.7154748bef6c8p-1
#define HS_POWF_A4 0x1.71547652ab82bp0

// __math_oflowf / __math_uflowf / __math_may_uflowf results (round-to-nearest).
HS_HD float xflowf(uint32_t sign, float y) {
    float v = sign ? -y : y;
    return v * y;
}

// glibc __expf_fma.  `tab` = HS_EXP2F_TAB_INIT (the caller chooses its memory
// space: shared memory in the blend kernel, a static array on the host).
HS_HD float expf_glibc(float x, const uint64_t* tab) {
    const uint32_t ix = as_u32(x);
    const uint32_t abstop = (ix >> 20) & 0x7ff;
    const double xd = (double)x;
    if (abstop >= 0x42b) {  // |x| >= 88 or x is nan
        if (ix == 0xff800000u) return 0.0f;
        if (abstop >= 0x7f8) return x + x;
        if (x > 0x1.62e42ep6f) return xflowf(0, 0x1p97f);     // __math_oflowf
        if (x < -0x1.9fe368p6f) return xflowf(0, 0x1p-95f);   // __math_uflowf
        if (x < -0x1.9d1d9ep6f) return xflowf(0, 0x1.4p-75f); // __math_may_uflowf
    }
    // kd = round(x*N/ln2) via the shift trick; the FMA build fuses the product
    // into both the shift add and the reduction.
    double kd = dfma(HS_EXP2F_INVLN2_SCALED, xd, HS_EXP2F_SHIFT);
    const uint64_t ki = as_u64(kd);
    kd = kd - HS_EXP2F_SHIFT;
    const double r = dfma(HS_EXP2F_INVLN2_SCALED, xd, -kd);
    uint64_t t = tab[ki & 31];
    t += ki << 47;
    const double s = as_double(t);
    const double z = dfma(r, HS_EXP2F_POLY_SCALED0, HS_EXP2F_POLY_SCALED1);
    const double r2 = r * r;
    double y = dfma(r, HS_EXP2F_POLY_SCALED2, 1.0);
    y = dfma(z, r2, y);
    y = y * s;
    return (float)y;
}

HS_HD int powf_checkint(uint32_t iy) {
    int e = iy >> 23 & 0xff;
    if (e < 0x7f) return 0;
    if (e > 0x7f + 23) return 2;
    if (iy & ((1u << (0x7f + 23 - e)) - 1)) return 0;
    if (iy & (1u << (0x7f + 23 - e))) return 1;
    return 2;
}
HS_HD int powf_zeroinfnan(uint32_t ix) { return 2 * ix - 1 >= 2u * 0x7f800000u - 1; }

// __powf_fma restricted to the split law's domain: x normal positive, y finite
// non-zero with |y * log2(x)| < 126 (x = 1 - par in [0.01, 1), y = 1/K).  On
// that domain glibc takes exactly this path (no special-case branches).
HS_HD float powf_glibc_normal(float x, float y, const uint64_t* log2tab, const uint64_t* exptab) {
    const uint32_t ix = as_u32(x);
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (int)((tmp >> 19) & 15);
    const uint32_t top = tmp & 0xff800000u;
    const uint32_t iz = ix - top;
    const int k = (int32_t)top >> 23;
    const double invc = as_double(log2tab[2 * i]);
    const double logc = as_double(log2tab[2 * i + 1]);
    const double z = (double)as_float(iz);
    const double r = dfma(z, invc, -1.0);
    const double y0 = (double)k + logc;
    const double r2 = r * r;
    const double yy = dfma(r, HS_POWF_A0, HS_POWF_A1);
    const double p = dfma(r, HS_POWF_A2, HS_POWF_A3);
    const double r4 = r2 * r2;
    double q = dfma(r, HS_POWF_A4, y0);
    q = dfma(r2, p, q);
    const double ylogx = (double)y * dfma(yy, r4, q);
    double kd = ylogx + HS_EXP2F_SHIFT_SCALED;
    const uint64_t ki = as_u64(kd);
    kd = kd - HS_EXP2F_SHIFT_SCALED;
    const double rr = ylogx - kd;
    const double s = as_double(exptab[ki & 31] + (ki << 47));
    const double zz = dfma(rr, HS_EXP2F_POLY0, HS_EXP2F_POLY1);
    const double e = dfma(zz, rr * rr, dfma(rr, HS_EXP2F_POLY2, 1.0));
    return (float)(e * s);
}

// glibc __powf_fma.  `log2tab` = HS_POWF_LOG2_TAB_INIT, `exptab` = HS_EXP2F_TAB_INIT.
HS_HD float powf_glibc(float x, float y, const uint64_t* log2tab, const uint64_t* exptab) {
    uint32_t sign_bias = 0;
    uint32_t ix = as_u32(x), iy = as_u32(y);
    if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u || powf_zeroinfnan(iy)) {
        if (powf_zeroinfnan(iy)) {
            if (2 * iy == 0) return 1.0f;  // (signalling-nan quieting ignored)
            if (ix == 0x3f800000u) return 1.0f;
            if (2 * ix > 2u * 0x7f800000u || 2 * iy > 2u * 0x7f800000u) return x + y;
            if (2 * ix == 2 * 0x3f800000u) return 1.0f;
            if ((2 * ix < 2 * 0x3f800000u) == !(iy & 0x80000000u)) return 0.0f;
            return y * y;
        }
        if (powf_zeroinfnan(ix)) {
            float x2 = x * x;
            if ((ix & 0x80000000u) && powf_checkint(iy) == 1) x2 = -x2;
            return (iy & 0x80000000u) ? 1.0f / x2 : x2;
        }
        if (ix & 0x80000000u) {
            const int yint = powf_checkint(iy);
            if (yint == 0) return (x - x) / (x - x);  // __math_invalidf
            if (yint == 1) sign_bias = 1u << 20;      // SIGN_BIAS = 1 << (EXP2F_TABLE_BITS + 11)
            ix &= 0x7fffffffu;
        }
        if (ix < 0x00800000u) {
            ix = as_u32(x * 0x1p23f);
            ix &= 0x7fffffffu;
            ix -= 23u << 23;
        }
    }
    // log2_inline(ix)
    const uint32_t tmp = ix - 0x3f330000u;
    const int i = (int)((tmp >> 19) & 15);
    const uint32_t top = tmp & 0xff800000u;
    const uint32_t iz = ix - top;
    const int k = (int32_t)top >> 23;
    const double invc = as_double(log2tab[2 * i]);
    const double logc = as_double(log2tab[2 * i + 1]);
    const double z = (double)as_float(iz);
    const double r = dfma(z, invc, -1.0);
    const double y0 = (double)k + logc;
    const double r2 = r * r;
    double yy = dfma(r, HS_POWF_A0, HS_POWF_A1);
    const double p = dfma(r, HS_POWF_A2, HS_POWF_A3);
    const double r4 = r2 * r2;
    double q = dfma(r, HS_POWF_A4, y0);
    q = dfma(r2, p, q);
    const double logx = dfma(yy, r4, q);
    const double ylogx = (double)y * logx;
    if (((as_u64(ylogx) >> 47) & 0xffff) >= 0x80bf) {  // |y*log(x)| >= 126
        if (ylogx > 0x1.fffffffd1d571p+6) return xflowf(sign_bias, 0x1p97f);
        if (ylogx <= -150.0) return xflowf(sign_bias, 0x1p-95f);
        if (ylogx < -149.0) return xflowf(sign_bias, 0x1.4p-75f);
    }
    // exp2_inline(ylogx, sign_bias)
    double kd = ylogx + HS_EXP2F_SHIFT_SCALED;
    const uint64_t ki = as_u64(kd);
    kd = kd - HS_EXP2F_SHIFT_SCALED;
    const double rr = ylogx - kd;
    uint64_t t = exptab[ki & 31];
    const uint64_t ski = ki + sign_bias;
    t += ski << 47;
    const double s = as_double(t);
    const double zz = dfma(rr, HS_EXP2F_POLY0, HS_EXP2F_POLY1);
    const double rr2 = rr * rr;
    double e = dfma(rr, HS_EXP2F_POLY2, 1.0);
    e = dfma(zz, rr2, e);
    e = e * s;
    return (float)e;
}

}  // namespace hs_libm
