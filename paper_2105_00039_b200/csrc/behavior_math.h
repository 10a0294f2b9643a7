// behavior_math.h -- the arithmetic of the behaviour phase (reference
// engine.py:191-232 grow_and_divide, rng.py:41-54 unit_vector), bit-exact
// to what the reference computes through numpy on the AVX-512 CPUs it runs on.
// Compiles as CUDA device code (behavior.cuh) and as host C (the CPU tests
// build it with gcc -ffp-contract=off and compare it with numpy).
//
// * cbrt: numpy 2.x evaluates np.cbrt on AVX512_SKX CPUs with Intel SVML
//   (float64: __svml_cbrt8_ha, float32: __svml_cbrtf16), not with libm.  Both
//   are restated here operation for operation: getexp/getmant reduction, a
//   reciprocal estimate rounded to 4 (5) fraction bits -- its step points are
//   the hardware vrcp14 thresholds, measured (tools/svml/cbrt_probe.c,
//   cbrtf_probe.c: 20 M random doubles and every positive float match the
//   real routines bit for bit) -- table lookups and the same fma chain.
// * standard normal: numpy's ziggurat (random_standard_normal, 256 layers,
//   tables in ziggurat_tables.h) over the Philox4x64-10 stream numpy's
//   Generator(Philox(key=(uid, step))) produces; the tail uses glibc's
//   log1p (its FMA build), restated below; the wedge test compares against exp(),
//   where a 1-ulp difference between libm and the device could only matter
//   for a uniform within 1 ulp of the curve.
#pragma once

#include <math.h>
#include <stdint.h>

#ifdef __CUDACC__
#define CG_HD __device__ __forceinline__
#define CG_ZIG_CONST __device__ __constant__ static const
#else
#define CG_HD static inline
#define CG_ZIG_CONST static const
#endif

#include "ziggurat_tables.h"

namespace cgb {

CG_HD double u2d(uint64_t b)
{
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double d;
    __builtin_memcpy(&d, &b, 8);
    return d;
#endif
}
CG_HD uint64_t d2u(double d)
{
#ifdef __CUDA_ARCH__
    return (uint64_t)__double_as_longlong(d);
#else
    uint64_t b;
    __builtin_memcpy(&b, &d, 8);
    return b;
#endif
}
CG_HD float u2f(uint32_t b)
{
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    float f;
    __builtin_memcpy(&f, &b, 4);
    return f;
#endif
}
CG_HD uint32_t f2u(float f)
{
#ifdef __CUDA_ARCH__
    return __float_as_uint(f);
#else
    uint32_t b;
    __builtin_memcpy(&b, &f, 4);
    return b;
#endif
}
CG_HD double fmad_(double a, double b, double c)
{
#ifdef __CUDA_ARCH__
    return __fma_rn(a, b, c);
#else
    return fma(a, b, c);
#endif
}
CG_HD float fmaf_(float a, float b, float c)
{
#ifdef __CUDA_ARCH__
    return __fmaf_rn(a, b, c);
#else
    return fmaf(a, b, c);
#endif
}

// ------------------------------------------------------------------ cbrt (SVML)
// getexp / getmant of a finite nonzero x: |x| = m 2^e, m in [1, 2) (denormals normalised)
CG_HD double getmant_exp(double x, int &e)
{
    uint64_t b = d2u(x) & 0x7fffffffffffffffULL;
    int ex = (int)(b >> 52);
    if (ex == 0) {   // denormal: normalise
        int sh = 0;
        uint64_t m = b;
        while (!(m & (1ULL << 52))) {
            m <<= 1;
            ++sh;
        }
        e = -1022 - sh;
        return u2d((m & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);
    }
    e = ex - 1023;
    return u2d((b & 0x000fffffffffffffULL) | 0x3ff0000000000000ULL);
}

// numpy float64 np.cbrt on AVX512_SKX (__svml_cbrt8_ha); x finite, nonzero
CG_HD double cbrt_svml(double x)
{
    const uint64_t thr[8] = {0x3ff0842000000000ULL, 0x3ff1a7d000000000ULL, 0x3ff2f69000000000ULL, 0x3ff47ad000000000ULL,
                             0x3ff642c000000000ULL, 0x3ff8619000000000ULL, 0x3ffaf29000000000ULL, 0x3ffe1e2000000000ULL};
    // the remainder tables are indexed by the low 3 bits of e + 1.5 2^52 - 3k (0..2)
    const uint64_t T0[8] = {0x3ff0000000000000ULL, 0x3ff428a2f98d728bULL, 0x3ff965fea53d6e3dULL, 0,
                            0xbff0000000000000ULL, 0xbff428a2f98d728bULL, 0xbff965fea53d6e3dULL, 0};
    const uint64_t T1[8] = {0, 0xbc7ddc22548ea41eULL, 0xbc9f53e999952f09ULL, 0, 0, 0x3c7ddc22548ea41eULL,
                            0x3c9f53e999952f09ULL, 0};
    const uint64_t TA[9] = {0x3ff428a2f98d728bULL, 0x3ff361f35ca116ffULL, 0x3ff2b6b5edf6b54aULL, 0x3ff220e6dd675180ULL,
                            0x3ff19c3b38e975a8ULL, 0x3ff12589c21fb842ULL, 0x3ff0ba6ee5f9aad4ULL, 0x3ff059123d3a9848ULL,
                            0x3ff0000000000000ULL};
    const uint64_t TC[9] = {0xbc7ddc22548ea41eULL, 0x3c934f1f2588cb24ULL, 0xbc9623da69e513d4ULL, 0x3c930b0a26a8bb5cULL,
                            0xbc76b70b4d3bd257ULL, 0xbc9e13c8505a4a7aULL, 0x3c8dcc718f7857e5ULL, 0x3c770e4a1da627b9ULL,
                            0x0000000000000000ULL};
    int e2;
    const double m = getmant_exp(x, e2);
    int step = 0;   // r = 1 - step / 16: the vrcp14 estimate of 1/m rounded to 4 fraction bits
    for (int k = 0; k < 8; ++k) step += m >= u2d(thr[k]);
    const double r = 1.0 - step * 0.0625;
    const double ep = (double)e2 + u2d(0x4338000000000000ULL);
    const double v = fmad_(u2d(0x3fd5555555555556ULL), ep, -u2d(0x4320000000000000ULL));
    const double k = floor(v);
    const double t = fmad_(m, r, -1.0);
    const double rem = fmad_(-3.0, k, ep);
    const int ridx = (int)(d2u(rem) & 7);
    const int tidx = 8 - step;   // vpermt2pd index: r = 0.5 + tidx / 16 (r = 1.0: entry 8)
    const double t0 = u2d(T0[ridx]), t1 = u2d(T1[ridx]);
    const double ta = u2d(TA[tidx]), tc = u2d(TC[tidx]);
    const double H = t0 * ta;
    const double t2 = t * t;
    const double a0 = fmad_(u2d(0xbf882e3b6adeca62ULL), t, u2d(0x3f8bda24bae48875ULL));
    const double a1 = fmad_(u2d(0xbf9036b87c71d55fULL), t, u2d(0x3f9374ed9398b914ULL));
    const double a2 = fmad_(u2d(0xbf98090d77f2468eULL), t, u2d(0x3f9ee71141dcf569ULL));
    const double a3 = fmad_(u2d(0xbfa511e8d2b0363eULL), t, u2d(0x3faf9add3c0b7e31ULL));
    const double a4 = fmad_(u2d(0xbfbc71c71c71c741ULL), t, u2d(0x3fd5555555555557ULL));
    double q = fmad_(t2, a0, a1);
    const double hlo = fmad_(ta, t0, -H);
    q = fmad_(t2, q, a2);
    const double l1 = fmad_(tc, t0, hlo);
    const double L = fmad_(ta, t1, l1);
    q = fmad_(t2, q, a3);
    q = fmad_(t2, q, a4);
    const double s = fmad_(q, H * t, L);
    const double y = ldexp(s + H, (int)k);
    return x < 0 ? -y : y;
}

// numpy float32 np.cbrt on AVX512_SKX (__svml_cbrtf16); x finite, nonzero
CG_HD float cbrtf_svml(float x)
{
    const uint32_t thr[16] = {0x3f820780u, 0x3f864b80u, 0x3f8ada00u, 0x3f8fb800u, 0x3f94f300u, 0x3f9a9180u,
                              0x3fa0a180u, 0x3fa72f80u, 0x3fae4c80u, 0x3fb60a80u, 0x3fbe8380u, 0x3fc7ce00u,
                              0x3fd20d00u, 0x3fdd6800u, 0x3fea0e00u, 0x3ff84000u};
    const uint32_t T0[16] = {0x3f800000u, 0x3fa14518u, 0x3fcb2ff5u};
    const uint32_t T1[16] = {0x00000000u, 0xb2ce51afu, 0x32a7adc8u};
    const uint32_t TA[17] = {0x3fa14518u, 0x3f9e0b2bu, 0x3f9b0f9bu, 0x3f984a9au, 0x3f95b5afu, 0x3f934b6cu,
                             0x3f910737u, 0x3f8ee526u, 0x3f8ce1dau, 0x3f8afa6au, 0x3f892c4eu, 0x3f87754eu,
                             0x3f85d377u, 0x3f844510u, 0x3f82c892u, 0x3f815c9fu, 0x3f800000u};
    uint32_t b = f2u(x) & 0x7fffffffu;
    int e2;
    float m;
    if ((b >> 23) == 0) {   // denormal
        int sh = 0;
        uint32_t mm = b;
        while (!(mm & (1u << 23))) {
            mm <<= 1;
            ++sh;
        }
        e2 = -126 - sh;
        m = u2f((mm & 0x007fffffu) | 0x3f800000u);
    } else {
        e2 = (int)(b >> 23) - 127;
        m = u2f((b & 0x007fffffu) | 0x3f800000u);
    }
    int step = 0;   // r = 1 - step / 32
    for (int k = 0; k < 16; ++k) step += m >= u2f(thr[k]);
    const float r = 1.0f - step * 0.03125f;
    const float ep = (float)e2 + u2f(0x4b400000u);
    const float v = fmaf_(u2f(0x3eaaaaabu), ep, -u2f(0x4a800000u));
    const float k = floorf(v);
    const float t = fmaf_(m, r, -1.0f);
    const float b0 = fmaf_(u2f(0x3d7d057cu), t, u2f(0xbde3a363u));
    const float rem = fmaf_(-3.0f, k, ep);
    const int ridx = (int)(f2u(rem) & 15u);
    const int tidx = 16 - step;
    const float q = fmaf_(t, b0, u2f(0x3eaaaaaau));
    const float t0 = u2f(T0[ridx]), t1 = u2f(T1[ridx]), tr = u2f(TA[tidx]);
    const float s = fmaf_(q, t0 * t, t1);
    const float y = ldexpf((s + t0) * tr, (int)k);
    return x < 0 ? -y : y;
}

CG_HD double cbrt_np(double x) { return cbrt_svml(x); }
CG_HD float cbrt_np(float x) { return cbrtf_svml(x); }

// ------------------------------------------------------------------ log1p (glibc, FMA build)
// numpy's ziggurat tail calls libm log1p; on x86-64 CPUs with FMA/AVX2 glibc
// dispatches to __log1p_fma, fdlibm's s_log1p.c compiled with contraction.
// Restated from that build (libm.so.6, glibc 2.39): the same branches, the
// polynomial split R1 + z2 R2 + z4 R3 + z6 R4 with its fused steps, and the
// fused k ln2_lo / k ln2_hi terms (tests/test_behavior_math.py: equal to
// math.log1p on millions of arguments).
CG_HD double log1p_glibc(double x)
{
    const double ln2_hi = u2d(0x3fe62e42fee00000ULL), ln2_lo = u2d(0x3dea39ef35793c76ULL);
    const double Lp1 = u2d(0x3fe5555555555593ULL), Lp2 = u2d(0x3fd999999997fa04ULL), Lp3 = u2d(0x3fd2492494229359ULL),
                 Lp4 = u2d(0x3fcc71c51d8e78afULL), Lp5 = u2d(0x3fc7466496cb03deULL), Lp6 = u2d(0x3fc39a09d078c69fULL),
                 Lp7 = u2d(0x3fc2f112df3e5244ULL);
    const int32_t hx = (int32_t)(d2u(x) >> 32);
    const int32_t ax = hx & 0x7fffffff;
    int32_t k = 1, hu = 0;
    double f = 0.0, c = 0.0, u;
    if (hx <= 0x3fda8279) {                                   // x < 0.41422 (and all negatives)
        if ((uint32_t)ax > 0x3fefffffu) {                     // x <= -1
            if (x == -1.0) return u2d(0xfff0000000000000ULL);   // -inf
            return (x - x) / (x - x);
        }
        if ((uint32_t)ax <= 0x3e1fffffu) {                    // |x| < 2^-29
            if ((uint32_t)ax <= 0x3c8fffffu) return x;
            return fmad_(-(x * x), 0.5, x);
        }
        if ((uint32_t)hx + 0x402d413cu > 0x402d413cu) {       // -0.2929 < x < 0.41422: k = 0
            k = 0;
            f = x;
            hu = 1;
        }
    } else if (hx > 0x7fefffff) {
        return x + x;
    }
    if (k != 0) {
        if (hx <= 0x433fffff) {
            u = 1.0 + x;
            hu = (int32_t)(d2u(u) >> 32);
            k = (hu >> 20) - 1023;
            c = (k > 0) ? 1.0 - (u - x) : x - (u - 1.0);
            c = c / u;
        } else {
            u = x;
            hu = (int32_t)(d2u(u) >> 32);
            k = (hu >> 20) - 1023;
            c = 0.0;
        }
        hu &= 0x000fffff;
        if (hu <= 0x6a09d) {
            u = u2d(((uint64_t)(uint32_t)(hu | 0x3ff00000) << 32) | (d2u(u) & 0xffffffffULL));
        } else {
            k += 1;
            u = u2d(((uint64_t)(uint32_t)(hu | 0x3fe00000) << 32) | (d2u(u) & 0xffffffffULL));
            hu = (0x00100000 - hu) >> 2;
        }
        f = u - 1.0;
    }
    const double hfsq = (f * 0.5) * f;
    if (hu == 0) {   // |f| < 2^-20
        if (f == 0.0) {
            if (k == 0) return 0.0;
            const double kd = (double)k;
            return fmad_(kd, ln2_hi, fmad_(kd, ln2_lo, c));
        }
        const double R = fmad_(-f, u2d(0x3fe5555555555555ULL), 1.0) * hfsq;
        if (k == 0) return f - R;
        const double kd = (double)k;
        return fmad_(kd, ln2_hi, -((R - fmad_(kd, ln2_lo, c)) - f));
    }
    const double s = f / (2.0 + f);
    const double z = s * s;
    const double R2 = fmad_(z, Lp3, Lp2), R3 = fmad_(z, Lp5, Lp4), R4 = fmad_(z, Lp7, Lp6);
    const double z2 = z * z, z4 = z2 * z2, z6 = z4 * z2;
    double R = fmad_(z, Lp1, z2 * R2);
    R = fmad_(z4, R3, R);
    R = fmad_(z6, R4, R);
    const double sr = (R + hfsq) * s;
    if (k == 0) return f - (hfsq - sr);
    const double kd = (double)k;
    return fmad_(kd, ln2_hi, -((hfsq - (fmad_(kd, ln2_lo, c) + sr)) - f));
}

// ------------------------------------------------------------------ Philox4x64-10 (numpy's Philox)
CG_HD void mulhilo64(uint64_t a, uint64_t b, uint64_t &hi, uint64_t &lo)
{
#ifdef __CUDA_ARCH__
    lo = a * b;
    hi = __umul64hi(a, b);
#else
    const unsigned __int128 p = (unsigned __int128)a * b;
    lo = (uint64_t)p;
    hi = (uint64_t)(p >> 64);
#endif
}

struct Philox {
    uint64_t ctr[4], key[2], buf[4];
    int pos;
};

CG_HD void philox_init(Philox &g, uint64_t k0, uint64_t k1)
{
    g.ctr[0] = g.ctr[1] = g.ctr[2] = g.ctr[3] = 0;
    g.key[0] = k0;
    g.key[1] = k1;
    g.pos = 4;
}

CG_HD uint64_t philox_next(Philox &g)
{
    if (g.pos < 4) return g.buf[g.pos++];
    if (++g.ctr[0] == 0 && ++g.ctr[1] == 0 && ++g.ctr[2] == 0) ++g.ctr[3];
    uint64_t c0 = g.ctr[0], c1 = g.ctr[1], c2 = g.ctr[2], c3 = g.ctr[3];
    uint64_t k0 = g.key[0], k1 = g.key[1];
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B97F4A7C15ULL;
            k1 += 0xBB67AE8584CAA73BULL;
        }
        uint64_t hi0, lo0, hi1, lo1;
        mulhilo64(0xD2E7470EE14C6C93ULL, c0, hi0, lo0);
        mulhilo64(0xCA5A826395121157ULL, c2, hi1, lo1);
        const uint64_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    g.buf[0] = c0;
    g.buf[1] = c1;
    g.buf[2] = c2;
    g.buf[3] = c3;
    g.pos = 1;
    return c0;
}

CG_HD double philox_double(Philox &g) { return (double)(philox_next(g) >> 11) * (1.0 / 9007199254740992.0); }

// numpy random_standard_normal (distributions.c), ziggurat with 256 layers
CG_HD double standard_normal(Philox &g)
{
    for (;;) {
        uint64_t r = philox_next(g);
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const int sign = (int)(r & 1);
        const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
        double x = (double)rabs * u2d(cg_zig_wi[idx]);
        if (sign) x = -x;
        if (rabs < cg_zig_ki[idx]) return x;
        if (idx == 0) {
            for (;;) {
                const double xx = log1p_glibc(-philox_double(g)) * u2d(CG_ZIG_NEG_INV_R);
                const double yy = -log1p_glibc(-philox_double(g));
                if (yy + yy > xx * xx) return ((rabs >> 8) & 1) ? -(u2d(CG_ZIG_R) + xx) : u2d(CG_ZIG_R) + xx;
            }
        } else {
            const double fi0 = u2d(cg_zig_fi[idx - 1]), fi1 = u2d(cg_zig_fi[idx]);
            if ((fi0 - fi1) * philox_double(g) + fi1 < exp((-0.5 * x) * x)) return x;
        }
    }
}

// rng.py:41-54 unit_vector(uid, step): Generator(Philox(key=(uid, step))),
// standard_normal(3) until the norm exceeds 1e-12, v / norm
CG_HD void unit_vector(uint64_t uid, uint64_t step, double out[3])
{
    Philox g;
    philox_init(g, uid, step);
    for (;;) {
        const double v0 = standard_normal(g), v1 = standard_normal(g), v2 = standard_normal(g);
        const double n = sqrt(v0 * v0 + v1 * v1 + v2 * v2);
        if (n > 1e-12) {
            out[0] = v0 / n;
            out[1] = v1 / n;
            out[2] = v2 / n;
            return;
        }
    }
}

}  // namespace cgb
