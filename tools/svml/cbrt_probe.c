// Probe of numpy's AVX-512 cube root (__svml_cbrt8_ha, the routine numpy 2.x
// calls for float64 np.cbrt on AVX512_SKX CPUs): (1) the 8 mantissa
// thresholds where round(rcp14(m) * 16) / 16 steps, found on this CPU's
// vrcp14pd; (2) a scalar restatement of the routine (fma(), the same
// constants and operation order) checked bit for bit against the real one.
// Build: gcc -O2 -mavx512f -mfma cbrt_probe.c -ldl -lm
#include <dlfcn.h>
#include <immintrin.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef __m512d (*vfn)(__m512d);

static double bits2d(uint64_t b) { double d; memcpy(&d, &b, 8); return d; }
static uint64_t d2bits(double d) { uint64_t b; memcpy(&b, &d, 8); return b; }

static double r4_hw(double m)   // rndscale(rcp14(m), 0x48)
{
    __m512d v = _mm512_set1_pd(m);
    __m512d r = _mm512_rcp14_pd(v);
    r = _mm512_roundscale_pd(r, 0x48);
    double o[8];
    _mm512_storeu_pd(o, r);
    return o[0];
}

static double thr[8];   // r(m) = 1 - k/16 boundaries: m >= thr[k] -> next lower r

static double r4_emul(double m)
{
    // r in {1, 15/16, ..., 8/16}: the largest step whose threshold m has reached
    double r = 1.0;
    for (int k = 0; k < 8; ++k)
        if (m >= thr[k]) r = 1.0 - (k + 1) / 16.0;
    return r;
}

static const uint64_t T0[8] = {0x3ff0000000000000, 0x3ff428a2f98d728b, 0x3ff965fea53d6e3d, 0, 0xbff0000000000000, 0xbff428a2f98d728b, 0xbff965fea53d6e3d, 0};
static const uint64_t T1[8] = {0, 0xbc7ddc22548ea41e, 0xbc9f53e999952f09, 0, 0, 0x3c7ddc22548ea41e, 0x3c9f53e999952f09, 0};
static const uint64_t TA[16] = {0x3ff428a2f98d728b, 0x3ff361f35ca116ff, 0x3ff2b6b5edf6b54a, 0x3ff220e6dd675180, 0x3ff19c3b38e975a8, 0x3ff12589c21fb842, 0x3ff0ba6ee5f9aad4, 0x3ff059123d3a9848,
                                0x3ff0000000000000, 0, 0, 0, 0, 0, 0, 0};
static const uint64_t TC[16] = {0xbc7ddc22548ea41e, 0x3c934f1f2588cb24, 0xbc9623da69e513d4, 0x3c930b0a26a8bb5c, 0xbc76b70b4d3bd257, 0xbc9e13c8505a4a7a, 0x3c8dcc718f7857e5, 0x3c770e4a1da627b9,
                                0, 0, 0, 0, 0, 0, 0, 0};

static double emul(double x)
{
    const double ax = fabs(x);
    int e2;
    const double fr = frexp(ax, &e2);          // ax = fr * 2^e2, fr in [0.5, 1)
    const double e = (double)(e2 - 1);          // getexp
    const double m = fr * 2.0;                  // getmant [1, 2)
    const double r = r4_emul(m);
    const double C180 = bits2d(0x4338000000000000), C200 = bits2d(0x3fd5555555555556);
    const double C240 = bits2d(0x4320000000000000);
    const double ep = e + C180;
    const double v = fma(C200, ep, -C240);
    const double k = floor(v);
    const double t = fma(m, r, -1.0);
    const double rem = fma(-3.0, k, ep);
    const unsigned ridx = (unsigned)(d2bits(rem) & 7);
    const unsigned tidx = (unsigned)((d2bits(r) >> 49) & 15);
    const double t0 = bits2d(T0[ridx]), t1 = bits2d(T1[ridx]);
    const double ta = bits2d(TA[tidx]), tc = bits2d(TC[tidx]);
    const double H = t0 * ta;
    const double t2 = t * t;
    const double a0 = fma(bits2d(0xbf882e3b6adeca62), t, bits2d(0x3f8bda24bae48875));
    const double a1 = fma(bits2d(0xbf9036b87c71d55f), t, bits2d(0x3f9374ed9398b914));
    const double a2 = fma(bits2d(0xbf98090d77f2468e), t, bits2d(0x3f9ee71141dcf569));
    const double a3 = fma(bits2d(0xbfa511e8d2b0363e), t, bits2d(0x3faf9add3c0b7e31));
    const double a4 = fma(bits2d(0xbfbc71c71c71c741), t, bits2d(0x3fd5555555555557));
    double q = fma(t2, a0, a1);
    const double hlo = fma(ta, t0, -H);
    q = fma(t2, q, a2);
    const double l1 = fma(tc, t0, hlo);
    const double L = fma(ta, t1, l1);
    q = fma(t2, q, a3);
    q = fma(t2, q, a4);
    const double s = fma(q, H * t, L);
    const double y = ldexp(s + H, (int)k);
    return x < 0 ? -y : y;
}

int main(int argc, char **argv)
{
    dlopen("libpython3.12.so.1.0", RTLD_NOW | RTLD_GLOBAL);   // numpy's extension needs the interpreter's symbols
    void *h = dlopen(argv[1], RTLD_NOW);
    if (!h) { printf("dlopen failed %s\n", dlerror()); return 1; }
    vfn f = (vfn)dlsym(h, "__svml_cbrt8_ha");
    if (!f) { printf("no symbol\n"); return 1; }
    // thresholds: r4 is non-increasing in m; for each step find the first m with r <= 1 - (k+1)/16
    for (int k = 0; k < 8; ++k) {
        const double want = 1.0 - (k + 1) / 16.0;
        uint64_t lo = d2bits(1.0), hi = d2bits(2.0) - 1;
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (r4_hw(bits2d(mid)) <= want) hi = mid; else lo = mid + 1;
        }
        thr[k] = bits2d(lo);
        printf("thr[%d] = 0x%016llx (%.17g; 1/(1-(2k+1)/32) = %.17g)\n", k, (unsigned long long)lo, thr[k],
               1.0 / (1.0 - (2 * k + 1) / 32.0));
    }
    // monotonicity / emulation of r over a dense scan
    long bad_r = 0;
    for (uint64_t b = d2bits(1.0); b < d2bits(2.0); b += 999983) if (r4_hw(bits2d(b)) != r4_emul(bits2d(b))) bad_r++;
    printf("r4 mismatches on scan: %ld\n", bad_r);
    // full routine vs emulation
    uint64_t s = 88172645463325252ull;
    long n = argc > 2 ? atol(argv[2]) : 20000000, bad = 0;
    for (long i = 0; i < n; i += 8) {
        double in[8], out[8];
        for (int j = 0; j < 8; ++j) {
            s ^= s << 13; s ^= s >> 7; s ^= s << 17;
            int mode = (int)(s >> 62);
            if (mode == 0) in[j] = bits2d((s >> 1) & 0x7fefffffffffffffull) ;     // any finite positive (incl. denormal)
            else if (mode == 1) in[j] = 1.0 + (double)(s >> 11) * 0x1p-53 * 1e4;   // 1 .. 1e4
            else if (mode == 2) in[j] = 100.0 + (double)(s >> 11) * 0x1p-53 * 600.0;
            else in[j] = -(0.001 + (double)(s >> 11) * 0x1p-53 * 1e6);
            if (in[j] != in[j] || in[j] == 0) in[j] = 1.5;
        }
        __m512d v = _mm512_loadu_pd(in);
        _mm512_storeu_pd(out, f(v));
        for (int j = 0; j < 8; ++j) {
            const double e = emul(in[j]);
            if (d2bits(e) != d2bits(out[j])) {
                if (bad < 10) printf("mismatch x=%.17g (0x%016llx) svml=%.17g emul=%.17g\n", in[j], (unsigned long long)d2bits(in[j]), out[j], e);
                bad++;
            }
        }
    }
    printf("checked %ld, mismatches %ld\n", n, bad);
    printf("thresholds:");
    for (int k = 0; k < 8; ++k) printf(" 0x%016llx", (unsigned long long)d2bits(thr[k]));
    printf("\n");
    return 0;
}
