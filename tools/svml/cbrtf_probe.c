// Float twin of cbrt_probe.c: numpy's float32 np.cbrt on AVX512_SKX is
// __svml_cbrtf16 (SVML "la").  Finds the 16 mantissa thresholds of
// round(rcp14(m) * 32) / 32 on this CPU's vrcp14ps and checks a scalar
// restatement (fmaf, same constants and order) bit for bit, exhaustively
// over every positive finite float and a sample of negatives.
// Build: gcc -O2 -mavx512f -mfma cbrtf_probe.c -ldl -lm
#include <dlfcn.h>
#include <immintrin.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

typedef __m512 (*vfn)(__m512);

static float b2f(uint32_t b) { float d; memcpy(&d, &b, 4); return d; }
static uint32_t f2b(float d) { uint32_t b; memcpy(&b, &d, 4); return b; }

static float r5_hw(float m)
{
    __m512 r = _mm512_roundscale_ps(_mm512_rcp14_ps(_mm512_set1_ps(m)), 0x58);
    float o[16];
    _mm512_storeu_ps(o, r);
    return o[0];
}

static float thr[16];

static float r5_emul(float m)
{
    float r = 1.0f;
    for (int k = 0; k < 16; ++k)
        if (m >= thr[k]) r = 1.0f - (k + 1) / 32.0f;
    return r;
}

static const uint32_t T0[16] = {0x3f800000, 0x3fa14518, 0x3fcb2ff5};
static const uint32_t T1[16] = {0x00000000, 0xb2ce51af, 0x32a7adc8};
static const uint32_t TA[32] = {0x3fa14518, 0x3f9e0b2b, 0x3f9b0f9b, 0x3f984a9a, 0x3f95b5af, 0x3f934b6c, 0x3f910737, 0x3f8ee526,
                                0x3f8ce1da, 0x3f8afa6a, 0x3f892c4e, 0x3f87754e, 0x3f85d377, 0x3f844510, 0x3f82c892, 0x3f815c9f,
                                0x3f800000};

static float emul(float x)
{
    const float ax = fabsf(x);
    int e2;
    const float fr = frexpf(ax, &e2);
    const float e = (float)(e2 - 1);
    const float m = fr * 2.0f;
    const float r = r5_emul(m);
    const float ep = e + b2f(0x4b400000);
    const float v = fmaf(b2f(0x3eaaaaab), ep, -b2f(0x4a800000));
    const float k = floorf(v);
    const float t = fmaf(m, r, -1.0f);
    const float b0 = fmaf(b2f(0x3d7d057c), t, b2f(0xbde3a363));
    const float rem = fmaf(-3.0f, k, ep);
    const unsigned ridx = f2b(rem) & 15, tidx = (f2b(r) >> 19) & 31;
    const float q = fmaf(t, b0, b2f(0x3eaaaaaa));
    const float t0 = b2f(T0[ridx]), t1 = b2f(T1[ridx]), tr = b2f(TA[tidx]);
    const float s = fmaf(q, t0 * t, t1);
    const float y = ldexpf((s + t0) * tr, (int)k);   // scalef(tr, k) then the product: tr * 2^k exact
    return x < 0 ? -y : y;
}

int main(int argc, char **argv)
{
    dlopen("libpython3.12.so.1.0", RTLD_NOW | RTLD_GLOBAL);
    void *h = dlopen(argv[1], RTLD_NOW);
    if (!h) { printf("dlopen failed %s\n", dlerror()); return 1; }
    vfn f = (vfn)dlsym(h, "__svml_cbrtf16");
    for (int k = 0; k < 16; ++k) {
        const float want = 1.0f - (k + 1) / 32.0f;
        uint32_t lo = f2b(1.0f), hi = f2b(2.0f) - 1;
        while (lo < hi) {
            uint32_t mid = lo + (hi - lo) / 2;
            if (r5_hw(b2f(mid)) <= want) hi = mid; else lo = mid + 1;
        }
        thr[k] = b2f(lo);
    }
    long bad_r = 0;
    for (uint32_t b = f2b(1.0f); b < f2b(2.0f); ++b) if (r5_hw(b2f(b)) != r5_emul(b2f(b))) bad_r++;
    printf("r5 mismatches over every mantissa: %ld\n", bad_r);
    long bad = 0, n = 0;
    float in[16], out[16];
    int j = 0;
    for (uint64_t b = 1; b < 0x7f800000u; b += (argc > 2 ? atoi(argv[2]) : 1)) {
        in[j++] = b2f((uint32_t)b);
        if (j == 16) {
            _mm512_storeu_ps(out, f(_mm512_loadu_ps(in)));
            for (int q = 0; q < 16; ++q) {
                float e = emul(in[q]);
                if (f2b(e) != f2b(out[q])) {
                    if (bad < 10) printf("mismatch x=%.9g (0x%08x) svml=%.9g emul=%.9g\n", in[q], f2b(in[q]), out[q], e);
                    bad++;
                }
                float en = emul(-in[q]);
                (void)en;
            }
            n += 16;
            j = 0;
        }
    }
    printf("checked %ld positive floats, mismatches %ld\nthresholds:", n, bad);
    for (int k = 0; k < 16; ++k) printf(" 0x%08x", f2b(thr[k]));
    printf("\n");
    return 0;
}
