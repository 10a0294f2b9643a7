// Bit-for-bit check of the call-free f64 sqrt / division (csrc/common.cuh)
// against the library's IEEE __dsqrt_rn / __ddiv_rn, over random operands
// spread across the whole exponent range and over the ranges the pair loops
// see.  Built and run by tests/test_gpu_numerics.py; prints
// "<checked_sqrt> <fast_sqrt> <bad_sqrt> <checked_div> <fast_div> <bad_div>
//  <checked_seeded> <fast_seeded> <bad_seeded>" -- the last three: a / b for
// b = sqrt_nocall_r(x) divided with its own rsqrt estimate (div_seeded).
#include <cstdio>
#include <cstdint>

#include "../paper_2105_00039_b200/csrc/common.cuh"

__device__ __forceinline__ uint64_t mix(uint64_t x)
{
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdULL;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ULL;
    x ^= x >> 33;
    return x;
}

// operand k of stream s: a random mantissa with an exponent drawn either over
// the whole range or near 2^0 (the pair loops: squared distances and radii)
__device__ double operand(uint64_t k, int s)
{
    const uint64_t r = mix(k * 0x9E3779B97F4A7C15ULL + (uint64_t)s * 0x632BE59BD9B4E019ULL);
    const uint64_t mant = r & 0x000FFFFFFFFFFFFFULL;
    uint64_t e;
    const int mode = (int)((r >> 52) & 3);
    if (mode == 0) e = (mix(r) % 2047);                       // anything, incl. denormals / inf
    else e = 1023 - 40 + (mix(r) % 80);                       // 2^-40 .. 2^40
    uint64_t bits = (e << 52) | mant;
    if (mode == 3 && (r >> 60) & 1) bits |= 0x8000000000000000ULL;   // some negatives
    return __longlong_as_double((long long)bits);
}

__global__ void check(uint64_t n, unsigned long long *cnt)
{
    unsigned long long c[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t k = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k < n; k += (uint64_t)gridDim.x * blockDim.x) {
        const double x = operand(k, 0);
        bool ok = true;
        const double s = cg::sqrt_nocall(x, ok);
        c[0]++;
        if (ok) {
            c[1]++;
            const double ref = __dsqrt_rn(x);
            if (__double_as_longlong(s) != __double_as_longlong(ref)) c[2]++;
        }
        const double a = operand(k, 1), b = operand(k, 2);
        ok = true;
        const double q = cg::div_nocall(a, b, ok);
        c[3]++;
        if (ok) {
            c[4]++;
            const double ref = __ddiv_rn(a, b);
            if (__double_as_longlong(q) != __double_as_longlong(ref)) c[5]++;
        }
        // the pair loops: b = fl(sqrt(s2)), a the force magnitude; x spread
        // over the whole range and over 2^-40 .. 2^40
        const double x2 = fabs(operand(k, 3));
        ok = true;
        double rs;
        const double b2 = cg::sqrt_nocall_r(x2, ok, rs);
        const double a2 = operand(k, 4);
        const double q2 = cg::div_seeded(a2, b2, rs, ok);
        c[6]++;
        if (ok) {
            c[7]++;
            const double ref = __ddiv_rn(a2, __dsqrt_rn(x2));
            if (__double_as_longlong(q2) != __double_as_longlong(ref)) c[8]++;
        }
    }
    for (int i = 0; i < 9; ++i) atomicAdd(cnt + i, c[i]);
}

int main(int argc, char **argv)
{
    const unsigned long long n = argc > 1 ? strtoull(argv[1], nullptr, 10) : (1ull << 30);
    unsigned long long *d, h[9];
    cudaMalloc(&d, sizeof h);
    cudaMemset(d, 0, sizeof h);
    check<<<148 * 16, 256>>>(n, d);
    cudaError_t e = cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        printf("cuda error %s\n", cudaGetErrorString(e));
        return 1;
    }
    printf("%llu %llu %llu %llu %llu %llu %llu %llu %llu\n", h[0], h[1], h[2], h[3], h[4], h[5], h[6], h[7], h[8]);
    return 0;
}
