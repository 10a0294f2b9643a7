// behavior.cuh -- the behaviour phase on the device (reference engine.py:191-232
// grow_and_divide): every agent's volume grows, agents past the division
// diameter split.  The pool stays resident; daughters are appended after the
// live agents in ascending mother uid, exactly where the reference's
// append_many (pool.py:199-217) puts them.
//
//   grow_kernel      d <- cbrt((pi/6 d^3 + rate) / (pi/6)) in the pool dtype
//                    (SVML-exact cbrt, behavior_math.h); ripe agents
//                    (d >= division diameter) append (uid, index) to a list
//   uid_sort         the ripe list by uid: LSD radix sort, 8-bit digits over
//                    the bytes in which the uids differ (stable, own kernels)
//   divide_kernel    mother r of the sorted list: half volume for both, the
//                    daughter at mother radius / 4 along unit_vector(uid, step)
//                    (Philox4x64 + numpy's ziggurat), uid next_uid + r
#pragma once

#include "behavior_math.h"
#include "common.cuh"

namespace cg {

template <typename T>
__global__ void __launch_bounds__(kThreads) grow_kernel(int n, Rec<T> *__restrict__ rec, const uint64_t *__restrict__ uid,
                                                        T rate, T div_d, bool divide, uint64_t *__restrict__ ripe_key,
                                                        int *__restrict__ ripe_idx, unsigned *__restrict__ nripe)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    bool ripe = false;
    if (a < n) {
        const T k6 = (T)(3.141592653589793 / 6.0);   // T(_SIXTH_PI), engine.py:41, 204
        const T d = rec[a].d;
        const T vol = k6 * (d * d * d) + rate;
        const T nd = cgb::cbrt_np(vol / k6);
        rec[a].d = nd;
        ripe = divide && nd >= div_d;
    }
    // warp-aggregated append of the ripe agents (order is fixed by the sort)
    const unsigned m = __ballot_sync(0xffffffffu, ripe);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    unsigned base = 0;
    if (lane == __ffs(m) - 1) base = atomicAdd(nripe, (unsigned)__popc(m));
    base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
    if (ripe) {
        const unsigned p = base + __popc(m & ((1u << lane) - 1u));
        ripe_key[p] = uid[a];
        ripe_idx[p] = a;
    }
}

// ---------------------------------------------------------------- radix sort
constexpr int kSortTile = 2048;   // items per CTA tile (256 threads x 8 rounds)

// OR and AND of all keys: the bytes that differ are the only passes needed
__global__ void __launch_bounds__(kThreads) key_or_and(int n, const uint64_t *__restrict__ key,
                                                       unsigned long long *__restrict__ out)
{
    unsigned long long o = 0, a = ~0ull;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        o |= key[i];
        a &= key[i];
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        o |= __shfl_xor_sync(0xffffffffu, o, s);
        a &= __shfl_xor_sync(0xffffffffu, a, s);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(out, o);
        atomicAnd(out + 1, a);
    }
}

__global__ void __launch_bounds__(kThreads) radix_hist(int n, const uint64_t *__restrict__ key, int shift,
                                                       int *__restrict__ hist, int ntiles)
{
    __shared__ int h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const int t0 = blockIdx.x * kSortTile;
    for (int i = t0 + threadIdx.x; i < min(n, t0 + kSortTile); i += blockDim.x)
        atomicAdd(h + (int)((key[i] >> shift) & 0xff), 1);
    __syncthreads();
    hist[threadIdx.x * ntiles + blockIdx.x] = h[threadIdx.x];   // digit-major: one scan gives every offset
}

// stable scatter of one tile: rounds of 256 items in index order; within a
// round an item's place among equal digits is (lower warps' counts) + (lower
// lanes of its warp), found with match_any
__global__ void __launch_bounds__(kThreads) radix_scatter(int n, const uint64_t *__restrict__ key_in,
                                                          const int *__restrict__ val_in, uint64_t *__restrict__ key_out,
                                                          int *__restrict__ val_out, int shift,
                                                          const int *__restrict__ offs, int ntiles)
{
    __shared__ int run[256];
    __shared__ int wcnt[kThreads / 32][256];
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    run[tid] = offs[tid * ntiles + blockIdx.x];
    const int t0 = blockIdx.x * kSortTile;
    for (int r0 = t0; r0 < min(n, t0 + kSortTile); r0 += blockDim.x) {
        for (int q = 0; q < kThreads / 32; ++q) wcnt[q][tid] = 0;
        __syncthreads();
        const int i = r0 + tid;
        const bool ok = i < n;
        uint64_t k = 0;
        int dg = 256 + lane;   // distinct dummy digits for lanes past n
        if (ok) {
            k = key_in[i];
            dg = (int)((k >> shift) & 0xff);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, dg);
        const int below = __popc(peers & ((1u << lane) - 1u));
        if (ok && below == 0) wcnt[w][dg] = __popc(peers);
        __syncthreads();
        if (ok) {
            int pos = run[dg] + below;
            for (int q = 0; q < w; ++q) pos += wcnt[q][dg];
            key_out[pos] = k;
            val_out[pos] = val_in[i];
        }
        __syncthreads();
        int tot = 0;
        for (int q = 0; q < kThreads / 32; ++q) tot += wcnt[q][tid];
        run[tid] += tot;
        __syncthreads();
    }
}

// ---------------------------------------------------------------- division
template <typename T>
__global__ void __launch_bounds__(kThreads) divide_kernel(int k, int n, const uint64_t *__restrict__ ripe_uid,
                                                          const int *__restrict__ ripe_idx, Rec<T> *__restrict__ rec,
                                                          T *__restrict__ adh, uint64_t *__restrict__ uid,
                                                          T *__restrict__ dx, T *__restrict__ dy, T *__restrict__ dz,
                                                          int *__restrict__ pres, uint64_t next_uid, uint64_t step)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= k) return;
    const int i = ripe_idx[r];
    const T k6 = (T)(3.141592653589793 / 6.0);
    const Rec<T> m = rec[i];
    const T dm = m.d;
    const T vol = k6 * (dm * dm * dm);
    const T half = T(0.5) * vol;
    const T dh = cgb::cbrt_np(half / k6);
    double u[3];
    cgb::unit_vector(ripe_uid[r], step, u);
    const double sc = (double)dm * 0.5 / 4.0;   // float(dm) * 0.5 / 4.0
    Rec<T> dr;
    dr.x = (T)((double)m.x + u[0] * sc);        // float64 positions, then astype(pool dtype)
    dr.y = (T)((double)m.y + u[1] * sc);
    dr.z = (T)((double)m.z + u[2] * sc);
    dr.d = dh;
    const int j = n + r;
    rec[j] = dr;
    adh[j] = adh[i];
    uid[j] = next_uid + (uint64_t)r;
    dx[j] = dy[j] = dz[j] = T(0);
    if (pres) pres[j] = j;
    rec[i].d = dh;
}

// rng.py:41-54 unit_vector for a batch of uids (the drop-in for the
// reference's per-event generator; the division kernel calls the same code)
__global__ void __launch_bounds__(kThreads) unit_vector_kernel(int n, const uint64_t *__restrict__ uid, uint64_t step,
                                                               double *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) cgb::unit_vector(uid[i], step, out + 3 * i);
}

}  // namespace cg
