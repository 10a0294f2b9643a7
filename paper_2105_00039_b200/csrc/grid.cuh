// grid.cuh -- uniform-grid rebuild on the device (north-star kernel set (a)).
//
// Replaces reference spatial.build_grid (spatial.py:89-127), kernels.py:107-145
// (box ids + linked-cell chains) and the Z-order re-sort (morton.py:93-107,
// pool.py:228-239) with a counting sort into a box-sorted CSR layout:
//   K1 bbox_partial/bbox_final   pool.py:102-110 max_diameter + bounding_box
//   K2 box_keys                  kernels.py:107-129 box ids, warp-aggregated counts
//   K3 scan_*                    exclusive prefix sum of counts -> box offsets
//   K4 place + order_in_box      counting-sort scatter; members of a box ordered by uid
//                                (Morton order) or by (z, uid) (row-major order)
//   K5 morton_table              box -> Morton rank (boxes visited in Z-order)
//   K4b gather_records           apply the permutation (storage re-sort)
#pragma once

#include "common.cuh"

namespace cg {

// ---------------------------------------------------------------- K1 bbox
// Exact min/max reductions (order independent), widened to f64 like numpy's
// col.min()/col.max() -> np.array(float64).  7 values per block:
// min x,y,z, max x,y,z, max diameter.
template <typename T>
__global__ void bbox_partial(int n, const T *__restrict__ x, const T *__restrict__ y,
                             const T *__restrict__ z, const T *__restrict__ d,
                             double *__restrict__ partial)
{
    double v[7] = {INFINITY, INFINITY, INFINITY, -INFINITY, -INFINITY, -INFINITY, -INFINITY};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double px = (double)x[i], py = (double)y[i], pz = (double)z[i];
        v[0] = fmin(v[0], px); v[1] = fmin(v[1], py); v[2] = fmin(v[2], pz);
        v[3] = fmax(v[3], px); v[4] = fmax(v[4], py); v[5] = fmax(v[5], pz);
        v[6] = fmax(v[6], (double)d[i]);
    }
    __shared__ double red[7][kThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        double t = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double u = __shfl_xor_sync(0xffffffffu, t, o);
            t = k < 3 ? fmin(t, u) : fmax(t, u);
        }
        if (lane == 0) red[k][w] = t;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        const int k = threadIdx.x;
        double t = red[k][0];
        for (int q = 1; q < kThreads / 32; ++q) t = k < 3 ? fmin(t, red[k][q]) : fmax(t, red[k][q]);
        partial[blockIdx.x * 7 + k] = t;
    }
}

__global__ void bbox_final(int nblocks, const double *__restrict__ partial, double *__restrict__ out)
{
    if (threadIdx.x < 7) {
        const int k = threadIdx.x;
        double t = partial[k];
        for (int b = 1; b < nblocks; ++b) t = k < 3 ? fmin(t, partial[b * 7 + k]) : fmax(t, partial[b * 7 + k]);
        out[k] = t;
    }
}

// ---------------------------------------------------------------- K5 Morton table
// mrank[flat] = Morton rank of the box, minv[rank] = flat.  Rebuilt only when
// the grid dims change.
__global__ void morton_table(Geometry g, int *__restrict__ mrank, int *__restrict__ minv)
{
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < g.nb; b += gridDim.x * blockDim.x) {
        const int iz = b % g.dimz, rest = b / g.dimz;
        const int iy = rest % g.dimy, ix = rest / g.dimy;
        const int r = (int)morton_rank(ix, iy, iz, g.dimx, g.dimy, g.dimz);
        mrank[b] = r;
        minv[r] = b;
    }
}

// ---------------------------------------------------------------- K2 box keys
// kernels.py:113-128, bit for bit: ix = int64(floor((f64(p) - ox) / L)),
// clamped, flat = (ix*dimy + iy)*dimz + iz.  The counting-sort key is the box's
// visiting rank (Morton rank or flat id).  rank_in_box comes from the
// warp-aggregated atomic; its order is arbitrary and fixed up by K4.
__device__ __forceinline__ int axis_box(double p, double o, double L, int dim)
{
    long long k = (long long)floor((p - o) / L);
    if (k < 0) k = 0;
    else if (k >= dim) k = dim - 1;
    return (int)k;
}

template <typename T>
__device__ __forceinline__ int flat_box(const Geometry &g, T x, T y, T z)
{
    const int ix = axis_box((double)x, g.ox, g.L, g.dimx);
    const int iy = axis_box((double)y, g.oy, g.L, g.dimy);
    const int iz = axis_box((double)z, g.oz, g.L, g.dimz);
    return (ix * g.dimy + iy) * g.dimz + iz;
}

template <typename T>
__global__ void box_keys(int n, Geometry g, const T *__restrict__ x, const T *__restrict__ y,
                         const T *__restrict__ z, const int *__restrict__ mrank,
                         int *__restrict__ count, int *__restrict__ key, int *__restrict__ rank_in_box)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int flat = flat_box(g, x[i], y[i], z[i]);
    const int k = mrank ? __ldg(mrank + flat) : flat;
    rank_in_box[i] = agg_increment(count, k);
    key[i] = k;
}

// Keys from caller-supplied flat box ids (kernel-level force-phase drop-in).
__global__ void keys_from_flat(int n, const long long *__restrict__ box_index, int *__restrict__ count,
                               int *__restrict__ key, int *__restrict__ rank_in_box)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k = (int)box_index[i];
    rank_in_box[i] = agg_increment(count, k);
    key[i] = k;
}

template <typename T>
__global__ void double_column(int n, T *__restrict__ v)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = v[i] * T(2);
}

// Kernel-level drop-in for kernels.box_ids_parallel: flat ids only (int64).
template <typename T>
__global__ void box_ids_only(int n, Geometry g, const T *__restrict__ x, const T *__restrict__ y,
                             const T *__restrict__ z, long long *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = flat_box(g, x[i], y[i], z[i]);
}

// ---------------------------------------------------------------- K3 scan
// Three-phase exclusive scan of the per-box counts (tile = 256 x 8 items).
// Phase 1 also accumulates the StepStats grid figures (occupied boxes, max
// occupancy) into stat[0], stat[1].
constexpr int kScanItems = 8;
constexpr int kScanTile = kThreads * kScanItems;

__device__ __forceinline__ int block_exclusive_scan(int v, int &total)
{
    constexpr int kWarps = kThreads / 32;
    __shared__ int warp_off[kWarps];
    __shared__ int block_tot;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) warp_off[w] = inc;
    __syncthreads();
    if (w == 0) {
        const int t = lane < kWarps ? warp_off[lane] : 0;
        int s = t;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += u;
        }
        if (lane < kWarps) warp_off[lane] = s - t;
        if (lane == kWarps - 1) block_tot = s;
    }
    __syncthreads();
    const int excl = inc - v + warp_off[w];
    total = block_tot;
    __syncthreads();  // warp_off / block_tot are reused by the next call
    return excl;
}

__global__ void scan_tiles(int nb, const int *__restrict__ count, int *__restrict__ offset,
                           int *__restrict__ tile_sum, unsigned long long *__restrict__ stat)
{
    const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    int v[kScanItems];
    int s = 0, occ = 0, mx = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        v[k] = (base + k < nb) ? count[base + k] : 0;
        s += v[k];
        occ += v[k] > 0;
        mx = max(mx, v[k]);
    }
    int total;
    int run = block_exclusive_scan(s, total);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < nb) offset[base + k] = run;
        run += v[k];
    }
    if (threadIdx.x == 0) tile_sum[blockIdx.x] = total;
    occ = warp_sum(occ);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) {
        if (occ) atomicAdd(stat + 0, (unsigned long long)occ);
        atomicMax(stat + 1, (unsigned long long)mx);
    }
}

// Single block: exclusive scan of the tile sums in place (any count).
__global__ void scan_tile_sums(int ntiles, int *__restrict__ tile_sum)
{
    int carry = 0;
    for (int base = 0; base < ntiles; base += kThreads) {
        const int i = base + threadIdx.x;
        const int v = i < ntiles ? tile_sum[i] : 0;
        int total;
        const int ex = block_exclusive_scan(v, total);
        if (i < ntiles) tile_sum[i] = ex + carry;
        carry += total;
    }
}

__global__ void scan_add(int nb, int n, const int *__restrict__ tile_sum, int *__restrict__ offset)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < nb) offset[i] += tile_sum[i / kScanTile];
    if (i == 0) offset[nb] = n;
}

// ---------------------------------------------------------------- K4 place/order
__global__ void place(int n, const int *__restrict__ key, const int *__restrict__ rank_in_box,
                      const int *__restrict__ offset, int *__restrict__ tmp)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) tmp[offset[key[i]] + rank_in_box[i]] = i;
}

// Members of a box are re-ranked so slot order (the summation order of the
// sweep and the storage order after a sort) is a pure function of the
// population: by uid (Morton box order == the reference's lexsort((uid, code)),
// morton.py:67-74) or, for row-major box order, by (z, uid) so that every
// 3-box z-run of the stencil is z-sorted (the sweep's z-window relies on it).
template <typename T, bool BY_Z>
__global__ void order_in_box(int n, const int *__restrict__ tmp, const int *__restrict__ key,
                             const int *__restrict__ offset, const uint64_t *__restrict__ uid,
                             const T *__restrict__ zc, int *__restrict__ idx, int *__restrict__ skey)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int i = tmp[s];
    const int k = key[i];
    const int o0 = offset[k], o1 = offset[k + 1];
    const uint64_t u = uid[i];
    int q = 0;
    if (BY_Z) {
        const T zi = zc[i];
        for (int t = o0; t < o1; ++t) {
            const int j = __ldg(tmp + t);
            const T zj = zc[j];
            q += (zj < zi) || (zj == zi && __ldg(uid + j) < u);
        }
    } else {
        for (int t = o0; t < o1; ++t) q += (__ldg(uid + __ldg(tmp + t)) < u);
    }
    idx[o0 + q] = i;
    skey[o0 + q] = k;
}

// K4b: new storage slot s <- old storage index idx[s] (pool.py:228-239).
template <typename T>
__global__ void gather_records(int n, const int *__restrict__ idx,
                               const T *__restrict__ x0, const T *__restrict__ y0,
                               const T *__restrict__ z0, const T *__restrict__ d0,
                               const T *__restrict__ a0, const uint64_t *__restrict__ u0,
                               T *__restrict__ x1, T *__restrict__ y1, T *__restrict__ z1,
                               T *__restrict__ d1, T *__restrict__ a1, uint64_t *__restrict__ u1)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int i = idx[s];
    x1[s] = x0[i]; y1[s] = y0[i]; z1[s] = z0[i];
    d1[s] = d0[i]; a1[s] = a0[i]; u1[s] = u0[i];
}

}  // namespace cg
