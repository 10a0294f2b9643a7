// grid.cuh -- uniform-grid rebuild on the device (north-star kernel set (a)).
//
// Replaces reference spatial.build_grid (spatial.py:89-127), kernels.py:107-145
// (box ids + linked-cell chains) and the Z-order re-sort (morton.py:93-107,
// pool.py:228-239) with a counting sort into a box-sorted CSR:
//   bbox_slots / finish_step   pool.py:102-110 bounding_box (exact min/max, f64)
//   box_keys                   kernels.py:107-129 box ids + warp-aggregated counts
//   scan_lookback              exclusive prefix sum of counts -> box offsets
//                              (single pass, decoupled look-back; zeroes the counts)
//   place + order_gather       counting-sort scatter; members of a box ordered by
//                              (z, uid); emits the slot-order fp32 proxies, the
//                              slot -> box key and either the slot -> storage
//                              index or (relayout) the records themselves
//   morton_table, presentation the reference's storage order (Morton code, uid),
//                              materialised only when the host asks for it
// Boxes are visited in row-major flat order (z fastest): the 3 boxes of a
// stencil z-run are one contiguous slot range.
#pragma once

#include "common.cuh"

namespace cg {

// Per-step reduction slots: blocks spread their atomics over kSlots slots
// (blockIdx % kSlots) so no address sees more than a few hundred updates.
// slot layout: [0..2] min x,y,z (ordered u64), [3..5] max x,y,z, [6] evals,
// [7] candidates, [8] degenerate pairs, [9] max squared displacement
// (ordered u64), [10] neighbour-list overflows.
constexpr int kSlots = 512;
constexpr int kSlotWords = 11;

// reduction of slot word k: 0 = min, 1 = max, 2 = sum
__device__ __forceinline__ int slot_op(int k)
{
    return k < 3 ? 0 : (k < 6 || k == 9) ? 1 : 2;
}
__device__ __forceinline__ unsigned long long slot_combine(int k, unsigned long long a, unsigned long long b)
{
    const int op = slot_op(k);
    return op == 0 ? min(a, b) : op == 1 ? max(a, b) : a + b;
}

__device__ __forceinline__ double warp_min(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide min/max of 6 values + sums of 3 counters into one slot.
// Must be called by every thread of the block (kThreads threads).
__device__ __forceinline__ void block_to_slot(double lo[3], double hi[3], unsigned long long c[3],
                                              unsigned long long *__restrict__ slots)
{
    __shared__ double s_lo[3][kThreads / 32], s_hi[3][kThreads / 32];
    __shared__ unsigned long long s_c[3][kThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        lo[a] = warp_min(lo[a]);
        hi[a] = warp_max(hi[a]);
        c[a] = warp_sum(c[a]);
    }
    if (lane == 0) {
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            s_lo[a][w] = lo[a];
            s_hi[a][w] = hi[a];
            s_c[a][w] = c[a];
        }
    }
    __syncthreads();
    if (threadIdx.x < 9) {
        const int k = threadIdx.x, a = k % 3;
        unsigned long long *slot = slots + (blockIdx.x % kSlots) * kSlotWords;
        if (k < 3) {
            double v = s_lo[a][0];
            for (int q = 1; q < kThreads / 32; ++q) v = fmin(v, s_lo[a][q]);
            if (v != INFINITY) atomicMin(slot + a, enc_ordered(v));
        } else if (k < 6) {
            double v = s_hi[a][0];
            for (int q = 1; q < kThreads / 32; ++q) v = fmax(v, s_hi[a][q]);
            if (v != -INFINITY) atomicMax(slot + 3 + a, enc_ordered(v));
        } else {
            unsigned long long v = 0;
            for (int q = 0; q < kThreads / 32; ++q) v += s_c[a][q];
            if (v) atomicAdd(slot + 6 + a, v);
        }
    }
}

// Reset value of the slots (min slots at the top of the order, max at the bottom).
__device__ __forceinline__ unsigned long long slot_init(int word)
{
    return word < 3 ? ~0ull : 0ull;
}

__global__ void init_slots(unsigned long long *__restrict__ slots)
{
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < kSlots * kSlotWords; k += gridDim.x * blockDim.x)
        slots[k] = slot_init(k % kSlotWords);
}

// ---------------------------------------------------------------- K1 bbox
// Standalone exact bounding box of the stored positions (after an upload or a
// relayout-free first step); in steady state the sweep epilogue produces the
// same slots from the new positions.
template <typename T>
__global__ void __launch_bounds__(kThreads) bbox_slots(int n, const Rec<T> *__restrict__ rec,
                                                       unsigned long long *__restrict__ slots)
{
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    unsigned long long c[3] = {0, 0, 0};
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const Rec<T> r = rec[i];
        const double p[3] = {(double)r.x, (double)r.y, (double)r.z};
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            lo[a] = fmin(lo[a], p[a]);
            hi[a] = fmax(hi[a], p[a]);
        }
    }
    block_to_slot(lo, hi, c, slots);
}

// One block: fold the slots into stat[2..4] (evals, cands, ndeg) and the
// bbox out[0..5] (+ out[6] = max diameter, which the path never changes),
// then reset the slots for the next step.
enum { FINISH_COUNTERS = 1, FINISH_BBOX = 2 };

__global__ void finish_step(unsigned long long *__restrict__ slots, double max_diameter,
                            unsigned long long *__restrict__ stat, double *__restrict__ bbox_out,
                            int what)
{
    __shared__ unsigned long long red[kSlotWords][kThreads / 32];
    unsigned long long v[kSlotWords];
#pragma unroll
    for (int k = 0; k < kSlotWords; ++k) v[k] = slot_init(k);
    for (int s = threadIdx.x; s < kSlots; s += blockDim.x) {
#pragma unroll
        for (int k = 0; k < kSlotWords; ++k) {
            const unsigned long long u = slots[s * kSlotWords + k];
            v[k] = slot_combine(k, v[k], u);
            slots[s * kSlotWords + k] = slot_init(k);
        }
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < kSlotWords; ++k) {
        unsigned long long t = v[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long u = __shfl_xor_sync(0xffffffffu, t, o);
            t = slot_combine(k, t, u);
        }
        if (lane == 0) red[k][w] = t;
    }
    __syncthreads();
    if (threadIdx.x < kSlotWords) {
        const int k = threadIdx.x;
        unsigned long long t = red[k][0];
        for (int q = 1; q < kThreads / 32; ++q)
            t = slot_combine(k, t, red[k][q]);
        if (k < 6) {
            if (what & FINISH_BBOX) bbox_out[k] = dec_ordered(t);
        } else if (k < 9) {
            if (what & FINISH_COUNTERS) stat[2 + (k - 6)] = t;
        } else if (k == 9) {
            bbox_out[7] = t ? dec_ordered(t) : 0.0;   // max squared displacement of the step
        } else {
            if (what & FINISH_COUNTERS) stat[5] = t;  // neighbour-list overflows
            bbox_out[8] = (double)t;
        }
        if (k == 0 && (what & FINISH_BBOX)) bbox_out[6] = max_diameter;
    }
}

// max(diameter) and min(diameter) once per upload / behaviour phase (the
// mechanical step never changes diameters): out[0] = enc(max), out[1] =
// enc(-min).  A uniform pool (min == max) lets the list sweep take its pair
// constants from the host.
template <typename T>
__global__ void max_diam_kernel(int n, const Rec<T> *__restrict__ rec, unsigned long long *__restrict__ out)
{
    double v = -INFINITY, w = -INFINITY;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const double d = (double)rec[i].d;
        v = fmax(v, d);
        w = fmax(w, -d);
    }
    v = warp_max(v);
    w = warp_max(w);
    if ((threadIdx.x & 31) == 0 && v != -INFINITY) {
        atomicMax(out, enc_ordered(v));
        atomicMax(out + 1, enc_ordered(w));
    }
}

// max(uid) once per upload: every uid below 2^32 lets the sweep take its
// survivor sort keys from the proxies
__global__ void max_uid_kernel(int n, const uint64_t *__restrict__ uid, unsigned long long *__restrict__ out)
{
    unsigned long long v = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        v = max(v, (unsigned long long)uid[i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0 && v) atomicMax(out, v);
}

// ---------------------------------------------------------------- K5 Morton table
// mrank[flat] = Morton rank of the box, minv[rank] = flat.  Rebuilt only when
// the grid dims change (presentation order only).
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
// clamped, flat = (ix*dimy + iy)*dimz + iz.  rank_in_box comes from the
// warp-aggregated atomic; its order is arbitrary and fixed up by order_gather.
__device__ __forceinline__ int axis_box(double p, double o, double L, int dim)
{
    long long k = (long long)floor((p - o) / L);
    if (k < 0) k = 0;
    else if (k >= dim) k = dim - 1;
    return (int)k;
}

// Same value as axis_box without the IEEE division: t = (p - o) * (1/L) is
// within a few ulp of the correctly rounded quotient, so floor(t) is exact
// unless t lies within that distance of an integer -- only then divide.
__device__ __forceinline__ int axis_box_fast(double p, double o, double L, double invL, int dim)
{
    const double q = p - o;
    const double t = q * invL;
    const double k = floor(t);
    double f;
    if (t - k > 1e-12 * fabs(t) + 1e-300 && (k + 1.0) - t > 1e-12 * fabs(t) + 1e-300) f = k;
    else f = floor(q / L);   // near a box face: the reference's expression
    long long kk = (long long)f;
    if (kk < 0) kk = 0;
    else if (kk >= dim) kk = dim - 1;
    return (int)kk;
}

template <typename T>
__device__ __forceinline__ int flat_box_fast(const Geometry &g, double invL, T x, T y, T z)
{
    const int ix = axis_box_fast((double)x, g.ox, g.L, invL, g.gdimx) - g.xoff;
    const int iy = axis_box_fast((double)y, g.oy, g.L, invL, g.dimy);
    const int iz = axis_box_fast((double)z, g.oz, g.L, invL, g.dimz);
    return (ix * g.dimy + iy) * g.dimz + iz;
}

template <typename T>
__device__ __forceinline__ int flat_box(const Geometry &g, T x, T y, T z)
{
    const int ix = axis_box((double)x, g.ox, g.L, g.gdimx) - g.xoff;
    const int iy = axis_box((double)y, g.oy, g.L, g.dimy);
    const int iz = axis_box((double)z, g.oz, g.L, g.dimz);
    return (ix * g.dimy + iy) * g.dimz + iz;
}

// Ranks within a box come from one atomicAdd per run of equal keys in the
// warp (storage is box-sorted from the previous step, so keys arrive in runs;
// a key split over several runs just takes several atomics).
template <typename T>
__global__ void __launch_bounds__(kThreads) box_keys(int n, Geometry g, double invL, const Rec<T> *__restrict__ rec,
                                                     int *__restrict__ count, int2 *__restrict__ key_rank)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    int flat = -1 - lane;   // distinct dummy keys for lanes past n
    if (i < n) {
        const Rec<T> r = rec[i];
        flat = flat_box_fast(g, invL, r.x, r.y, r.z);
    }
    const int prev = __shfl_up_sync(0xffffffffu, flat, 1);
    const bool start = lane == 0 || prev != flat;
    const unsigned starts = __ballot_sync(0xffffffffu, start);
    const unsigned upto = starts & (0xffffffffu >> (31 - lane));   // run starts at or below lane
    const int leader = 31 - __clz(upto);
    const unsigned after = starts & ~(0xffffffffu >> (31 - leader));   // starts above the leader
    const int run_end = after ? __ffs(after) - 1 : 32;
    int base = 0;
    if (start && i < n) base = atomicAdd(count + flat, run_end - lane);
    base = __shfl_sync(0xffffffffu, base, leader);
    if (i < n) key_rank[i] = make_int2(flat, base + (lane - leader));
}

// Keys from caller-supplied flat box ids (kernel-level force-phase drop-in).
__global__ void keys_from_flat(int n, const long long *__restrict__ box_index, int *__restrict__ count,
                               int2 *__restrict__ key_rank)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int k = (int)box_index[i];
    key_rank[i] = make_int2(k, agg_increment(count, k));
}

template <typename T>
__global__ void double_diameter(int n, Rec<T> *__restrict__ rec)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) rec[i].d = rec[i].d * T(2);
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
// Single-pass exclusive scan with decoupled look-back (tiles of 256 x 16
// boxes, dynamic tile order so predecessors always make progress).  Reads the
// counts, writes the offsets (nb + 1 entries, offset[nb] = total), zeroes the
// counts for the next build, and accumulates the StepStats grid figures
// (occupied boxes, max occupancy) into stat[0], stat[1].
// MORTON: the counts are taken in Morton rank order from an existing CSR
// (cnt(r) = off[minv[r]+1] - off[minv[r]]) -- the presentation order scan.
constexpr int kScanItems = 16;
constexpr int kScanTile = kThreads * kScanItems;

struct ScanState {
    unsigned long long *status;   // per tile: (flag << 32) | value;  flag 1 = aggregate, 2 = prefix
    unsigned *ticket;             // dynamic tile counter
};

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

// Reduce-then-scan (grid path): scan_reduce writes each tile's sum,
// scan_tilesums scans them in one CTA, scan_down produces the offsets,
// zeroes the counts and accumulates the grid statistics.
__device__ __forceinline__ void load_tile(int nb, const int *__restrict__ count, int base, int v[kScanItems])
{
    if (base + kScanItems <= nb) {
        const int4 *p = reinterpret_cast<const int4 *>(count + base);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            const int4 u = p[q];
            v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) v[k] = base + k < nb ? count[base + k] : 0;
    }
}

__global__ void __launch_bounds__(kThreads) scan_reduce(int nb, const int *__restrict__ count,
                                                        int *__restrict__ tile_sum)
{
    int v[kScanItems];
    load_tile(nb, count, blockIdx.x * kScanTile + threadIdx.x * kScanItems, v);
    int s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) s += v[k];
    s = __reduce_add_sync(0xffffffffu, (unsigned)s);
    __shared__ int ws[kThreads / 32];
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int t = 0;
        for (int w = 0; w < kThreads / 32; ++w) t += ws[w];
        tile_sum[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(1024) scan_tilesums(int ntiles, int *__restrict__ tile_sum)
{
    // exclusive scan in place, 1024 threads, any count
    __shared__ int warp_tot[32];
    __shared__ int carry_sh;
    if (threadIdx.x == 0) carry_sh = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int base = 0; base < ntiles; base += 1024) {
        const int i = base + threadIdx.x;
        const int v = i < ntiles ? tile_sum[i] : 0;
        int inc = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) warp_tot[w] = inc;
        __syncthreads();
        if (w == 0) {
            const int t = warp_tot[lane];
            int s2 = t;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int u = __shfl_up_sync(0xffffffffu, s2, o);
                if (lane >= o) s2 += u;
            }
            warp_tot[lane] = s2 - t;
        }
        __syncthreads();
        const int carry = carry_sh;
        if (i < ntiles) tile_sum[i] = carry + warp_tot[w] + inc - v;
        __syncthreads();
        if (threadIdx.x == 1023) carry_sh = carry + warp_tot[31] + inc;
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) scan_down(int nb, int *__restrict__ count,
                                                      const int *__restrict__ tile_sum, int *__restrict__ offset,
                                                      unsigned long long *__restrict__ stat)
{
    const int base = blockIdx.x * kScanTile + threadIdx.x * kScanItems;
    int v[kScanItems];
    load_tile(nb, count, base, v);
    int s = 0, occ = 0, mx = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        s += v[k];
        occ += v[k] > 0;
        mx = max(mx, v[k]);
    }
    int total;
    int run = block_exclusive_scan(s, total) + tile_sum[blockIdx.x];
    if (base + kScanItems <= nb) {
        int4 *po = reinterpret_cast<int4 *>(offset + base);
        int4 *pc = reinterpret_cast<int4 *>(count + base);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            int4 o;
            o.x = run; run += v[4 * q];
            o.y = run; run += v[4 * q + 1];
            o.z = run; run += v[4 * q + 2];
            o.w = run; run += v[4 * q + 3];
            po[q] = o;
            pc[q] = make_int4(0, 0, 0, 0);
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            if (base + k < nb) {
                offset[base + k] = run;
                count[base + k] = 0;
            }
            run += v[k];
        }
    }
    if (base <= nb - 1 && nb - 1 < base + kScanItems) offset[nb] = run;
    occ = __reduce_add_sync(0xffffffffu, (unsigned)occ);
    mx = (int)__reduce_max_sync(0xffffffffu, (unsigned)mx);
    if ((threadIdx.x & 31) == 0 && stat) {
        if (occ) atomicAdd(stat + 0, (unsigned long long)occ);
        if (mx) atomicMax(stat + 1, (unsigned long long)mx);
    }
}

template <bool MORTON>
__global__ void __launch_bounds__(kThreads) scan_lookback(int nb, int *__restrict__ count,
                                                          const int *__restrict__ src_off,
                                                          const int *__restrict__ minv,
                                                          int *__restrict__ offset, ScanState S,
                                                          unsigned long long *__restrict__ stat)
{
    __shared__ unsigned tile_sh;
    __shared__ int prefix_sh;
    if (threadIdx.x == 0) tile_sh = atomicAdd(S.ticket, 1u);
    __syncthreads();
    const int tile = (int)tile_sh;
    const int base = tile * kScanTile + threadIdx.x * kScanItems;
    int v[kScanItems];
    int s = 0, occ = 0, mx = 0;
    if (!MORTON && base + kScanItems <= nb) {
        int4 *p = reinterpret_cast<int4 *>(count + base);
#pragma unroll
        for (int q = 0; q < kScanItems / 4; ++q) {
            const int4 u = p[q];
            v[4 * q] = u.x; v[4 * q + 1] = u.y; v[4 * q + 2] = u.z; v[4 * q + 3] = u.w;
            p[q] = make_int4(0, 0, 0, 0);
        }
    } else {
#pragma unroll
        for (int k = 0; k < kScanItems; ++k) {
            const int b = base + k;
            if (b < nb) {
                if (MORTON) {
                    const int f = __ldg(minv + b);
                    v[k] = __ldg(src_off + f + 1) - __ldg(src_off + f);
                } else {
                    v[k] = count[b];
                    count[b] = 0;
                }
            } else {
                v[k] = 0;
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        s += v[k];
        occ += v[k] > 0;
        mx = max(mx, v[k]);
    }
    int total;
    const int run0 = block_exclusive_scan(s, total);
    // publish, then look back (warp 0)
    if (threadIdx.x < 32) {
        if (tile == 0) {
            if (threadIdx.x == 0) {
                atomicExch(S.status, (2ull << 32) | (unsigned)total);
                prefix_sh = 0;
            }
        } else {
            if (threadIdx.x == 0) atomicExch(S.status + tile, (1ull << 32) | (unsigned)total);
            int excl = 0;
            int pos = tile - 1;   // this lane inspects tile pos - lane
            while (true) {
                const int t = pos - (int)threadIdx.x;
                unsigned long long st = t >= 0 ? *((volatile unsigned long long *)(S.status + t)) : (2ull << 32);
                unsigned flag = (unsigned)(st >> 32);
                // wait until every inspected predecessor has published
                while (__any_sync(0xffffffffu, flag == 0)) {
                    st = t >= 0 ? *((volatile unsigned long long *)(S.status + t)) : (2ull << 32);
                    flag = (unsigned)(st >> 32);
                }
                const unsigned prefix_mask = __ballot_sync(0xffffffffu, flag == 2);
                // sum values from lane 0 up to (and including) the first prefix lane
                const int stop = prefix_mask ? __ffs(prefix_mask) - 1 : 31;
                int val = ((int)threadIdx.x <= stop && t >= 0) ? (int)(unsigned)st : 0;
                val = warp_sum(val);
                excl += val;
                if (prefix_mask) break;
                pos -= 32;
            }
            if (threadIdx.x == 0) {
                atomicExch(S.status + tile, (2ull << 32) | (unsigned)(excl + total));
                prefix_sh = excl;
            }
        }
    }
    __syncthreads();
    int run = run0 + prefix_sh;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (base + k < nb) offset[base + k] = run;
        run += v[k];
    }
    if (base + kScanItems >= nb && base < nb + kScanItems && base <= nb && base + kScanItems > nb - 1)
        ;   // (the last element's successor is written below)
    if (base <= nb - 1 && nb - 1 < base + kScanItems) offset[nb] = run;
    if (stat) {
        occ = warp_sum(occ);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if ((threadIdx.x & 31) == 0) {
            if (occ) atomicAdd(stat + 0, (unsigned long long)occ);
            if (mx) atomicMax(stat + 1, (unsigned long long)mx);
        }
    }
}

// ---------------------------------------------------------------- K4 place/order

__global__ void __launch_bounds__(kThreads) place(int n, const int2 *__restrict__ key_rank,
                                                  const int *__restrict__ offset, int *__restrict__ tmp)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int2 kr = key_rank[i];
    tmp[__ldg(offset + kr.x) + kr.y] = i;
}

// fp32 proxies in slot order, one 32-byte record per slot pair so the sweep
// loads two candidates with one sector pair and tests them with one packed
// FADD2/FFMA2 chain:
//   p[8q .. 8q+7] = (x_2q, x_2q+1, y_2q, y_2q+1, z_2q, z_2q+1, u_2q, u_2q+1)
// u = the low 32 bits of the uid (the survivor sort key when every uid is
// below 2^32 -- the sweep then never loads the uid column).
// x/y box-local (|err| <= ulp(L)), z grid-relative (monotone, so z-sorted
// boxes stay sorted).  The candidate's radius is not stored: the sweep bounds
// it by the pool's largest radius (conservative).
struct Proxies {
    float *p;
};

template <typename T>
__device__ __forceinline__ void put_proxy(const Proxies &P, const Geometry &g, int s, int ix, int iy, T x, T y, T z,
                                          uint64_t uid)
{
    float *r = P.p + 8 * (s >> 1) + (s & 1);
    r[0] = (float)((double)x - (g.ox + (double)(ix + g.xoff) * g.L));
    r[2] = (float)((double)y - (g.oy + (double)iy * g.L));
    r[4] = (float)((double)z - g.oz);
    reinterpret_cast<unsigned *>(r)[6] = (unsigned)uid;
}

// Members of a box are re-ranked by (z, uid) -- a pure function of the
// population, so slot order (the stencil summation order and the storage
// order after a relayout) is deterministic -- and every 3-box z-run of a
// stencil is one z-sorted slot range.  Emits skey/prox per slot and either
// idx (slot -> storage) or, when RELAYOUT, the records in slot order.
template <typename T, bool RELAYOUT>
__global__ void __launch_bounds__(kThreads) order_gather(
    int n, Geometry g, BoxDecode bd, const int *__restrict__ tmp, const int2 *__restrict__ key_rank,
    const int *__restrict__ offset, const Rec<T> *__restrict__ rec, const T *__restrict__ adh,
    const uint64_t *__restrict__ uid, int *__restrict__ skey, Proxies prox,
    int *__restrict__ idx, Rec<T> *__restrict__ orec, T *__restrict__ oadh, uint64_t *__restrict__ ouid,
    int *__restrict__ pkey)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int i = tmp[s];
    const int k = key_rank[i].x;
    const int o0 = __ldg(offset + k), o1 = __ldg(offset + k + 1);
    const Rec<T> ri = rec[i];
    const T zi = ri.z;
    const uint64_t ui = uid[i];
    int q = 0;
    for (int t = o0; t < o1; ++t) {
        const int j = __ldg(tmp + t);
        const T zj = rec[j].z;
        q += (zj < zi) || (zj == zi && uid[j] < ui);
    }
    const int dst = o0 + q;
    int ix, iy, iz;
    decode_box(bd, k, ix, iy, iz);
    skey[dst] = k;
    put_proxy<T>(prox, g, dst, ix, iy, ri.x, ri.y, zi, ui);
    if (RELAYOUT) {
        orec[dst] = ri;
        oadh[dst] = adh[i];
        ouid[dst] = ui;
        if (pkey) pkey[dst] = k;
    } else {
        idx[dst] = i;
        if (pkey) pkey[i] = k;
    }
}

// Sparse pools: the counting-sort scatter is the whole CSR build -- members
// of a box keep their (arbitrary) atomic rank, the sweep sums each agent's
// pairs in uid order.  One thread per storage index writes idx / skey / the
// proxies of its slot, and (sort steps) its box key for the lazy reference
// storage order.
template <typename T>
__global__ void __launch_bounds__(kThreads) place_full(int n, Geometry g, BoxDecode bd,
                                                       const int2 *__restrict__ key_rank,
                                                       const int *__restrict__ offset, const Rec<T> *__restrict__ rec,
                                                       int *__restrict__ idx, int *__restrict__ skey,
                                                       Proxies prox, int *__restrict__ pkey,
                                                       const uint64_t *__restrict__ uid)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int2 kr = key_rank[i];
    const int slot = __ldg(offset + kr.x) + kr.y;
    int ix, iy, iz;
    decode_box(bd, kr.x, ix, iy, iz);
    idx[slot] = i;
    skey[slot] = kr.x;
    const Rec<T> r = rec[i];
    put_proxy<T>(prox, g, slot, ix, iy, r.x, r.y, r.z, uid[i]);
    if (pkey) pkey[i] = kr.x;
}

// place_full + relayout in one pass: the agent's whole record goes straight
// to its slot (storage becomes slot order; no slot -> storage index needed).
template <typename T>
__global__ void __launch_bounds__(kThreads) place_relayout(
    int n, Geometry g, BoxDecode bd, const int2 *__restrict__ key_rank, const int *__restrict__ offset,
    const Rec<T> *__restrict__ rec, const T *__restrict__ adh, const uint64_t *__restrict__ uid,
    int *__restrict__ skey, Proxies prox, const int *__restrict__ pkey_sort_in, int *__restrict__ pkey_out,
    Rec<T> *__restrict__ orec, T *__restrict__ oadh, uint64_t *__restrict__ ouid)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int2 kr = key_rank[i];
    const int slot = __ldg(offset + kr.x) + kr.y;
    int ix, iy, iz;
    decode_box(bd, kr.x, ix, iy, iz);
    const Rec<T> r = rec[i];
    skey[slot] = kr.x;
    put_proxy<T>(prox, g, slot, ix, iy, r.x, r.y, r.z, uid[i]);
    orec[slot] = r;
    oadh[slot] = adh[i];
    ouid[slot] = uid[i];
    // pkey: this step's box when it is a sort step, else the carried value
    if (pkey_out) pkey_out[slot] = pkey_sort_in ? pkey_sort_in[i] : kr.x;
}

// Move the records into slot order (locality for the sweep; the paper's
// Z-order data sort).  pkey travels with them.
template <typename T>
__global__ void __launch_bounds__(kThreads) relayout_records(
    int n, const int *__restrict__ idx, const Rec<T> *__restrict__ rec, const T *__restrict__ adh,
    const uint64_t *__restrict__ uid, const int *__restrict__ pkey, Rec<T> *__restrict__ orec,
    T *__restrict__ oadh, uint64_t *__restrict__ ouid, int *__restrict__ opkey)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int i = idx[s];
    orec[s] = rec[i];
    oadh[s] = adh[i];
    ouid[s] = uid[i];
    if (pkey) opkey[s] = pkey[i];
}

// ---------------------------------------------------------------- presentation
// The reference's storage order after a sorted step (morton.py:67-74,
// lexsort((uid, code))) is materialised lazily, at download/export time, from
// pkey (box of every agent at the last sort step) and uid:
//   1. sort storage indices by uid,  2. stable-sort them by Morton rank of pkey,
//   3. pres[order[r]] = r.
__global__ void morton_keys(int n, const int *__restrict__ order, const int *__restrict__ pkey,
                            const int *__restrict__ mrank, unsigned *__restrict__ out)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) out[r] = (unsigned)__ldg(mrank + pkey[order[r]]);
}

// ---------------------------------------------------------------- presentation order
// The reference's storage order after a sort step (morton.py:67-74,
// pool.py:228-239): ascending (Morton code of the agent's box, uid).  A
// counting sort by the box's Morton rank (pres_count -> scan -> pres_scatter)
// puts every box's agents in one segment; inside a segment an agent's place
// is the number of segment members with a smaller uid (pres_rank; boxes hold
// a handful of agents, the few crowded ones take pres_rank_big: one CTA per
// segment, uids staged through shared memory).  pres[a] = reference
// position of storage index a.
constexpr int kPresSmallSeg = 256;

__global__ void __launch_bounds__(kThreads) pres_count(int n, const int *__restrict__ pkey,
                                                       const int *__restrict__ mrank, int *__restrict__ cnt,
                                                       int *__restrict__ rkey, int *__restrict__ slot)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const int r = __ldg(mrank + __ldg(pkey + a));
    rkey[a] = r;
    slot[a] = atomicAdd(cnt + r, 1);
}

__global__ void __launch_bounds__(kThreads) pres_scatter(int n, const int *__restrict__ rkey,
                                                         const int *__restrict__ slot, const int *__restrict__ off,
                                                         int *__restrict__ seg)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a < n) seg[__ldg(off + rkey[a]) + slot[a]] = a;
}

__global__ void __launch_bounds__(kThreads) pres_rank(int n, const int *__restrict__ rkey,
                                                      const int *__restrict__ slot, const int *__restrict__ off,
                                                      const int *__restrict__ seg, const uint64_t *__restrict__ uid,
                                                      int *__restrict__ pres, int *__restrict__ big,
                                                      unsigned *__restrict__ nbig)
{
    const int a = blockIdx.x * blockDim.x + threadIdx.x;
    if (a >= n) return;
    const int r = rkey[a];
    const int s0 = __ldg(off + r), s1 = __ldg(off + r + 1);
    if (s1 - s0 > kPresSmallSeg) {   // crowded box: one CTA sorts it (listed once, by its slot-0 agent)
        if (slot[a] == 0) big[atomicAdd(nbig, 1u)] = r;
        return;
    }
    const uint64_t u = uid[a];
    int rank = 0;
    for (int p = s0; p < s1; ++p) rank += uid[__ldg(seg + p)] < u;
    pres[a] = s0 + rank;
}

__global__ void __launch_bounds__(1024) pres_rank_big(const int *__restrict__ big, const unsigned *__restrict__ nbig,
                                                      const int *__restrict__ off, const int *__restrict__ seg,
                                                      const uint64_t *__restrict__ uid, int *__restrict__ pres)
{
    __shared__ uint64_t tile[1024];
    for (unsigned b = blockIdx.x; b < *nbig; b += gridDim.x) {
        const int r = big[b];
        const int s0 = off[r], s1 = off[r + 1];
        for (int base = s0; base < s1; base += blockDim.x) {   // this thread's agent: seg[base + tid]
            const int p = base + threadIdx.x;
            const int a = p < s1 ? seg[p] : -1;
            const uint64_t u = a >= 0 ? uid[a] : 0;
            int rank = 0;
            for (int t0 = s0; t0 < s1; t0 += blockDim.x) {   // uids of the segment, one tile at a time
                __syncthreads();
                if (t0 + (int)threadIdx.x < s1) tile[threadIdx.x] = uid[seg[t0 + threadIdx.x]];
                __syncthreads();
                const int m = min((int)blockDim.x, s1 - t0);
                for (int q = 0; q < m; ++q) rank += tile[q] < u;
            }
            if (a >= 0) pres[a] = s0 + rank;
        }
        __syncthreads();
    }
}

__global__ void invert_perm(int n, const int *__restrict__ order, int *__restrict__ pres)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) pres[order[r]] = r;
}

// SoA host columns <-> device records (upload / download).  unpack writes
// component c of agent i to out[pres ? pres[i] : i].
template <typename T>
__global__ void pack_records(int n, const T *__restrict__ x, const T *__restrict__ y, const T *__restrict__ z,
                             const T *__restrict__ d, Rec<T> *__restrict__ rec)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    Rec<T> r;
    r.x = x[i];
    r.y = y[i];
    r.z = z[i];
    r.d = d[i];
    rec[i] = r;
}

template <typename T>
__global__ void unpack_component(int n, const Rec<T> *__restrict__ rec, int c, const int *__restrict__ pres,
                                 T *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const Rec<T> r = rec[i];
    const T v = c == 0 ? r.x : (c == 1 ? r.y : (c == 2 ? r.z : r.d));
    out[pres ? pres[i] : i] = v;
}

// dst[pres[i]] = src[i] (download / export in the reference's order)
template <typename W>
__global__ void scatter_by(int n, const int *__restrict__ pres, const W *__restrict__ src, W *__restrict__ dst)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[pres[i]] = src[i];
}

__global__ void iota(int n, int *__restrict__ v)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = i;
}

// storage-order box index of the last grid (for exports)
__global__ void key_of_storage(int n, const int2 *__restrict__ key_rank, int *__restrict__ out)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = key_rank[i].x;
}

}  // namespace cg
