// slab.cuh -- x-slab decomposition of the step across GPUs.
// Every rank derives the same global geometry from an all-reduced bbox; rank r
// owns the agents whose global box plane ix lies in [X_r, X_r+1),
// X_k = floor(k * dimx / world), and sees the agents of planes X_r - 1 and
// X_r+1 as this step's ghosts.  ONE exchange round per step:
//   slab_dest          per owned agent: owner rank q under the new geometry,
//                      and whether it is a ghost of q+1 (plane X_q+1 - 1) /
//                      of q-1 (plane X_q); per-destination histogram of
//                      (migrants, lo ghosts, hi ghosts)
//   slab_lists         outgoing agents / holes / tail movers
//   slab_pack_out      outgoing records grouped by destination rank, each
//                      destination's run = [migrants][its lo ghosts][its hi ghosts]
//   slab_fill_holes    tail agents that stay move into the holes departures left
//   slab_unpack_segs   received runs: migrants appended to the owned set, lo
//                      ghosts then hi ghosts after it
// A record is the agent's full state: x, y, z, d, adh, dx, dy, dz (pool dtype)
// and uid -- so migration moves the whole pool row (pool.py:58-66).
#pragma once

#include "common.cuh"
#include "grid.cuh"

namespace cg {

template <typename T>
struct SlabRecord {
    T v[8];          // x, y, z, diameter, adherence, disp x, y, z
    uint64_t uid;
};

template <typename T>
struct SlabCols {
    Rec<T> *rec;
    T *adh, *dx, *dy, *dz;
    uint64_t *uid;
};

constexpr int kMaxWorld = 64;

struct SlabBounds {
    int world;
    int x[kMaxWorld + 1];   // plane bounds X_0 .. X_world
};

__device__ __forceinline__ int slab_owner(const SlabBounds &B, int ix)
{
    int r = 0;
    while (r + 1 < B.world && B.x[r + 1] <= ix) ++r;
    return r;
}

// dest byte: owner rank (6 bits) | 0x40 ghost of owner+1 | 0x80 ghost of owner-1
constexpr unsigned char kGhostUp = 0x40, kGhostDown = 0x80;

// hist layout (kHist entries): [3q + 0] migrants to q (q != rank), [3q + 1]
// lo ghosts of q, [3q + 2] hi ghosts of q, [3 world] agents that stay
constexpr int kHist = 3 * kMaxWorld + 1;

template <typename T>
__global__ void __launch_bounds__(kThreads) slab_dest(int n, Geometry g, SlabBounds B, int rank,
                                                     const Rec<T> *__restrict__ rec,
                                                     unsigned char *__restrict__ dest,
                                                     unsigned long long *__restrict__ counts)
{
    // grid-stride; per-block histogram in shared memory so the global counters
    // see one atomic per (block, bin) -- a same-address atomic per warp
    // serialised at L2 (0.45 ms at C4)
    __shared__ unsigned hist[kHist];
    const int W = B.world;
    for (int k = threadIdx.x; k <= 3 * W; k += blockDim.x) hist[k] = 0;
    __syncthreads();
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int ix = axis_box((double)rec[i].x, g.ox, g.L, g.gdimx);
        const int q = slab_owner(B, ix);
        const bool up = q + 1 < W && ix == B.x[q + 1] - 1;   // in the lo ghost plane of q + 1
        const bool down = q > 0 && ix == B.x[q];               // in the hi ghost plane of q - 1
        dest[i] = (unsigned char)(q | (up ? kGhostUp : 0) | (down ? kGhostDown : 0));
        const unsigned act = __activemask();
        const int bin = q == rank ? 3 * W : 3 * q;
        const unsigned peers = __match_any_sync(act, bin);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + bin, (unsigned)__popc(peers));
        if (up) atomicAdd(hist + 3 * (q + 1) + 1, 1u);
        if (down) atomicAdd(hist + 3 * (q - 1) + 2, 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k <= 3 * W; k += blockDim.x)
        if (hist[k]) atomicAdd(counts + k, (unsigned long long)hist[k]);
}

// list[atomic cursor++] = v for the lanes with pred: one atomic per warp
__device__ __forceinline__ void warp_append(bool pred, unsigned *cursor, int *list, int v)
{
    const unsigned act = __activemask();
    const unsigned m = __ballot_sync(act, pred);
    if (!m) return;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(m) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(cursor, (unsigned)__popc(m));
    base = __shfl_sync(act, base, leader);
    if (pred) list[base + __popc(m & ((1u << lane) - 1))] = v;
}

// outgoing (leaving, or a ghost of a neighbour) -> out; holes = departures
// below n_keep; movers = staying agents at or above n_keep (|holes| == |movers|)
__global__ void slab_lists(int n, int n_keep, int rank, const unsigned char *__restrict__ dest,
                           int *__restrict__ out, int *__restrict__ holes, int *__restrict__ movers,
                           unsigned *__restrict__ cnt /* out, holes, movers */)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned char d = dest[i];
    const bool leaving = (d & 63) != rank;
    warp_append(leaving || (d & (kGhostUp | kGhostDown)), cnt + 0, out, i);
    warp_append(leaving && i < n_keep, cnt + 1, holes, i);
    warp_append(!leaving && i >= n_keep, cnt + 2, movers, i);
}

template <typename T>
__device__ __forceinline__ void load_record(const SlabCols<T> &C, int i, SlabRecord<T> &r)
{
    const Rec<T> p = C.rec[i];
    r.v[0] = p.x;
    r.v[1] = p.y;
    r.v[2] = p.z;
    r.v[3] = p.d;
    r.v[4] = C.adh[i];
    r.v[5] = C.dx[i];
    r.v[6] = C.dy[i];
    r.v[7] = C.dz[i];
    r.uid = C.uid[i];
}

template <typename T>
__device__ __forceinline__ void store_record(const SlabCols<T> &C, int i, const SlabRecord<T> &r)
{
    Rec<T> p;
    p.x = r.v[0];
    p.y = r.v[1];
    p.z = r.v[2];
    p.d = r.v[3];
    C.rec[i] = p;
    C.adh[i] = r.v[4];
    C.dx[i] = r.v[5];
    C.dy[i] = r.v[6];
    C.dz[i] = r.v[7];
    C.uid[i] = r.uid;
}

// outgoing records: run (destination q, kind) starts at seg_off[3q + kind]
// (kind 0 migrant, 1 lo ghost of q, 2 hi ghost of q); order within a run is
// arbitrary (the step's results do not depend on storage order)
template <typename T>
__global__ void slab_pack_out(int nout, int rank, const int *__restrict__ out_list,
                              const unsigned char *__restrict__ dest, const unsigned long long *__restrict__ seg_off,
                              unsigned *__restrict__ cursor, SlabCols<T> C, SlabRecord<T> *__restrict__ out)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nout) return;
    const int i = out_list[k];
    const unsigned char d = dest[i];
    const int q = d & 63;
    SlabRecord<T> rec;
    load_record(C, i, rec);
    if (q != rank) out[seg_off[3 * q] + atomicAdd(cursor + 3 * q, 1u)] = rec;
    if (d & kGhostUp) out[seg_off[3 * (q + 1) + 1] + atomicAdd(cursor + 3 * (q + 1) + 1, 1u)] = rec;
    if (d & kGhostDown) out[seg_off[3 * (q - 1) + 2] + atomicAdd(cursor + 3 * (q - 1) + 2, 1u)] = rec;
}

template <typename T>
__global__ void slab_fill_holes(int nmove, const int *__restrict__ holes, const int *__restrict__ movers,
                                SlabCols<T> C)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= nmove) return;
    SlabRecord<T> rec;
    load_record(C, movers[k], rec);
    store_record(C, holes[k], rec);
}

// received runs -> storage: seg k covers records [start[k], start[k+1]) of the
// receive buffer and lands at storage dst[k] + (record - start[k])
struct SlabSegs {
    int nseg;
    long long start[3 * kMaxWorld + 1];
    int dst[3 * kMaxWorld];
};

template <typename T>
__global__ void slab_unpack_segs(int total, SlabSegs S, const SlabRecord<T> *__restrict__ in, SlabCols<T> C)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= total) return;
    int s = 0;
    while (S.start[s + 1] <= k) ++s;
    store_record(C, S.dst[s] + (int)(k - S.start[s]), in[k]);
}

}  // namespace cg
