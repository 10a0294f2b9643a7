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
    int band;               // ghost planes on each side of a slab (1; 3 with neighbour lists)
    int x[kMaxWorld + 1];   // plane bounds X_0 .. X_world
};

__device__ __forceinline__ int slab_owner(const SlabBounds &B, int ix)
{
    int r = 0;
    while (r + 1 < B.world && B.x[r + 1] <= ix) ++r;
    return r;
}

// f(q', kind) for every other rank q' whose ghost band holds plane ix (owned
// by q): kind 1 = within band planes below q''s slab, 2 = above it
template <typename F>
__device__ __forceinline__ void for_each_ghost_dest(const SlabBounds &B, int ix, int q, F &&f)
{
    for (int r = q + 1; r < B.world && B.x[r] - B.band <= ix; ++r) f(r, 1);
    for (int r = q - 1; r >= 0 && B.x[r + 1] + B.band > ix; --r) f(r, 2);
}

// dest byte: owner rank (6 bits) | 0x40 ghost of some other rank
constexpr unsigned char kGhostAny = 0x40;

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
        bool ghost = false;
        for_each_ghost_dest(B, ix, q, [&](int r, int kind) {
            atomicAdd(hist + 3 * r + kind, 1u);
            ghost = true;
        });
        dest[i] = (unsigned char)(q | (ghost ? kGhostAny : 0));
        const unsigned act = __activemask();
        const int bin = q == rank ? 3 * W : 3 * q;
        const unsigned peers = __match_any_sync(act, bin);
        if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(hist + bin, (unsigned)__popc(peers));
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
    warp_append(leaving || (d & kGhostAny), cnt + 0, out, i);
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
__global__ void slab_pack_out(int nout, int rank, Geometry g, SlabBounds B, const int *__restrict__ out_list,
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
    if (d & kGhostAny) {
        const int ix = axis_box((double)rec.v[0], g.ox, g.L, g.gdimx);
        for_each_ghost_dest(B, ix, q, [&](int r, int kind) {
            out[seg_off[3 * r + kind] + atomicAdd(cursor + 3 * r + kind, 1u)] = rec;
        });
    }
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


// ------------------------------------------------------------ neighbour lists across slabs
// Between list rebuilds the partition is frozen: every rank keeps its owned
// agents and the ghost set it received at the rebuild (a band of 3 planes on
// each side, so every agent that can enter an owned agent's 27 boxes before
// the next rebuild is present), and each step the owners refresh the ghosts'
// records.  Indices are the build step's (relaid) indices; the buffers are
// addressed at index - rot (lo ghosts in the front headroom).

// ghost table: a hash map uid -> ghost index over [0, lo) U [lo + n_owned,
// n_total) (open addressing, linear probing; a slot is claimed through its
// value word, -1 = empty), so refresh records can be matched by uid without
// sorting.  Built once per list epoch.
__device__ __forceinline__ unsigned uid_hash(uint64_t u, unsigned mask)
{
    u ^= u >> 33;
    u *= 0xff51afd7ed558ccdULL;
    u ^= u >> 33;
    return (unsigned)u & mask;
}

__global__ void slab_ghost_hash(int n_total, int lo, int n_owned, const uint64_t *__restrict__ uid,
                                uint64_t *__restrict__ hkey, int *__restrict__ hval, unsigned mask)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int ng = n_total - n_owned;
    if (k >= ng) return;
    const int i = k < lo ? k : k + n_owned;
    const uint64_t u = uid[i];
    for (unsigned h = uid_hash(u, mask);; h = (h + 1) & mask) {
        if (atomicCAS(hval + h, -1, i) == -1) {
            hkey[h] = u;
            return;
        }
    }
}

__device__ __forceinline__ int ghost_lookup(const uint64_t *__restrict__ hkey, const int *__restrict__ hval,
                                            unsigned mask, uint64_t u)
{
    for (unsigned h = uid_hash(u, mask);; h = (h + 1) & mask) {
        const int v = hval[h];
        if (v < 0) return -1;
        if (hkey[h] == u) return v;
    }
}

// refresh lists: owned agents in another rank's ghost band (at the build
// positions), pass 0 counts per (rank, kind) bin, pass 1 fills the runs
template <typename T, bool FILL>
__global__ void slab_refresh_lists(int n_owned, int lo, Geometry g, SlabBounds B, const Rec<T> *__restrict__ rec,
                                   unsigned long long *__restrict__ counts, const unsigned long long *__restrict__ run_off,
                                   unsigned *__restrict__ cursor, int *__restrict__ list)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n_owned) return;
    const int i = lo + k;
    const int ix = axis_box((double)rec[i].x, g.ox, g.L, g.gdimx);
    const int q = slab_owner(B, ix);
    for_each_ghost_dest(B, ix, q, [&](int r, int kind) {
        const int bin = 3 * r + kind;
        if (FILL) list[run_off[bin] + atomicAdd(cursor + bin, 1u)] = i;
        else atomicAdd(counts + bin, 1ull);
    });
}

template <typename T>
__global__ void slab_refresh_pack(int count, const int *__restrict__ list, SlabCols<T> C,
                                  SlabRecord<T> *__restrict__ out)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    SlabRecord<T> r;
    load_record(C, list[k], r);
    out[k] = r;
}

// the first refresh of a list epoch: every received record finds its ghost
// by uid (r2g remembers it: the runs arrive in the same order every step of
// the epoch); later refreshes only check the uid (slab_refresh_apply).
// Unmatched records count in *mismatch, read back with the next bbox.
template <typename T>
__global__ void slab_refresh_match(int count, const SlabRecord<T> *__restrict__ in, const uint64_t *__restrict__ hkey,
                                   const int *__restrict__ hval, unsigned mask, int *__restrict__ r2g,
                                   Rec<T> *__restrict__ rec, unsigned *__restrict__ mismatch)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const SlabRecord<T> r = in[p];
    const int g = ghost_lookup(hkey, hval, mask, r.uid);
    r2g[p] = g;
    if (g < 0) {
        atomicAdd(mismatch, 1u);
        return;
    }
    Rec<T> v;
    v.x = r.v[0];
    v.y = r.v[1];
    v.z = r.v[2];
    v.d = r.v[3];
    rec[g] = v;
}

template <typename T>
__global__ void slab_refresh_apply(int count, const SlabRecord<T> *__restrict__ in, const int *__restrict__ r2g,
                                   const uint64_t *__restrict__ uid, Rec<T> *__restrict__ rec,
                                   unsigned *__restrict__ mismatch)
{
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const SlabRecord<T> r = in[p];
    const int g = r2g[p];
    if (g < 0 || uid[g] != r.uid) {
        atomicAdd(mismatch, 1u);
        return;
    }
    Rec<T> v;
    v.x = r.v[0];
    v.y = r.v[1];
    v.z = r.v[2];
    v.d = r.v[3];
    rec[g] = v;
}

}  // namespace cg
