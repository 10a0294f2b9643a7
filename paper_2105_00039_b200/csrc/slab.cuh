// slab.cuh -- x-slab decomposition kernels (multi-GPU).
//
// Every rank derives the same global geometry from an all-reduced bbox; rank r
// owns the agents whose global box plane ix lies in [X0(r), X1(r)),
// X_k = floor(k * dimx / world).  Per step (driven by distributed.py):
//   slab_dest          owner rank of every owned agent under the new geometry
//   slab_list_*        departures / holes / tail movers (compaction lists)
//   slab_pack          departing agents -> send buffer, grouped by destination
//   slab_fill_holes    tail agents that stay move into the holes departures left
//   slab_unpack        received records appended (arrivals, or this step's ghosts)
//   slab_halo_list     owned agents in planes X0 (-> rank r-1) and X1-1 (-> r+1)
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

template <typename T>
__global__ void slab_dest(int n, Geometry g, SlabBounds B, const Rec<T> *__restrict__ rec,
                          unsigned char *__restrict__ dest, unsigned long long *__restrict__ counts)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ix = axis_box((double)rec[i].x, g.ox, g.L, g.gdimx);
    const int r = slab_owner(B, ix);
    dest[i] = (unsigned char)r;
    const unsigned peers = __match_any_sync(__activemask(), r);
    if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(counts + r, (unsigned long long)__popc(peers));
}

// departures (dest != rank) -> dep; holes = departures below n_keep; movers =
// staying agents at or above n_keep (|holes| == |movers|)
__global__ void slab_lists(int n, int n_keep, int rank, const unsigned char *__restrict__ dest,
                           int *__restrict__ dep, int *__restrict__ holes, int *__restrict__ movers,
                           unsigned *__restrict__ cnt /* dep, holes, movers */)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const bool leaving = dest[i] != rank;
    if (leaving) dep[atomicAdd(cnt + 0, 1u)] = i;
    if (leaving && i < n_keep) holes[atomicAdd(cnt + 1, 1u)] = i;
    if (!leaving && i >= n_keep) movers[atomicAdd(cnt + 2, 1u)] = i;
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

// departing agents into the send buffer at dest_off[dest] + running cursor
template <typename T>
__global__ void slab_pack(int ndep, const int *__restrict__ dep, const unsigned char *__restrict__ dest,
                          const unsigned long long *__restrict__ dest_off, unsigned *__restrict__ cursor,
                          SlabCols<T> C, SlabRecord<T> *__restrict__ out)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= ndep) return;
    const int i = dep[k];
    const int r = dest[i];
    SlabRecord<T> rec;
    load_record(C, i, rec);
    out[dest_off[r] + atomicAdd(cursor + r, 1u)] = rec;
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

// same, with the hole count read on the device
template <typename T>
__global__ void slab_fill_holes_dev(const unsigned *__restrict__ nmove, const int *__restrict__ holes,
                                    const int *__restrict__ movers, SlabCols<T> C)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= (int)*nmove) return;
    SlabRecord<T> rec;
    load_record(C, movers[k], rec);
    store_record(C, holes[k], rec);
}

template <typename T>
__global__ void slab_unpack(int count, int base, const SlabRecord<T> *__restrict__ in, SlabCols<T> C,
                            unsigned long long *__restrict__ maxd_enc)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    const SlabRecord<T> rec = in[k];
    store_record(C, base + k, rec);
    if (maxd_enc) atomicMax(maxd_enc, enc_ordered((double)rec.v[3]));
}

// owned agents in the boundary planes: ix == lo_plane -> list 0, ix == hi_plane -> list 1
template <typename T>
__global__ void slab_halo_list(int n, Geometry g, int lo_plane, int hi_plane, const Rec<T> *__restrict__ rec,
                               int *__restrict__ lo_list, int *__restrict__ hi_list, unsigned *__restrict__ cnt)
{
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int ix = axis_box((double)rec[i].x, g.ox, g.L, g.gdimx);
    if (ix == lo_plane) lo_list[atomicAdd(cnt + 0, 1u)] = i;
    if (ix == hi_plane) hi_list[atomicAdd(cnt + 1, 1u)] = i;
}

template <typename T>
__global__ void slab_gather_records(int count, const int *__restrict__ list, SlabCols<T> C,
                                    SlabRecord<T> *__restrict__ out)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= count) return;
    SlabRecord<T> rec;
    load_record(C, list[k], rec);
    out[k] = rec;
}

}  // namespace cg
