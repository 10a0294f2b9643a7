// query.cuh -- uniform-radius neighbour queries on the device grid (SURVEY.md
// 8f row 2): reference kernels.grid_neighbor_counts / grid_neighbor_fill
// (kernels.py:427-520) behind spatial.neighbor_counts / neighbor_csr
// (spatial.py:138-169).
//
// Predicate exactly as the reference's: widened to f64,
// dx = f64(p_j) - f64(p_i) (per axis), d2 = (dx*dx + dy*dy) + dz*dz (no FMA:
// -fmad=false), kept iff d2 <= radius*radius -- a closed ball, NOT the force
// phase's (ri + rj) - dist > 0.  Candidates: the other agents of the clamped
// 27-box stencil.  Rows of the CSR table ascend by neighbour uid
// (kernels.py:471-480); indices are reference storage positions.
#pragma once

#include "common.cuh"
#include "grid.cuh"

namespace cg {

template <typename T>
struct QueryArgs {
    int n;
    Geometry g;
    BoxDecode bd;
    const int *skey;      // slot -> flat box
    const int *idx;       // slot -> storage (nullptr = identity)
    const int *off;       // flat -> first slot
    const Rec<T> *rec;    // storage order
    const uint64_t *uid;
    const int *pres;      // storage -> reference position (nullptr = identity)
    double r2;
    long long *counts;          // per reference position (count pass)
    const long long *indptr;    // per reference position (fill pass)
    long long *indices;         // reference positions of the neighbours
};

template <typename T, bool FILL>
__global__ void __launch_bounds__(kThreads) neighbor_kernel(QueryArgs<T> Q)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= Q.n) return;
    const int i = Q.idx ? __ldg(Q.idx + s) : s;
    int ix, iy, iz;
    decode_box(Q.bd, __ldg(Q.skey + s), ix, iy, iz);
    const Rec<T> me = Q.rec[i];
    const double qx = (double)me.x, qy = (double)me.y, qz = (double)me.z;
    const int ri = Q.pres ? Q.pres[i] : i;
    long long w = FILL ? Q.indptr[ri] : 0;
    long long c = 0;
    const int x0 = max(ix - 1, 0), x1 = min(ix + 1, Q.g.dimx - 1);
    const int y0 = max(iy - 1, 0), y1 = min(iy + 1, Q.g.dimy - 1);
    const int z0 = max(iz - 1, 0), z1 = min(iz + 1, Q.g.dimz - 1);
    for (int ax = x0; ax <= x1; ++ax)
        for (int ay = y0; ay <= y1; ++ay) {
            const int base = (ax * Q.g.dimy + ay) * Q.g.dimz;
            const int t0 = __ldg(Q.off + base + z0), t1 = __ldg(Q.off + base + z1 + 1);
            for (int t = t0; t < t1; ++t) {
                const int j = Q.idx ? __ldg(Q.idx + t) : t;
                if (j == i) continue;
                const Rec<T> o = Q.rec[j];
                const double dx = (double)o.x - qx, dy = (double)o.y - qy, dz = (double)o.z - qz;
                if (dx * dx + dy * dy + dz * dz <= Q.r2) {
                    if (FILL) {
                        Q.indices[w++] = Q.pres ? Q.pres[j] : j;   // sorted by uid afterwards
                    } else {
                        ++c;
                    }
                }
            }
        }
    if (!FILL) Q.counts[ri] = c;
}

// rows in reference numbering sorted by the uid of the neighbour; the uid of a
// reference position comes from the inverse map (ref -> storage)
__global__ void sort_rows_by_uid(int n, const long long *__restrict__ indptr, long long *__restrict__ indices,
                                 const int *__restrict__ ref2st, const uint64_t *__restrict__ uid)
{
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const long long lo = indptr[r], hi = indptr[r + 1];
    for (long long a = lo + 1; a < hi; ++a) {
        const long long v = indices[a];
        const uint64_t kv = uid[ref2st ? ref2st[v] : v];
        long long b = a - 1;
        while (b >= lo && uid[ref2st ? ref2st[indices[b]] : indices[b]] > kv) {
            indices[b + 1] = indices[b];
            --b;
        }
        indices[b + 1] = v;
    }
}

}  // namespace cg
