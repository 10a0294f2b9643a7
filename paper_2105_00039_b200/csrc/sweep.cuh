// sweep.cuh -- 27-box sphere-sphere force sweep, adherence gate, capped
// displacement and apply (north-star kernel (b)).
//
// Restates reference kernels.py:148-277 (_gather_stencil, _sum_forces_sorted,
// _write_displacement) and engine.py:323-327 (apply) per agent:
//   * candidates = every other agent in the clamped 3x3x3 box stencil, boxes
//     visited in ascending (ax, ay, az) (kernels.py:163-172); m counts them;
//   * pass 1 keeps candidates with (ri + rj) - sqrt(dx*dx + dy*dy + dz*dz) > 0
//     evaluated in the pool dtype, no FMA (kernels.py:196-205); nk counts them;
//   * SUM_UID: kept pairs are accumulated in ascending uid order
//     (kernels.py:206-257), so displacements are bit-identical to the
//     reference.  A per-thread sorted buffer of KCAP kept pairs is filled per
//     round; a dense neighbourhood (nk > KCAP) takes ceil(nk / KCAP) rounds.
//   * SUM_STENCIL: kept pairs accumulated in stencil order (boxes ascending,
//     members of a box by uid) -- deterministic, within ~1e-15 of the reference.
//
// Grid layout: agents sit in box-sorted CSR order.  `off[k]`..
// `off[k+1]` are the slots of the box with visiting rank k; `slot_key[s]` is the
// rank of slot s's box; `rank_of` maps flat box -> rank (NULL = identity) and
// `flat_of` the inverse.  SORTED: slot == storage index (storage was re-sorted
// this step); otherwise `idx[slot]` gives the storage index.
#pragma once

#include "common.cuh"

namespace cg {

enum { SUM_UID = 0, SUM_STENCIL = 1 };

template <typename T>
struct SweepArgs {
    int n;
    Geometry g;
    const Rec<T> *rec;
    const T *adh;
    const uint64_t *uid;
    const int *idx;        // slot -> storage (unsorted mode)
    const int *slot_key;   // slot -> box rank
    const int *off;        // rank -> first slot (nb + 1 entries)
    const int *rank_of;    // flat -> rank, NULL if identity
    const int *flat_of;    // rank -> flat, NULL if identity
    Params<T> p;
    T *disp_x, *disp_y, *disp_z;
    Rec<T> *new_rec;            // NULL when frozen
    int *rec_m, *rec_nk;        // per storage index, NULL unless recording
    unsigned long long *block_counters;  // 3 per block
};

template <typename T>
__device__ __forceinline__ T tsqrt(T v);
template <>
__device__ __forceinline__ double tsqrt<double>(double v) { return sqrt(v); }
template <>
__device__ __forceinline__ float tsqrt<float>(float v) { return sqrtf(v); }

template <typename T, bool SORTED, int SUM, int KCAP>
__global__ void __launch_bounds__(kThreads) sweep_kernel(SweepArgs<T> A)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c_m = 0, c_nk = 0, c_deg = 0;
    if (s < A.n) {
        const int a = SORTED ? s : __ldg(A.idx + s);
        const int key = __ldg(A.slot_key + s);
        const int flat = A.flat_of ? __ldg(A.flat_of + key) : key;
        const int iz = flat % A.g.dimz, rest = flat / A.g.dimz;
        const int iy = rest % A.g.dimy, ix = rest / A.g.dimy;
        const int x0 = max(ix - 1, 0), x1 = min(ix + 1, A.g.dimx - 1);
        const int y0 = max(iy - 1, 0), y1 = min(iy + 1, A.g.dimy - 1);
        const int z0 = max(iz - 1, 0), z1 = min(iz + 1, A.g.dimz - 1);

        const T half = T(0.5);
        const Rec<T> me = A.rec[a];
        const T xi = me.x, yi = me.y, zi = me.z;
        const T ri = me.d * half;
        const uint64_t ui = A.uid[a];
        const T zero = A.p.zero;

        // pair predicate, kernels.py:198-203 (exact expression order)
        auto collides = [&](int j, T &dx, T &dy, T &dz, T &dist, T &rj) -> bool {
            const Rec<T> o = A.rec[j];
            dx = xi - o.x;
            dy = yi - o.y;
            dz = zi - o.z;
            dist = tsqrt<T>(dx * dx + dy * dy + dz * dz);
            rj = o.d * half;
            const T delta = (ri + rj) - dist;
            return delta > zero;
        };

        T fx = zero, fy = zero, fz = zero;
        int nd = 0;
        // force of one kept pair, kernels.py:230-257
        auto accumulate = [&](int j, T dx, T dy, T dz, T dist, T rj) {
            const T rsum = ri + rj;
            const T delta = rsum - dist;
            const T req = (ri * rj) / rsum;
            const T mag = A.p.kappa * delta - A.p.gamma * tsqrt<T>(req * delta);
            if (dist > zero) {
                const T sc = mag / dist;
                fx = fx + sc * dx;
                fy = fy + sc * dy;
                fz = fz + sc * dz;
            } else {
                ++nd;
                const uint64_t uj = A.uid[j];
                double ux, uy, uz;
                degenerate_dir(ui < uj ? ui : uj, ui < uj ? uj : ui, ux, uy, uz);
                const double sign = ui < uj ? 1.0 : -1.0;
                fx = fx + (T)((double)mag * (sign * ux));
                fy = fy + (T)((double)mag * (sign * uy));
                fz = fz + (T)((double)mag * (sign * uz));
            }
        };

        // stencil walk in reference order; visit(j) for every candidate j != a
        auto walk = [&](auto &&visit) {
            for (int ax = x0; ax <= x1; ++ax)
                for (int ay = y0; ay <= y1; ++ay) {
                    const int base = (ax * A.g.dimy + ay) * A.g.dimz;
                    for (int az = z0; az <= z1; ++az) {
                        const int fb = base + az;
                        const int kb = A.rank_of ? __ldg(A.rank_of + fb) : fb;
                        const int t1 = __ldg(A.off + kb + 1);
                        for (int t = __ldg(A.off + kb); t < t1; ++t) {
                            const int j = SORTED ? t : __ldg(A.idx + t);
                            if (j != a) visit(j);
                        }
                    }
                }
        };

        int m = 0, nk = 0;
        if (SUM == SUM_STENCIL) {
            walk([&](int j) {
                ++m;
                T dx, dy, dz, dist, rj;
                if (collides(j, dx, dy, dz, dist, rj)) {
                    ++nk;
                    accumulate(j, dx, dy, dz, dist, rj);
                }
            });
        } else {
            // uid-ordered accumulation in rounds of at most KCAP kept pairs
            uint64_t bu[KCAP];
            int bj[KCAP];
            uint64_t floor_uid = 0;
            bool first = true;
            int done = 0;
            do {
                int bn = 0;
                walk([&](int j) {
                    T dx, dy, dz, dist, rj;
                    if (first) ++m;
                    if (!collides(j, dx, dy, dz, dist, rj)) return;
                    if (first) ++nk;
                    const uint64_t uj = A.uid[j];
                    if (!first && uj <= floor_uid) return;
                    int q;
                    if (bn < KCAP) {
                        q = bn++;
                    } else if (uj < bu[KCAP - 1]) {
                        q = KCAP - 1;
                    } else {
                        return;
                    }
                    while (q > 0 && bu[q - 1] > uj) {
                        bu[q] = bu[q - 1];
                        bj[q] = bj[q - 1];
                        --q;
                    }
                    bu[q] = uj;
                    bj[q] = j;
                });
                for (int q = 0; q < bn; ++q) {
                    T dx, dy, dz, dist, rj;
                    collides(bj[q], dx, dy, dz, dist, rj);
                    accumulate(bj[q], dx, dy, dz, dist, rj);
                }
                done += bn;
                if (bn) floor_uid = bu[bn - 1];
                first = false;
            } while (done < nk);
        }

        // _write_displacement, kernels.py:266-277
        const T norm = tsqrt<T>(fx * fx + fy * fy + fz * fz);
        T ddx = zero, ddy = zero, ddz = zero;
        if (!(norm <= A.p.adh_scale * A.adh[a])) {
            T sc = A.p.timestep;
            if (norm * sc > A.p.max_disp) sc = A.p.max_disp / norm;
            ddx = fx * sc;
            ddy = fy * sc;
            ddz = fz * sc;
        }
        A.disp_x[a] = ddx;
        A.disp_y[a] = ddy;
        A.disp_z[a] = ddz;
        if (A.new_rec) {             // engine.py:325-327 (two-phase: separate buffer)
            Rec<T> nr;
            nr.x = xi + ddx;
            nr.y = yi + ddy;
            nr.z = zi + ddz;
            nr.d = me.d;
            A.new_rec[a] = nr;
        }
        if (A.rec_m) {
            A.rec_m[a] = m;
            A.rec_nk[a] = nk;
        }
        c_m = m;
        c_nk = nk;
        c_deg = nd;
    }
    // counters: warp -> block -> one slot per block (no same-address atomics)
    c_m = warp_sum(c_m);
    c_nk = warp_sum(c_nk);
    c_deg = warp_sum(c_deg);
    __shared__ unsigned long long red[3][kThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][w] = c_nk;
        red[1][w] = c_m;
        red[2][w] = c_deg;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long t = 0;
        for (int q = 0; q < kThreads / 32; ++q) t += red[threadIdx.x][q];
        A.block_counters[blockIdx.x * 3 + threadIdx.x] = t;
    }
}

// Sum the per-block counters into stat[2..4] (evals, cands, ndeg).
__global__ void reduce_counters(int nblocks, const unsigned long long *__restrict__ bc,
                                unsigned long long *__restrict__ stat)
{
    unsigned long long v[3] = {0, 0, 0};
    for (int b = threadIdx.x; b < nblocks; b += blockDim.x)
        for (int k = 0; k < 3; ++k) v[k] += bc[b * 3 + k];
    __shared__ unsigned long long red[3][kThreads / 32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k = 0; k < 3; ++k) {
        const unsigned long long t = warp_sum(v[k]);
        if (lane == 0) red[k][w] = t;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long t = 0;
        for (int q = 0; q < kThreads / 32; ++q) t += red[threadIdx.x][q];
        stat[2 + threadIdx.x] = t;
    }
}

}  // namespace cg
