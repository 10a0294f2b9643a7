// sweep_proxy.cuh -- the production 27-box sweep (v6).
//
// Same results as sweep.cuh (reference kernels.py:148-277 + engine.py:323-327).
// Layout it relies on (built by grid.cuh every step):
//   * agents in box-sorted slot order (off[rank] .. off[rank+1] per box; boxes
//     in row-major order, members of a box by (z, uid) -- so every 3-box
//     z-run of a stencil row is one contiguous, z-sorted slot range);
//   * prox[slot] = float4(x - x_box_lo, y - y_box_lo, z - z_origin, radius):
//     a 16-byte fp32 proxy of the agent, box-local in x/y (precision ulp(L)),
//     grid-relative in z (monotone, so z-runs stay sorted).
// Per agent (one thread):
//   phase 1 walk the 9 stencil rows; skip rows out of reach in x/y; in each
//           z-run skip/stop on z; test 4 proxies per iteration (LDG.128, L1)
//           with a conservative fp32 bound (reach + margin >= every possible
//           reference-kept distance); survivors go to a per-thread list
//           (stencil summation: walk order, flushed into phase 2 when full;
//           uid summation: the kScap smallest uids, further rounds if needed);
//   phase 2 for each listed pair: the exact f64 predicate of kernels.py:198-203
//           and, if kept, the pair force of kernels.py:230-257, summed in list
//           order -- the reference's uid order, or a fixed stencil order.
// m (stencil candidates) is the sum of the 27 box counts minus one.
#pragma once

#include "common.cuh"
#include "sweep.cuh"

namespace cg {

struct ProxyArgs {
    const float4 *prox;    // slot order
    float margin;          // absolute fp32 prefilter margin (host-computed)
};

constexpr int kCounterSlots = 512;

// slot-order proxy of every agent (after the grid build, and after the
// storage re-sort when there is one)
template <typename T, bool SORTED>
__global__ void make_proxy(int n, Geometry g, const int *__restrict__ idx,
                           const int *__restrict__ slot_key, const int *__restrict__ flat_of,
                           const T *__restrict__ x, const T *__restrict__ y, const T *__restrict__ z,
                           const T *__restrict__ d, float4 *__restrict__ prox)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n) return;
    const int a = SORTED ? s : __ldg(idx + s);
    const int k = __ldg(slot_key + s);
    const int flat = flat_of ? __ldg(flat_of + k) : k;
    const int iy = (flat / g.dimz) % g.dimy, ix = flat / (g.dimz * g.dimy);
    float4 p;
    p.x = (float)((double)x[a] - (g.ox + (double)ix * g.L));
    p.y = (float)((double)y[a] - (g.oy + (double)iy * g.L));
    p.z = (float)((double)z[a] - g.oz);
    p.w = (float)(d[a] * T(0.5));
    prox[s] = p;
}

template <typename T, bool SORTED, int SUM, bool ROWMAJOR, int KSCAP>
__global__ void __launch_bounds__(kThreads) sweep_proxy_kernel(SweepArgs<T> A, ProxyArgs P)
{
    constexpr bool UIDMODE = SUM == SUM_UID;
    extern __shared__ int list_sm[];                 // [KSCAP][kThreads], dynamic
    __shared__ unsigned long long red[3][kThreads / 32];
    int *mylist = list_sm + threadIdx.x;
#define LST(k) mylist[(k) * kThreads]

    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c_m = 0, c_nk = 0, c_deg = 0;
    if (s < A.n) {
        const T half = T(0.5);
        const T zero = A.p.zero;
        const int a = SORTED ? s : __ldg(A.idx + s);
        const int key = __ldg(A.slot_key + s);
        const int flat = A.flat_of ? __ldg(A.flat_of + key) : key;
        const int iz = flat % A.g.dimz, rest = flat / A.g.dimz;
        const int iy = rest % A.g.dimy, ix = rest / A.g.dimy;
        const float4 me = __ldg(P.prox + s);
        const T xi = A.x[a], yi = A.y[a], zi = A.z[a];
        const T ri = A.d[a] * half;
        const uint64_t ui = A.uid[a];
        const float Lf = (float)A.g.L;
        const float reach = me.w + 0.5f * Lf + P.margin;
        const float reach2 = reach * reach;
        const float zlo = me.z - reach, zhi = me.z + reach;
        const int z0 = max(iz - 1, 0), z1 = min(iz + 1, A.g.dimz - 1);

        // scan slots [t, t1) of one z-run (row-major) or one box (Morton)
        auto scan = [&](int t, const int t1, const float mx, const float my, auto &&visit) {
            if (ROWMAJOR) {
                if (t1 - t > 24) {
                    int lo = t, hi = t1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (__ldg(&P.prox[mid].z) < zlo) lo = mid + 1; else hi = mid;
                    }
                    t = lo;
                } else {
                    while (t < t1 && __ldg(&P.prox[t].z) < zlo) ++t;
                }
            }
            for (; t < t1; t += 4) {
                float4 o[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] = __ldg(P.prox + (t + k < t1 ? t + k : t));
                bool pass[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float ddx = mx - o[k].x, ddy = my - o[k].y, ddz = me.z - o[k].z;
                    const float d2 = __fmaf_rn(ddx, ddx, __fmaf_rn(ddy, ddy, ddz * ddz));
                    pass[k] = (t + k < t1) && d2 <= reach2 && (t + k != s);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (pass[k]) visit(t + k);
                if (ROWMAJOR && o[3].z > zhi) break;   // o[3]: last in range, or a copy of o[0]
            }
        };
        // phase-1 walk; returns m
        auto walk = [&](auto &&visit) -> int {
            int mm = -1;
            for (int ox = -1; ox <= 1; ++ox) {
                const int nx = ix + ox;
                if (nx < 0 || nx >= A.g.dimx) continue;
                // x distance to the neighbour row (box-local frame: own box is [0, L))
                const float gx = ox == 0 ? 0.f : fmaxf(0.f, ox < 0 ? me.x : Lf - me.x);
                const float mx = me.x - (float)ox * Lf;
                for (int oy = -1; oy <= 1; ++oy) {
                    const int ny = iy + oy;
                    if (ny < 0 || ny >= A.g.dimy) continue;
                    const float gy = oy == 0 ? 0.f : fmaxf(0.f, oy < 0 ? me.y : Lf - me.y);
                    const float my = me.y - (float)oy * Lf;
                    const int base = (nx * A.g.dimy + ny) * A.g.dimz;
                    const bool reachable = gx * gx + gy * gy <= reach2;
                    if (ROWMAJOR) {
                        const int t0 = __ldg(A.off + base + z0), t1 = __ldg(A.off + base + z1 + 1);
                        mm += t1 - t0;
                        if (reachable) scan(t0, t1, mx, my, visit);
                    } else {
                        for (int zz = z0; zz <= z1; ++zz) {
                            const int kb = __ldg(A.rank_of + base + zz);
                            const int t0 = __ldg(A.off + kb), t1 = __ldg(A.off + kb + 1);
                            mm += t1 - t0;
                            if (reachable) scan(t0, t1, mx, my, visit);
                        }
                    }
                }
            }
            return mm;
        };

        T fx = zero, fy = zero, fz = zero;
        int nk = 0, nd = 0, m = 0;
        // phase 2 for list entries [0, cnt): exact predicate + force, in order
        auto evaluate = [&](int cnt) {
            for (int p = 0; p < cnt; ++p) {
                const int t = LST(p);
                const int j = SORTED ? t : __ldg(A.idx + t);
                const T dx = xi - A.x[j], dy = yi - A.y[j], dz = zi - A.z[j];   // kernels.py:198-203
                const T dist = tsqrt<T>(dx * dx + dy * dy + dz * dz);
                const T rj = A.d[j] * half;
                const T rsum = ri + rj;
                const T delta = rsum - dist;
                if (!(delta > zero)) continue;
                ++nk;                                                            // kernels.py:230-257
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
            }
        };
        auto cand_uid = [&](int t) -> uint64_t { return A.uid[SORTED ? t : __ldg(A.idx + t)]; };

        if (!UIDMODE) {
            // survivors in walk order; a full list is evaluated and reused
            int ns = 0;
            m = walk([&](int t) {
                LST(ns) = t;
                if (++ns == KSCAP) {
                    evaluate(ns);
                    ns = 0;
                }
            });
            evaluate(ns);
        } else {
            // rounds of the KSCAP smallest uids above floor_uid, ascending
            int surv_total = 0, done = 0;
            uint64_t floor_uid = 0;
            bool first = true;
            do {
                int ns = 0;
                const int mm = walk([&](int t) {
                    if (first) ++surv_total;
                    const uint64_t ut = cand_uid(t);
                    if (!first && ut <= floor_uid) return;
                    int p;
                    if (ns < KSCAP) p = ns++;
                    else if (ut < cand_uid(LST(KSCAP - 1))) p = KSCAP - 1;
                    else return;
                    while (p > 0 && cand_uid(LST(p - 1)) > ut) {
                        LST(p) = LST(p - 1);
                        --p;
                    }
                    LST(p) = t;
                });
                if (first) m = mm;
                evaluate(ns);
                done += ns;
                if (ns) floor_uid = cand_uid(LST(ns - 1));
                first = false;
            } while (done < surv_total);
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
        if (A.new_x) {                 // engine.py:325-327 (separate buffer: two-phase)
            A.new_x[a] = xi + ddx;
            A.new_y[a] = yi + ddy;
            A.new_z[a] = zi + ddz;
        }
        if (A.rec_m) {
            A.rec_m[a] = m;
            A.rec_nk[a] = nk;
        }
        c_m = m;
        c_nk = nk;
        c_deg = nd;
    }
#undef LST
    c_m = warp_sum(c_m);
    c_nk = warp_sum(c_nk);
    c_deg = warp_sum(c_deg);
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
        atomicAdd(A.block_counters + (blockIdx.x % kCounterSlots) * 3 + threadIdx.x, t);
    }
}

}  // namespace cg
