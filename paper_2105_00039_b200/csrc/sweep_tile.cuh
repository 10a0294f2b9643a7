// sweep_tile.cuh -- tiled 27-box sweep for sparse pools (production path at
// C4's ~2 agents per box).
//
// Same results as sweep7.cuh (reference kernels.py:148-277 + engine.py:323-327).
// One CTA per TX x TY x TZ block of boxes (the core); the core plus a one-box
// halo is staged in shared memory once, with coalesced loads of the halo's
// column runs (row-major slots: the boxes of a column are one slot range):
//   * fp32 proxies in a tile-local frame (x, y, z - tile centre; SoA, each
//     column run starting at an even index so pairs load as one LDS.64),
//   * the exact pool-dtype records (x, y, z, diameter) and the uids.
// Then one thread per core agent:
//   phase 1  walks its 9 stencil column runs in shared memory, testing two
//            candidates per packed FADD2/FFMA2 chain against the conservative
//            reach (r_i + max radius + margin);
//   phase 2  sorts its survivors by uid (the reference's summation order,
//            kernels.py:206-225) and evaluates the exact predicate and pair
//            force from the staged records;
//   epilogue as sweep7 (gate, cap, apply, counters, bbox shell).
// Agents with more than KS survivors, and every agent of a tile whose halo does
// not fit the staging capacity, are deferred to sweep7_overflow.
#pragma once

#include "common.cuh"
#include "grid.cuh"
#include "sweep7.cuh"

namespace cg {

struct TileCfg {
    int tx, ty, tz;          // core boxes per tile
    int ntx, nty, ntz;       // tiles per axis
    int cap;                 // staged agents (even)
    int max_cols;            // (tx + 2) * (ty + 2)
    float margin;            // prefilter margin for the tile-local frame
};

// dynamic shared memory layout (bytes), for pool dtype T
template <typename T>
struct TileLayout {
    size_t xs, ys, zs, xe, ye, ze, de, uid, bz, boff, total;
    __host__ __device__ TileLayout(int cap, int max_cols, int tz)
    {
        size_t o = 0;
        auto take = [&](size_t bytes) {
            const size_t r = o;
            o = (o + bytes + 15) & ~size_t(15);
            return r;
        };
        xe = take(sizeof(T) * cap);
        ye = take(sizeof(T) * cap);
        ze = take(sizeof(T) * cap);
        de = take(sizeof(T) * cap);
        uid = take(sizeof(uint64_t) * cap);
        xs = take(sizeof(float) * cap);
        ys = take(sizeof(float) * cap);
        zs = take(sizeof(float) * cap);
        bz = take(sizeof(unsigned char) * cap);
        boff = take(sizeof(int) * max_cols * (tz + 3));
        total = o;
    }
};

template <typename T, int KS>
__global__ void __launch_bounds__(kThreads, 3) sweep_tile_kernel(Sweep7Args<T> A, TileCfg C)
{
    extern __shared__ __align__(16) unsigned char tsm[];
    __shared__ int col_raw0[64];          // first global slot of each halo column run
    __shared__ int col_base[64];          // first staged index of each halo column run
    __shared__ int core_pref[17];         // prefix of core targets per core column
    __shared__ int core_first[16];        // staged index of each core column's first target
    __shared__ int s_total, s_overflow;
    __shared__ float xlo[16], ylo[16];    // tile-frame lower face of each halo box column
    __shared__ unsigned short lst[KS][kThreads];

    const TileLayout<T> Lay(C.cap, C.max_cols, C.tz);
    T *xe = reinterpret_cast<T *>(tsm + Lay.xe);
    T *ye = reinterpret_cast<T *>(tsm + Lay.ye);
    T *ze = reinterpret_cast<T *>(tsm + Lay.ze);
    T *de = reinterpret_cast<T *>(tsm + Lay.de);
    uint64_t *us = reinterpret_cast<uint64_t *>(tsm + Lay.uid);
    float *xs = reinterpret_cast<float *>(tsm + Lay.xs);
    float *ys = reinterpret_cast<float *>(tsm + Lay.ys);
    float *zs = reinterpret_cast<float *>(tsm + Lay.zs);
    unsigned char *bz = tsm + Lay.bz;
    int *boff = reinterpret_cast<int *>(tsm + Lay.boff);

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // ---- tile geometry (z fastest across blocks: neighbours share halo data in L2)
    const int tile = blockIdx.x;
    const int tzi = tile % C.ntz, rest = tile / C.ntz;
    const int tyi = rest % C.nty, txi = rest / C.nty;
    const int cx0 = txi * C.tx, cy0 = tyi * C.ty, cz0 = tzi * C.tz;
    const int cx1 = min(cx0 + C.tx, A.g.dimx), cy1 = min(cy0 + C.ty, A.g.dimy), cz1 = min(cz0 + C.tz, A.g.dimz);
    const int hx0 = max(cx0 - 1, 0), hy0 = max(cy0 - 1, 0), hz0 = max(cz0 - 1, 0);
    const int hx1 = min(cx1 + 1, A.g.dimx), hy1 = min(cy1 + 1, A.g.dimy), hz1 = min(cz1 + 1, A.g.dimz);
    const int HX = hx1 - hx0, HY = hy1 - hy0, HZ = hz1 - hz0;
    const int ncols = HX * HY;
    const int BW = HZ + 1;                // box offsets per column run
    // tile centre (frame of the fp32 proxies)
    const double ccx = A.g.ox + 0.5 * (double)(cx0 + cx1 + 2 * A.g.xoff) * A.g.L;
    const double ccy = A.g.oy + 0.5 * (double)(cy0 + cy1) * A.g.L;
    const double ccz = A.g.oz + 0.5 * (double)(cz0 + cz1) * A.g.L;

    // ---- 1. global box offsets of every halo column run
    for (int q = threadIdx.x; q < ncols * BW; q += blockDim.x) {
        const int k = q / BW, zz = q - k * BW;
        const int lx = k / HY, ly = k - lx * HY;
        const int base = ((hx0 + lx) * A.g.dimy + (hy0 + ly)) * A.g.dimz + hz0;
        boff[q] = __ldg(A.off + base + zz);
    }
    if (threadIdx.x <= HX) xlo[threadIdx.x] = (float)(A.g.ox + (double)(hx0 + A.g.xoff + (int)threadIdx.x) * A.g.L - ccx);
    if (threadIdx.x >= 32 && threadIdx.x - 32 <= HY)
        ylo[threadIdx.x - 32] = (float)(A.g.oy + (double)(hy0 + (int)threadIdx.x - 32) * A.g.L - ccy);
    __syncthreads();
    // ---- 2. staged bases (each run starts at an even index) + core targets
    if (warp == 0) {
        int carry = 0;
        for (int k0 = 0; k0 < ncols; k0 += 32) {
            const int k = k0 + lane;
            int len = 0;
            if (k < ncols) {
                col_raw0[k] = boff[k * BW];
                len = (boff[k * BW + HZ] - boff[k * BW] + 1) & ~1;
            }
            int inc = len;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (k < ncols) col_base[k] = carry + inc - len;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) {
            s_total = carry;
            s_overflow = carry > C.cap;
        }
    }
    __syncthreads();
    // rebase the box offsets into staged indices
    for (int q = threadIdx.x; q < ncols * BW; q += blockDim.x) {
        const int k = q / BW;
        boff[q] = boff[q] - col_raw0[k] + col_base[k];
    }
    const int ccols = (cx1 - cx0) * (cy1 - cy0), CY = cy1 - cy0;
    const int lx0 = cx0 - hx0, ly0 = cy0 - hy0, lz0 = cz0 - hz0, lz1 = cz1 - hz0;
    __syncthreads();
    if (warp == 0) {
        int cnt = 0, first = 0;
        if (lane < ccols) {
            const int k = (lane / CY + lx0) * HY + (lane % CY + ly0);
            first = boff[k * BW + lz0];
            cnt = boff[k * BW + lz1] - first;
        }
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane < ccols) {
            core_pref[lane] = inc - cnt;
            core_first[lane] = first;
        }
        if (lane == ccols - 1) core_pref[ccols] = inc;
    }
    const bool overflow = s_overflow;
    // ---- 3. stage the halo runs (one warp per run, coalesced)
    if (!overflow) {
        for (int k = warp; k < ncols; k += kThreads / 32) {
            const int g0 = col_raw0[k], b0 = col_base[k];
            const int len = boff[k * BW + HZ] - b0;
            for (int p = lane; p < len; p += 32) {
                const int sl = g0 + p;
                const int j = A.idx ? __ldg(A.idx + sl) : sl;
                const T x = A.x[j], y = A.y[j], z = A.z[j];
                const int e = b0 + p;
                xe[e] = x;
                ye[e] = y;
                ze[e] = z;
                de[e] = A.d[j];
                us[e] = A.uid[j];
                xs[e] = (float)((double)x - ccx);
                ys[e] = (float)((double)y - ccy);
                zs[e] = (float)((double)z - ccz);
                int ix, iy, iz;
                decode_box(A.bd, __ldg(A.skey + sl), ix, iy, iz);
                bz[e] = (unsigned char)(iz - hz0);
            }
            if ((len & 1) && lane == 0) {   // pad the run to an even length: far away
                xs[b0 + len] = 3.0e37f;
                ys[b0 + len] = 3.0e37f;
                zs[b0 + len] = 3.0e37f;
            }
        }
    }
    __syncthreads();

    unsigned c_m = 0, c_nk = 0, c_nd = 0;
    const int ntargets = core_pref[ccols];
    const float Lf = (float)A.g.L;
    for (int t = threadIdx.x; t < ntargets; t += blockDim.x) {
        int cj = 0;
        while (cj + 1 < ccols && core_pref[cj + 1] <= t) ++cj;
        const int e = core_first[cj] + (t - core_pref[cj]);
        const int lx = cj / CY + lx0, ly = cj % CY + ly0;
        const int kself = lx * HY + ly;
        const int s = col_raw0[kself] + (e - col_base[kself]);   // global slot
        if (overflow) {
            A.ovf[atomicAdd(A.ovf_count, 1u)] = s;
            continue;
        }
        const int a = A.idx ? __ldg(A.idx + s) : s;
        if (a >= A.n_owned) continue;   // a ghost: candidate only
        const int lz = bz[e];
        const float mex = xs[e], mey = ys[e], mez = zs[e];
        const T half = T(0.5), zero = A.p.zero;
        const T xi = xe[e], yi = ye[e], zi = ze[e];
        const T ri = de[e] * half;
        const float reach = (float)ri + A.rmax + C.margin;
        const float reach2 = reach * reach;
        const f32x2 mx2 = f2_splat(mex), my2 = f2_splat(mey), mz2 = f2_splat(mez);
        const int bz0 = max(lz - 1, 0), bz1 = min(lz + 1, HZ - 1);

        // ---- phase 1
        int m = -1, ns = 0, total = 0;
#pragma unroll 1
        for (int ox = -1; ox <= 1; ++ox) {
            const int nx = lx + ox;
            if ((unsigned)nx >= (unsigned)HX) continue;
            const float gx = ox == 0 ? 0.f : fmaxf(0.f, ox < 0 ? mex - xlo[lx] : xlo[lx + 1] - mex);
#pragma unroll 1
            for (int oy = -1; oy <= 1; ++oy) {
                const int ny = ly + oy;
                if ((unsigned)ny >= (unsigned)HY) continue;
                const int k = nx * HY + ny;
                const int r0 = boff[k * BW + bz0], r1 = boff[k * BW + bz1 + 1];
                m += r1 - r0;
                const float gy = oy == 0 ? 0.f : fmaxf(0.f, oy < 0 ? mey - ylo[ly] : ylo[ly + 1] - mey);
                if (gx * gx + gy * gy > reach2) continue;
                for (int q = r0 & ~1; q < r1; q += 2) {
                    const f32x2 zz = *reinterpret_cast<const f32x2 *>(zs + q);
                    const f32x2 yy = *reinterpret_cast<const f32x2 *>(ys + q);
                    const f32x2 xx = *reinterpret_cast<const f32x2 *>(xs + q);
                    const f32x2 dz = f2_sub(mz2, zz);
                    f32x2 d2 = f2_mul(dz, dz);
                    const f32x2 dy = f2_sub(my2, yy);
                    d2 = f2_fma(dy, dy, d2);
                    const f32x2 dx = f2_sub(mx2, xx);
                    d2 = f2_fma(dx, dx, d2);
                    float d2a, d2b;
                    f2_unpack(d2, d2a, d2b);
                    const bool pa = d2a <= reach2 && q >= r0 && q != e;
                    const bool pb = d2b <= reach2 && q + 1 < r1 && q + 1 != e;
                    if (pa || pb) {
                        if (pa) {
                            if (ns < KS) lst[ns++][threadIdx.x] = (unsigned short)q;
                            ++total;
                        }
                        if (pb) {
                            if (ns < KS) lst[ns++][threadIdx.x] = (unsigned short)(q + 1);
                            ++total;
                        }
                    }
                }
            }
        }
        if (total > KS) {
            A.ovf[atomicAdd(A.ovf_count, 1u)] = s;
            continue;
        }
        // ---- phase 2: survivors in ascending uid (insertion sort), exact math
        for (int p = 1; p < ns; ++p) {
            const unsigned short v = lst[p][threadIdx.x];
            const uint64_t u = us[v];
            int q = p;
            while (q > 0 && us[lst[q - 1][threadIdx.x]] > u) {
                lst[q][threadIdx.x] = lst[q - 1][threadIdx.x];
                --q;
            }
            lst[q][threadIdx.x] = v;
        }
        T fx = zero, fy = zero, fz = zero;
        int nk = 0, nd = 0;
        T last_rj = T(-1), last_req = zero;
#pragma unroll 1
        for (int p = 0; p < ns; ++p) {
            const int j = lst[p][threadIdx.x];
            const T dx = xi - xe[j], dy = yi - ye[j], dz = zi - ze[j];   // kernels.py:198-203
            const T rj = de[j] * half;
            const T dist = tsqrt<T>(dx * dx + dy * dy + dz * dz);
            const T rsum = ri + rj;
            const T delta = rsum - dist;
            if (!(delta > zero)) continue;
            ++nk;                                                    // kernels.py:230-257
            if (rj != last_rj) {
                last_rj = rj;
                last_req = (ri * rj) / rsum;
            }
            const T mag = A.p.kappa * delta - A.p.gamma * tsqrt<T>(last_req * delta);
            if (dist > zero) {
                const T sc = mag / dist;
                fx = fx + sc * dx;
                fy = fy + sc * dy;
                fz = fz + sc * dz;
            } else {
                ++nd;
                const uint64_t ui = us[e], uj = us[j];
                double ux, uy, uz;
                degenerate_dir(ui < uj ? ui : uj, ui < uj ? uj : ui, ux, uy, uz);
                const double sign = ui < uj ? 1.0 : -1.0;
                fx = fx + (T)((double)mag * (sign * ux));
                fy = fy + (T)((double)mag * (sign * uy));
                fz = fz + (T)((double)mag * (sign * uz));
            }
        }
        // ---- epilogue: kernels.py:266-277, engine.py:325-327
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
        if (A.new_x) {
            const T nxp = xi + ddx, nyp = yi + ddy, nzp = zi + ddz;
            A.new_x[a] = nxp;
            A.new_y[a] = nyp;
            A.new_z[a] = nzp;
            const double p3[3] = {(double)nxp, (double)nyp, (double)nzp};
            unsigned long long *slot = A.slots + (blockIdx.x % kSlots) * kSlotWords;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (p3[q] <= A.shell_lo[q]) atomicMin(slot + q, enc_ordered(p3[q]));
                if (p3[q] >= A.shell_hi[q]) atomicMax(slot + 3 + q, enc_ordered(p3[q]));
            }
        }
        if (A.rec_m) {
            A.rec_m[a] = m;
            A.rec_nk[a] = nk;
        }
        c_m += (unsigned)m;
        c_nk += (unsigned)nk;
        c_nd += (unsigned)nd;
    }
    warp_counters(A.slots, c_m, c_nk, c_nd);
}

}  // namespace cg
