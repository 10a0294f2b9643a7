// sweep_tile.cuh -- tiled 27-box sweep: one CTA per 3-D block of boxes.
//
// Same results as sweep.cuh (reference kernels.py:148-277 + engine.py:323-327),
// organised for the B200:
//   stage   the tile's TX x TY x TZ boxes plus a one-box halo are copied into
//           shared memory, one warp per contiguous segment (a row of boxes in
//           row-major order, a box in Morton order): per agent a float4
//           (x, y, z relative to the tile centre, radius) and its storage index;
//   phase 1 one lane per core agent walks its 9 stencil rows (each a run of <= 3
//           boxes).  Rows beyond reach in x/y are skipped; in row-major order
//           each run is z-sorted, so the lane skips/stops on z; the rest gets a
//           conservative fp32 distance test (kPrefilterUlps margin).  Survivors
//           go to the lane's shared-memory list -- in walk order (stencil
//           summation) or as the SCAP smallest uids (uid summation);
//   phase 2 the lane evaluates its list in order: exact f64 predicate of
//           kernels.py:198-203 and, if kept, the pair force of
//           kernels.py:230-257 added to the running sum -- so the sum is the
//           reference's (uid order) or a fixed stencil order.  Decoupling the
//           f64 pair math from the candidate loop keeps the warp converged in
//           both loops.
// A lane with more than SCAP survivors takes further rounds.  m (stencil
// candidates) is the sum of the 27 box counts minus one.  A tile whose halo
// exceeds the staging capacity reads candidates from global memory.
#pragma once

#include "common.cuh"
#include "sweep.cuh"
#include "sweep_proxy.cuh"

namespace cg {

struct TileShape {
    int tx, ty, tz;         // core boxes per tile
    int ntx, nty, ntz;      // tiles per axis
    int cap;                // staged agents capacity
    int max_halo_boxes;
    int debug_stop;         // profiling aid: 1 = stop after staging, 2 = after phase 1
};

template <typename T>
struct TileArgs {
    SweepArgs<T> s;
    TileShape t;
};

// fp32 prefilter margin: staged coordinates are relative to the tile centre,
// |coord| <= ext.  Rounding of the stored coordinates, of the fp32
// differences and of the fp32 squared distance stays below 8 ulp(ext); 64 ulp
// is used.  The reach bound ri + rj <= ri + L/2 holds because box_length >=
// max diameter (spatial.py:101-106).
constexpr float kPrefilterUlps = 64.0f;
constexpr int kScap = 32;        // survivors listed per lane per round
constexpr int kWarps = kThreads / 32;

template <typename T>
struct TileSmem {
    int total, core, overflow;
    int core_base[kThreads + 1];
    int list[kScap][kThreads];      // [k][thread]: conflict-free per-lane lists
    unsigned long long red[3][kWarps];
};

template <typename T, bool SORTED, int SUM, bool ZSORTED>
__global__ void __launch_bounds__(kThreads, 2) sweep_tile_kernel(TileArgs<T> TA)
{
    constexpr bool UIDMODE = SUM == SUM_UID;
    const SweepArgs<T> &A = TA.s;
    const TileShape &S = TA.t;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    TileSmem<T> &F = *reinterpret_cast<TileSmem<T> *>(smem_raw);
    float4 *rec = reinterpret_cast<float4 *>(smem_raw + ((sizeof(TileSmem<T>) + 15) & ~size_t(15)));
    int *rslot = reinterpret_cast<int *>(rec + S.cap);
    int *bstart = rslot + S.cap;
    int *bcnt = bstart + S.max_halo_boxes;
    int *bbase = bcnt + S.max_halo_boxes;

    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // ---- tile geometry
    const int tile = blockIdx.x;
    const int tz = tile % S.ntz, rest = tile / S.ntz;
    const int ty = rest % S.nty, tx = rest / S.nty;
    const int cx0 = tx * S.tx, cy0 = ty * S.ty, cz0 = tz * S.tz;
    const int cx1 = min(cx0 + S.tx, A.g.dimx), cy1 = min(cy0 + S.ty, A.g.dimy),
              cz1 = min(cz0 + S.tz, A.g.dimz);
    const int hx0 = max(cx0 - 1, 0), hy0 = max(cy0 - 1, 0), hz0 = max(cz0 - 1, 0);
    const int hx1 = min(cx1 + 1, A.g.dimx), hy1 = min(cy1 + 1, A.g.dimy), hz1 = min(cz1 + 1, A.g.dimz);
    const int HX = hx1 - hx0, HY = hy1 - hy0, HZ = hz1 - hz0;
    const int nhb = HX * HY * HZ;
    const double ccx = A.g.ox + (0.5 * (cx0 + cx1)) * A.g.L;
    const double ccy = A.g.oy + (0.5 * (cy0 + cy1)) * A.g.L;
    const double ccz = A.g.oz + (0.5 * (cz0 + cz1)) * A.g.L;

    // ---- halo box table + exclusive scan of counts
    for (int hb = threadIdx.x; hb < nhb; hb += blockDim.x) {
        const int lz = hb % HZ, r2 = hb / HZ;
        const int ly = r2 % HY, lx = r2 / HY;
        const int flat = ((hx0 + lx) * A.g.dimy + (hy0 + ly)) * A.g.dimz + (hz0 + lz);
        const int k = A.rank_of ? __ldg(A.rank_of + flat) : flat;
        const int s0 = __ldg(A.off + k);
        bstart[hb] = s0;
        bcnt[hb] = __ldg(A.off + k + 1) - s0;
    }
    __syncthreads();
    if (warp == 0) {
        int carry = 0;
        for (int base = 0; base < nhb; base += 32) {
            const int i = base + lane;
            const int v = i < nhb ? bcnt[i] : 0;
            int inc = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            if (i < nhb) bbase[i] = carry + inc - v;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) {
            F.total = carry;
            F.overflow = carry > S.cap;
        }
    }
    const int lx0 = cx0 - hx0, ly0 = cy0 - hy0, lz0 = cz0 - hz0;
    const int CY = cy1 - cy0, CZ = cz1 - cz0;
    const int ncore_rows = (cx1 - cx0) * CY;
    __syncthreads();
    const int total = F.total;
    if (total == 0) return;
    const bool staged = !F.overflow;

    if (staged) {
        // one warp per contiguous segment: a halo row (row-major: the HZ boxes of
        // a row are consecutive slots) or a single box (Morton order)
        const int nseg = A.rank_of ? nhb : HX * HY;
        for (int sg = warp; sg < nseg; sg += kWarps) {
            const int hb0 = A.rank_of ? sg : sg * HZ;
            const int hb1 = A.rank_of ? sg : sg * HZ + HZ - 1;
            const int g0 = bstart[hb0], b0 = bbase[hb0];
            const int len = bbase[hb1] + bcnt[hb1] - b0;
            for (int e = lane; e < len; e += 32) {
                const int slot = g0 + e;
                const int j = SORTED ? slot : __ldg(A.idx + slot);
                float4 r;
                r.x = (float)((double)A.x[j] - ccx);
                r.y = (float)((double)A.y[j] - ccy);
                r.z = (float)((double)A.z[j] - ccz);
                r.w = (float)(A.d[j] * T(0.5));
                rec[b0 + e] = r;
                rslot[b0 + e] = j;
            }
        }
    }
    if (threadIdx.x == 0) {
        int acc = 0;
        for (int r = 0; r < ncore_rows; ++r) {
            const int hb0 = ((lx0 + r / CY) * HY + (ly0 + r % CY)) * HZ + lz0;
            const int hb1 = hb0 + CZ - 1;
            F.core_base[r] = acc;
            acc += bbase[hb1] + bcnt[hb1] - bbase[hb0];
        }
        F.core_base[ncore_rows] = acc;
        F.core = acc;
    }
    __syncthreads();
    const int ncore = F.core;
    if (S.debug_stop == 1) return;

    const T half = T(0.5);
    const T zero = A.p.zero;
    const float Lf = (float)A.g.L;
    unsigned long long c_m = 0, c_nk = 0, c_deg = 0;
    int *mylist = &F.list[0][threadIdx.x];      // element k at mylist[k * kThreads]
#define LST(k) mylist[(k) * kThreads]

    for (int c = threadIdx.x; c < ncore; c += blockDim.x) {
        const bool active = true;
        int q = -1, a = -1, blx = 0, bly = 0, blz = 0;
        T xi = zero, yi = zero, zi = zero, ri = zero;
        uint64_t ui = 0;
        float4 me = make_float4(0.f, 0.f, 0.f, 0.f);
        float reach = 0.f, reach2 = -1.0f;
        float fxlo = 0.f, fylo = 0.f;   // tile-frame coordinates of the own box's low faces
        int m = 0;
        if (active) {
            int lo = 0, hi = ncore_rows - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (F.core_base[mid] <= c) lo = mid; else hi = mid - 1;
            }
            const int r = lo;
            const int hbrow = ((lx0 + r / CY) * HY + (ly0 + r % CY)) * HZ + lz0;
            q = bbase[hbrow] + (c - F.core_base[r]);
            lo = hbrow;
            hi = hbrow + CZ - 1;
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (bbase[mid] <= q) lo = mid; else hi = mid - 1;
            }
            const int hb = lo;
            blz = hb % HZ;
            bly = (hb / HZ) % HY;
            blx = hb / (HZ * HY);
            const int slot = bstart[hb] + (q - bbase[hb]);
            a = staged ? rslot[q] : (SORTED ? slot : __ldg(A.idx + slot));
            xi = A.x[a];
            yi = A.y[a];
            zi = A.z[a];
            ri = A.d[a] * half;
            ui = A.uid[a];
            me.x = (float)((double)xi - ccx);
            me.y = (float)((double)yi - ccy);
            me.z = (float)((double)zi - ccz);
            me.w = (float)(A.d[a] * half);
            const float ext = fmaxf(fmaxf(fabsf(me.x), fabsf(me.y)), fabsf(me.z)) + 2.0f * Lf;
            reach = me.w + 0.5f * Lf + kPrefilterUlps * ext * 5.9604645e-8f;
            reach2 = reach * reach;
            fxlo = (float)(A.g.ox + (double)(hx0 + blx) * A.g.L - ccx);
            fylo = (float)(A.g.oy + (double)(hy0 + bly) * A.g.L - ccy);
        }
        auto cand_storage = [&](int e) { return staged ? rslot[e] : e; };
        auto cand_uid = [&](int e) -> uint64_t { return A.uid[cand_storage(e)]; };

        // test staged elements [t, t1) of one stencil row-run, 4 per iteration
        // (independent chains for ILP); z-sorted runs skip below zlo and stop
        // above zhi
        const float zlo = me.z - reach, zhi = me.z + reach;
        auto scan_run = [&](int t, const int t1, const float rr2, auto &&visit) {
            if (ZSORTED) {
                if (t1 - t > 16) {
                    int lo = t, hi = t1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (rec[mid].z < zlo) lo = mid + 1; else hi = mid;
                    }
                    t = lo;
                } else {
                    while (t < t1 && rec[t].z < zlo) ++t;
                }
            }
            for (; t < t1; t += 4) {
                float4 o[4];
                bool pass[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) o[k] = rec[t + k < t1 ? t + k : t];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float ddx = me.x - o[k].x, ddy = me.y - o[k].y, ddz = me.z - o[k].z;
                    const float d2 = __fmaf_rn(ddx, ddx, __fmaf_rn(ddy, ddy, ddz * ddz));
                    pass[k] = (t + k < t1) && d2 <= rr2 && (t + k != q);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (pass[k]) visit(t + k);
                if (ZSORTED && o[3].z > zhi) break;   // o[3] is the last in range or a copy of o[0]
            }
        };
        // phase-1 walk: visit(e) for every prefilter survivor e (staged index, or
        // storage index when the tile is not staged).  Returns m (stencil members
        // other than the agent, kernels.py:163-172).
        auto walk = [&](auto &&visit) -> int {
            int mm = -1;
            for (int ox = -1; ox <= 1; ++ox) {
                const int nx = blx + ox;
                if (nx < 0 || nx >= HX) continue;
                // distance from the agent to the neighbour row's x-slab (0 for own)
                const float gx = ox == 0 ? 0.f : fmaxf(0.f, ox < 0 ? me.x - fxlo : fxlo + Lf - me.x);
                for (int oy = -1; oy <= 1; ++oy) {
                    const int ny = bly + oy;
                    if (ny < 0 || ny >= HY) continue;
                    const float gy = oy == 0 ? 0.f : fmaxf(0.f, oy < 0 ? me.y - fylo : fylo + Lf - me.y);
                    const int rowb = (nx * HY + ny) * HZ;
                    const int z0 = max(blz - 1, 0), z1 = min(blz + 1, HZ - 1);
                    const int t0 = bbase[rowb + z0];
                    const int t1 = bbase[rowb + z1] + bcnt[rowb + z1];
                    mm += t1 - t0;
                    // rows out of reach in x/y are skipped (the margin in reach2
                    // absorbs the fp32 rounding of the face coordinates)
                    const float rz2 = reach2 - gx * gx - gy * gy;
                    if (rz2 < 0.f) continue;
                    if (staged) {
                        scan_run(t0, t1, reach2, visit);
                    } else {
                        for (int zz = z0; zz <= z1; ++zz) {
                            const int b = rowb + zz;
                            for (int t = 0; t < bcnt[b]; ++t) {
                                const int slot = bstart[b] + t;
                                const int j = SORTED ? slot : __ldg(A.idx + slot);
                                if (j == a) continue;
                                const float ddx = me.x - (float)((double)A.x[j] - ccx);
                                const float ddy = me.y - (float)((double)A.y[j] - ccy);
                                const float ddz = me.z - (float)((double)A.z[j] - ccz);
                                const float d2 = __fmaf_rn(ddx, ddx, __fmaf_rn(ddy, ddy, ddz * ddz));
                                if (d2 <= reach2) visit(j);
                            }
                        }
                    }
                }
            }
            return mm;
        };

        T fx = zero, fy = zero, fz = zero;
        int nk = 0, nd = 0;
        int surv_total = 0, done = 0;
        uint64_t floor_uid = 0;
        bool first = true;
        bool finished = !active;
        while (!finished) {
            // ---- phase 1: this round's list
            int ns = 0;
            if (UIDMODE) {
                // the kScap smallest uids above floor_uid, ascending
                const int mm = walk([&](int e) {
                    if (first) ++surv_total;
                    const uint64_t ue = cand_uid(e);
                    if (!first && ue <= floor_uid) return;
                    int p;
                    if (ns < kScap) p = ns++;
                    else if (ue < cand_uid(LST(kScap - 1))) p = kScap - 1;
                    else return;
                    while (p > 0 && cand_uid(LST(p - 1)) > ue) {
                        LST(p) = LST(p - 1);
                        --p;
                    }
                    LST(p) = e;
                });
                if (first) m = mm;
            } else {
                // survivors [done, done + kScap) in walk order
                int seen = 0;
                const int mm = walk([&](int e) {
                    if (seen >= done && ns < kScap) LST(ns++) = e;
                    ++seen;
                });
                if (first) {
                    surv_total = seen;
                    m = mm;
                }
            }
            // ---- phase 2: exact predicate + pair force, accumulated in list order
            for (int p = 0; p < (S.debug_stop == 2 ? 0 : ns); ++p) {
                const int j = cand_storage(LST(p));
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
            done += ns;
            if (UIDMODE && ns) floor_uid = cand_uid(LST(ns - 1));
            first = false;
            finished = done >= surv_total;
        }

        if (active) {
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
            if (A.new_x) {
                A.new_x[a] = xi + ddx;
                A.new_y[a] = yi + ddy;
                A.new_z[a] = zi + ddz;
            }
            if (A.rec_m) {
                A.rec_m[a] = m;
                A.rec_nk[a] = nk;
            }
            c_m += m;
            c_nk += nk;
            c_deg += nd;
        }
    }
#undef LST
    c_m = warp_sum(c_m);
    c_nk = warp_sum(c_nk);
    c_deg = warp_sum(c_deg);
    if (lane == 0) {
        F.red[0][warp] = c_nk;
        F.red[1][warp] = c_m;
        F.red[2][warp] = c_deg;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long t = 0;
        for (int p = 0; p < kWarps; ++p) t += F.red[threadIdx.x][p];
        atomicAdd(A.block_counters + (blockIdx.x % kCounterSlots) * 3 + threadIdx.x, t);
    }
}

template <typename T>
inline size_t tile_smem_bytes(const TileShape &S)
{
    size_t b = (sizeof(TileSmem<T>) + 15) & ~size_t(15);
    b += (size_t)S.cap * (sizeof(float4) + sizeof(int));
    b += (size_t)S.max_halo_boxes * 3 * sizeof(int);
    return b;
}

}  // namespace cg
