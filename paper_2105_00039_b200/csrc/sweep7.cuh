// sweep7.cuh -- the production 27-box sweep (north-star kernel (b)).
//
// Same results as the reference force phase (kernels.py:148-277) plus apply
// (engine.py:323-327) and the next step's bounding box (pool.py:102-110):
//   * one thread per slot (agents in box-sorted slot order: row-major boxes,
//     members of a box by (z, uid), so every 3-box z-run of a stencil column
//     is one contiguous, z-sorted slot range);
//   * phase 1 walks the 9 stencil columns; columns whose x/y distance exceeds
//     the reach are skipped, each column's run is cut once the z-sorted
//     proxies pass z + reach, and candidates are tested two at a time with
//     packed fp32 arithmetic (FADD2/FMUL2/FFMA2 on pair-interleaved proxies,
//     grid.cuh) against a conservative bound (reach = r_i + max radius +
//     margin >= every distance the exact test can keep);
//   * survivors go to a per-thread list in shared memory; phase 2 evaluates
//     the exact predicate (kernels.py:198-203) and, if kept, the pair force
//     (kernels.py:230-257) in the pool dtype with the reference's expression
//     order (no FMA: the library is built with -fmad=false), summing in walk
//     order (SUM_STENCIL) or ascending uid (SUM_UID, bit-identical to the
//     reference); the next survivor's record is loaded while the current pair
//     is evaluated;
//   * the pair constant req = (ri*rj)/(ri+rj) is reused while rj repeats
//     (uniform pools: one division per agent instead of one per pair);
//   * epilogue: adherence gate + cap (kernels.py:266-277), displacement and
//     new position written in storage order; counters (one REDUX + atomic per
//     warp) and the exact bbox of the new positions (ordered-u64 atomics, only
//     from agents within max_displacement of the old bbox faces -- no other
//     agent can be extreme) go into the per-step reduction slots (grid.cuh).
// m (stencil candidates) is the sum of the 27 clamped box counts minus one,
// exactly what _gather_stencil enumerates.
#pragma once

#include <type_traits>

#include "common.cuh"
#include "grid.cuh"
#include "sweep.cuh"

namespace cg {

template <typename T>
struct Sweep7Args {
    int n;
    Geometry g;
    BoxDecode bd;
    Proxies prox;            // slot order, pair-interleaved
    const int *skey;         // slot -> flat box
    const int *idx;          // slot -> storage index, nullptr = identity (relaid out)
    const int *off;          // flat box -> first slot (nb + 1 entries)
    const Rec<T> *rec;       // x, y, z, diameter (storage order)
    const T *adh;
    const uint64_t *uid;
    Params<T> p;
    float rmax;              // largest radius of the pool (rounded up)
    float margin;            // absolute prefilter margin
    T *disp_x, *disp_y, *disp_z;
    Rec<T> *new_rec;            // nullptr when frozen
    int *rec_m, *rec_nk;        // storage order, nullptr unless recording
    unsigned long long *slots;  // per-step reduction slots
    double shell_lo[3], shell_hi[3];   // bbox shell: old lo + max move, old hi - max move
    int *ovf;                   // slots of agents deferred to the overflow kernel
    unsigned *ovf_count;
    int n_owned;                // targets: [own_lo, own_lo + n_owned); the rest are slab ghosts (candidates)
    bool uid32;                 // every uid < 2^32: survivor sort keys come from the proxies
    int own_lo;                 // targets are storage indices [own_lo, own_lo + n_owned): a relaid
                                // slab sub-grid keeps its lo ghosts in front of the owned agents
    // neighbour lists (LIST builds): partners within ri + rj + skin, uid order
    int *nbr;                   // [list_cap][nbr_stride] storage indices
    int *nbr_n;                 // per storage index
    long long nbr_stride;
    T skin;
    float skin_f;               // skin rounded up, for the prefilter reach
    int list_cap;               // list entries per agent (more: the list set is not used)
    // dense uid-mode agents with more survivors than the warp's shared-memory
    // queue: a second warp pass with per-warp queues in global memory
    int *big_q;                 // [warps][big_cap]
    uint64_t *big_u;            // [warps][big_cap]
    void *big_f;                // [warps][big_cap][3] pool dtype
    int big_cap;                // power of two
    int *ovf2;                  // agents beyond big_cap: the thread-per-agent rounds
    unsigned *ovf2_count;
    // UNI (every diameter equal, fp64): the pair constants in the kernel's
    // expression order -- rsum = ri + ri, req = (ri * ri) / rsum, lim = rsum + skin
    T u_rsum, u_req, u_lim;
    // LIST: the two sub-lists (partners within ri + rj + sub1_d / sub2_d,
    // sub2_d < sub1_d < skin, list order) written with the list, so the list
    // steps after a build sweep the short sub-list at once; nullptr: not written
    int *sub1, *sub1_n, *sub2, *sub2_n;
    T sub1_d, sub2_d, u_sub1, u_sub2;   // u_*: UNI, rsum + sub*_d
};

constexpr int kListCap = 48;    // list width of sparse pools (dense pools: sized from the density)

// slot -> storage index: the idx map, or the slot itself (relaid storage)
template <typename A_t>
__device__ __forceinline__ int storage_of(const A_t &A, int s)
{
    return A.idx ? __ldg(A.idx + s) : s;
}

// packed fp32x2 helpers (sm_100a FADD2 / FMUL2 / FFMA2)
typedef unsigned long long f32x2;
__device__ __forceinline__ f32x2 f2_splat(float a)
{
    f32x2 r;
    asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(a));
    return r;
}
__device__ __forceinline__ f32x2 f2_sub(f32x2 a, f32x2 b)
{
    f32x2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 f2_mul(f32x2 a, f32x2 b)
{
    f32x2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f32x2 f2_fma(f32x2 a, f32x2 b, f32x2 c)
{
    f32x2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ void f2_unpack(f32x2 v, float &lo, float &hi)
{
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}

// UIDMODE: sum each agent's pairs in ascending uid (lists sorted per lane);
// ZSORTED: members of a box are z-sorted (dense path), so a column run can be
// cut at z + reach; FLUSH: evaluate the list whenever it fills (stencil order).
// DEFER: an agent with more than KS survivors is handed to the overflow
// kernel (slot appended to A.ovf) instead of taking further walks here.
// LIST: also record every partner within ri + rj + skin (uid order) in the
// agent's neighbour list; the walk then covers the 5x5x5 box stencil (a
// partner within ri + rmax + skin <= 2L can sit two boxes away), while m still
// counts the reference's 27 boxes.
// UNI: a uniform pool; rj, rsum, req and the list limit are kernel constants.
// NT: threads per CTA (the per-thread survivor lists are [KS][NT] in shared memory).
// PACKED (uid order, every uid < 2^32): one 64-bit entry per survivor,
// uid32 << 32 | slot -- one load, compare and store per insertion-sort move
// (C2 sweep 0.826 -> 0.761 ms, C4 list build 3.27 -> 3.23 ms).
template <typename T, bool UIDMODE, bool ZSORTED, int KS, bool FLUSH, bool DEFER, bool LIST = false,
          bool KEY32 = false, bool UNI = false, int NT = kThreads>
__device__ __forceinline__ void sweep_agent(const Sweep7Args<T> &A, const int s, unsigned &c_m,
                                            unsigned &c_nk, unsigned &c_nd, float &dmax2)
{
    constexpr bool PACKED = KEY32 && UIDMODE;
    __shared__ int lst[PACKED ? 1 : KS][PACKED ? 1 : NT];
    __shared__ uint64_t ukey[(UIDMODE && !PACKED) ? KS : 1][(UIDMODE && !PACKED) ? NT : 1];
    __shared__ uint64_t pk[PACKED ? KS : 1][PACKED ? NT : 1];
    static_assert(!(UIDMODE && FLUSH), "uid order needs the whole list");
#define LST(k) lst[k][threadIdx.x]
#define UKEY(k) ukey[k][threadIdx.x]
#define PK(k) pk[k][threadIdx.x]
#define SLOT(k) (PACKED ? (int)(unsigned)PK(k) : LST(k))
    {
        const int key = __ldg(A.skey + s);
        int ix, iy, iz;
        decode_box(A.bd, key, ix, iy, iz);
        const int a = storage_of(A, s);
        if ((unsigned)(a - A.own_lo) >= (unsigned)A.n_owned) return;   // a ghost: candidate only
        const T half = T(0.5), zero = A.p.zero;
        const float *myp = A.prox.p + 8 * (s >> 1) + (s & 1);
        const float mex = __ldg(myp), mey = __ldg(myp + 2), mez = __ldg(myp + 4);
        const float Lf = (float)A.g.L;
        const Rec<T> me = A.rec[a];
        const float reach = (float)(me.d * half) + A.rmax + A.margin + (LIST ? A.skin_f : 0.f);
        const float reach2 = reach * reach;
        const float zhi = mez + reach;
        const f32x2 mz2 = f2_splat(mez);
        constexpr int R = LIST ? 2 : 1;
        const int z0m = max(iz - 1, 0), z1m = min(iz + 1, A.g.dimz - 1);
        int z0 = z0m, z1 = z1m;
        if (LIST) {   // the boxes two away in z only when the reach crosses the box face
            const float zl = mez - (float)iz * Lf;
            if (zl < reach - Lf) z0 = max(iz - 2, 0);
            if (Lf - zl < reach - Lf) z1 = min(iz + 2, A.g.dimz - 1);
        }
        // slot pair q = ta / 2 lives in 16-byte words 2q (x pair, y pair) and 2q + 1 (z pair)
        const ulonglong2 *PR = reinterpret_cast<const ulonglong2 *>(A.prox.p);

        // phase-1 walk over the 9 stencil columns; visit(t) per survivor, in
        // slot order (the agent itself included: phase 2 skips it); after()
        // runs once per batch that produced survivors
        auto walk = [&](auto &&visit, auto &&after) -> int {
            int mm = -1;
#pragma unroll 1
            for (int ox = -R; ox <= R; ++ox) {
                const int nx = ix + ox;
                if ((unsigned)nx >= (unsigned)A.g.dimx) continue;
                const float gx = ox == 0 ? 0.f
                                         : fmaxf(0.f, (ox < 0 ? mex : Lf - mex) + (float)(abs(ox) - 1) * Lf);
                if (LIST && (ox == -2 || ox == 2) && gx * gx > reach2) continue;   // plane out of reach
                const f32x2 mx2 = f2_splat(mex - (float)ox * Lf);
#pragma unroll 1
                for (int oy = -R; oy <= R; ++oy) {
                    const int ny = iy + oy;
                    if ((unsigned)ny >= (unsigned)A.g.dimy) continue;
                    if (LIST && (ox == -2 || ox == 2 || oy == -2 || oy == 2)) {
                        // outer ring: no part of m, skipped unless within reach
                        const float gy2 = fmaxf(0.f, (oy < 0 ? mey : Lf - mey) + (float)(abs(oy) - 1) * Lf);
                        const float gyy = oy == 0 ? 0.f : gy2;
                        if (gx * gx + gyy * gyy > reach2) continue;
                    }
                    const int base = (nx * A.g.dimy + ny) * A.g.dimz;
                    const int t0 = __ldg(A.off + base + z0), t1 = __ldg(A.off + base + z1 + 1);
                    if (!LIST) {
                        mm += t1 - t0;
                    } else if (abs(ox) <= 1 && abs(oy) <= 1) {
                        // the walked run is wider than the 3-box column only near a z face
                        const int m1 = z1 == z1m ? t1 : __ldg(A.off + base + z1m + 1);
                        const int m0 = z0 == z0m ? t0 : __ldg(A.off + base + z0m);
                        mm += m1 - m0;
                    }
                    const float gy = oy == 0 ? 0.f
                                             : fmaxf(0.f, (oy < 0 ? mey : Lf - mey) + (float)(abs(oy) - 1) * Lf);
                    if (gx * gx + gy * gy > reach2) continue;
                    const f32x2 my2 = f2_splat(mey - (float)oy * Lf);
                    // two slot pairs per iteration (both loads in flight); the proxy
                    // array is padded past n, masks drop slots outside [t0, t1)
                    for (int ta = t0 & ~1; ta < t1; ta += 4) {
                        const ulonglong2 xa = __ldg(PR + ta), za = __ldg(PR + ta + 1);
                        const ulonglong2 xb = __ldg(PR + ta + 2), zb = __ldg(PR + ta + 3);
                        f32x2 d, ea, eb;
                        d = f2_sub(mz2, za.x);
                        ea = f2_mul(d, d);
                        d = f2_sub(mz2, zb.x);
                        eb = f2_mul(d, d);
                        d = f2_sub(my2, xa.y);
                        ea = f2_fma(d, d, ea);
                        d = f2_sub(my2, xb.y);
                        eb = f2_fma(d, d, eb);
                        d = f2_sub(mx2, xa.x);
                        ea = f2_fma(d, d, ea);
                        d = f2_sub(mx2, xb.x);
                        eb = f2_fma(d, d, eb);
                        float a0, a1, b0, b1;
                        f2_unpack(ea, a0, a1);
                        f2_unpack(eb, b0, b1);
                        // common case (~85 %): no candidate of the four is in reach --
                        // one compare; slot bounds only matter inside the branch
                        if (fminf(fminf(a0, a1), fminf(b0, b1)) <= reach2) {
                            const bool p0 = a0 <= reach2 && ta >= t0;
                            const bool p1 = a1 <= reach2 && ta + 1 < t1;
                            const bool p2 = b0 <= reach2 && ta + 2 < t1;
                            const bool p3 = b1 <= reach2 && ta + 3 < t1;
                            if (p0) visit(ta, (unsigned)za.y);
                            if (p1) visit(ta + 1, (unsigned)(za.y >> 32));
                            if (p2) visit(ta + 2, (unsigned)zb.y);
                            if (p3) visit(ta + 3, (unsigned)(zb.y >> 32));
                            after();
                        }
                        if (ZSORTED) {
                            float zl, zh;
                            f2_unpack(zb.x, zl, zh);
                            if (zh > zhi) break;   // z-sorted run (past t1 only ends the loop sooner)
                        }
                    }
                }
            }
            return mm;
        };

        const T xi = me.x, yi = me.y, zi = me.z;
        const T ri = me.d * half;
        T fx = zero, fy = zero, fz = zero;
        int nk = 0, nd = 0, nl = 0, n1 = 0, n2 = 0;
        T last_rj = T(-1), last_req = zero;
        // NOCALL (the main kernel when an overflow kernel follows): call-free
        // sqrt / division (common.cuh); an operand outside their fast range,
        // or coincident centres, hands the agent to the overflow kernel,
        // which uses the library routines
        constexpr bool NOCALL = DEFER && !FLUSH;
        bool ok = true;
        auto xsqrt = [&](T v) -> T { return NOCALL ? tsqrt_nocall(v, ok) : tsqrt<T>(v); };
        auto xdiv = [&](T a_, T b_) -> T { return NOCALL ? tdiv_nocall(a_, b_, ok) : a_ / b_; };
        // phase 2 for list entries [0, cnt), in list order; the next entry's
        // record is in flight while the current pair is evaluated
        auto evaluate = [&](int cnt_) {
            int p = 0;
            if (p < cnt_ && SLOT(p) == s) ++p;
            if (p >= cnt_) return;
            int j = storage_of(A, SLOT(p));
            Rec<T> o = A.rec[j];
#pragma unroll 1
            while (p < cnt_) {
                const int jc = j;
                const Rec<T> co = o;
                ++p;
                if (p < cnt_ && SLOT(p) == s) ++p;   // the agent itself
                if (p < cnt_) {
                    j = storage_of(A, SLOT(p));
                    o = A.rec[j];
                }
                const T dx = xi - co.x, dy = yi - co.y, dz = zi - co.z;   // kernels.py:198-203
                const T rj = UNI ? zero : co.d * half;
                T rs = zero;   // NOCALL: dist's rsqrt estimate seeds the division by dist
                const T dist = NOCALL ? tsqrt_nocall_r(dx * dx + dy * dy + dz * dz, ok, rs)
                                      : tsqrt<T>(dx * dx + dy * dy + dz * dz);
                const T rsum = UNI ? A.u_rsum : ri + rj;
                if (LIST && dist <= (UNI ? A.u_lim : rsum + A.skin)) {
                    if (nl < A.list_cap) {
                        A.nbr[nl * A.nbr_stride + a] = jc;
                        if (A.sub1 && dist <= (UNI ? A.u_sub1 : rsum + A.sub1_d)) {
                            A.sub1[n1 * A.nbr_stride + a] = jc;
                            ++n1;
                            if (dist <= (UNI ? A.u_sub2 : rsum + A.sub2_d)) {
                                A.sub2[n2 * A.nbr_stride + a] = jc;
                                ++n2;
                            }
                        }
                    }
                    ++nl;
                }
                const T delta = rsum - dist;
                if (!(delta > zero)) continue;
                ++nk;                                                    // kernels.py:230-257
                if (UNI) {
                    last_req = A.u_req;
                } else if (rj != last_rj) {
                    last_rj = rj;
                    last_req = xdiv(ri * rj, rsum);
                }
                const T mag = A.p.kappa * delta - A.p.gamma * xsqrt(last_req * delta);
                if (NOCALL || dist > zero) {   // NOCALL: dist == 0 fails the division's range test
                    const T sc = NOCALL ? tdiv_seeded(mag, dist, rs, ok) : mag / dist;
                    fx = fx + sc * dx;
                    fy = fy + sc * dy;
                    fz = fz + sc * dz;
                } else {
                    ++nd;
                    const uint64_t ui = A.uid[a], uj = A.uid[jc];
                    double ux, uy, uz;
                    degenerate_dir(ui < uj ? ui : uj, ui < uj ? uj : ui, ux, uy, uz);
                    const double sign = ui < uj ? 1.0 : -1.0;
                    fx = fx + (T)((double)mag * (sign * ux));
                    fy = fy + (T)((double)mag * (sign * uy));
                    fz = fz + (T)((double)mag * (sign * uz));
                }
            }
        };

        int m;
        if (!UIDMODE && FLUSH) {
            // dense neighbourhoods: the list is evaluated whenever it fills up
            int ns = 0;
            m = walk([&](int t, unsigned) { LST(ns++) = t; },
                     [&]() {
                         if (ns > KS - 4) {   // a batch appends up to 4
                             evaluate(ns);
                             ns = 0;
                         }
                     });
            evaluate(ns);
        } else if (!UIDMODE) {
            // collect the first KS survivors, evaluate; on overflow walk again,
            // collecting the next KS (walk order is deterministic)
            int ns = 0, total = 0;
            m = walk(
                [&](int t, unsigned) {
                    if (ns < KS) LST(ns++) = t;
                    ++total;
                },
                [] {});
            if (DEFER && total > KS) {
                A.ovf[atomicAdd(A.ovf_count, 1u)] = s;
                return;
            }
            evaluate(ns);
            for (int done = KS; done < total; done += KS) {
                int seen = 0;
                ns = 0;
                walk(
                    [&](int t, unsigned) {
                        if (seen >= done && ns < KS) LST(ns++) = t;
                        ++seen;
                    },
                    [] {});
                evaluate(ns);
            }
        } else {
            auto cand_uid = [&](int t) -> uint64_t { return A.uid[storage_of(A, t)]; };
            // first walk: keep the first KS survivors, count all of them (the
            // agent itself is not one: nothing to sort or skip later)
            int ns = 0, total = 0;
            m = walk(
                [&](int t, unsigned u) {
                    if (t == s) return;
                    if (ns < KS) {
                        if constexpr (PACKED) {
                            PK(ns) = ((uint64_t)u << 32) | (unsigned)t;
                        } else {
                            LST(ns) = t;
                            UKEY(ns) = A.uid32 ? (uint64_t)u : cand_uid(t);
                        }
                        ++ns;
                    }
                    ++total;
                },
                [] {});
            if (DEFER && total > KS) {
                A.ovf[atomicAdd(A.ovf_count, 1u)] = s;
                return;
            }
            if (total <= KS) {
                // insertion sort by uid, then one evaluation in uid order (measured
                // against a one-ahead pipelined compare and a binary search + 4-way
                // unrolled shift: within +-3 %, profiles/r2/ab_r2k.jsonl)
                for (int p = 1; p < ns; ++p) {
                    if constexpr (PACKED) {
                        const uint64_t v = PK(p);
                        int q = p;
                        while (q > 0 && PK(q - 1) > v) {
                            PK(q) = PK(q - 1);
                            --q;
                        }
                        PK(q) = v;
                    } else {
                        const uint64_t u = UKEY(p);
                        const int v = LST(p);
                        int q = p;
                        while (q > 0 && UKEY(q - 1) > u) {
                            UKEY(q) = UKEY(q - 1);
                            LST(q) = LST(q - 1);
                            --q;
                        }
                        UKEY(q) = u;
                        LST(q) = v;
                    }
                }
                evaluate(ns);
            } else {
                // dense neighbourhood: rounds of the KS smallest uids above floor_uid
                int done = 0;
                uint64_t floor_uid = 0;
                bool first = true;
                while (done < total) {
                    int nr = 0;
                    walk(
                        [&](int t, unsigned u) {
                            if (t == s) return;
                            if constexpr (PACKED) {   // keys packed with the slot: same order as by uid
                                const uint64_t v = ((uint64_t)u << 32) | (unsigned)t;
                                if (!first && v <= floor_uid) return;
                                int q;
                                if (nr < KS) q = nr++;
                                else if (v < PK(KS - 1)) q = KS - 1;
                                else return;
                                while (q > 0 && PK(q - 1) > v) {
                                    PK(q) = PK(q - 1);
                                    --q;
                                }
                                PK(q) = v;
                            } else {
                                const uint64_t ut = (KEY32 || A.uid32) ? (uint64_t)u : cand_uid(t);
                                if (!first && ut <= floor_uid) return;
                                int q;
                                if (nr < KS) q = nr++;
                                else if (ut < UKEY(KS - 1)) q = KS - 1;
                                else return;
                                while (q > 0 && UKEY(q - 1) > ut) {
                                    UKEY(q) = UKEY(q - 1);
                                    LST(q) = LST(q - 1);
                                    --q;
                                }
                                UKEY(q) = ut;
                                LST(q) = t;
                            }
                        },
                        [] {});
                    evaluate(nr);
                    done += nr;
                    if (nr) floor_uid = PACKED ? PK(nr - 1) : UKEY(nr - 1);
                    first = false;
                }
            }
        }

        if (NOCALL && !ok) {   // redone by the overflow kernel (library sqrt / division)
            A.ovf[atomicAdd(A.ovf_count, 1u)] = s;
            return;
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
        if (LIST) {
            A.nbr_n[a] = nl;
            if (A.sub1) {
                A.sub1_n[a] = n1;
                A.sub2_n[a] = n2;
            }
            if (nl > A.list_cap) atomicAdd(A.slots + (blockIdx.x % kSlots) * kSlotWords + 10, 1ull);
        }
        if (LIST || ZSORTED)   // the step's largest displacement (list validity / build decision)
            dmax2 = fmaxf(dmax2, (float)((double)ddx * ddx + (double)ddy * ddy + (double)ddz * ddz));
        if (A.new_rec) {               // engine.py:325-327 (separate buffer: two-phase)
            const T nxp = xi + ddx, nyp = yi + ddy, nzp = zi + ddz;
            Rec<T> nr;
            nr.x = nxp;
            nr.y = nyp;
            nr.z = nzp;
            nr.d = me.d;
            A.new_rec[a] = nr;
            // next step's bbox: only agents inside the boundary shell can be extreme
            // (the extreme agent moved by at most max_displacement)
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
#undef LST
#undef UKEY
#undef PK
#undef SLOT
}

// counters: one REDUX per warp, one atomic per warp and counter
__device__ __forceinline__ void warp_counters(unsigned long long *slots, unsigned c_m, unsigned c_nk,
                                              unsigned c_nd)
{
    c_m = __reduce_add_sync(0xffffffffu, c_m);
    c_nk = __reduce_add_sync(0xffffffffu, c_nk);
    c_nd = __reduce_add_sync(0xffffffffu, c_nd);
    if ((threadIdx.x & 31) == 0) {
        unsigned long long *slot = slots + (blockIdx.x % kSlots) * kSlotWords;
        if (c_nk) atomicAdd(slot + 6, (unsigned long long)c_nk);
        if (c_m) atomicAdd(slot + 7, (unsigned long long)c_m);
        if (c_nd) atomicAdd(slot + 8, (unsigned long long)c_nd);
    }
}

// the largest squared displacement of the step (neighbour-list validity),
// one atomic per warp into the block's slot
__device__ __forceinline__ void warp_dmax(unsigned long long *slots, float dmax2)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dmax2 = fmaxf(dmax2, __shfl_xor_sync(0xffffffffu, dmax2, o));
    if ((threadIdx.x & 31) == 0 && dmax2 > 0.f)
        atomicMax(slots + (blockIdx.x % kSlots) * kSlotWords + 9, enc_ordered((double)dmax2));
}

template <typename T, bool UIDMODE, bool ZSORTED, int KS, bool FLUSH, int MINB, bool LIST = false, bool KEY32 = false,
          bool UNI = false, int NT = kThreads>
__global__ void __launch_bounds__(NT, MINB) sweep7_kernel(Sweep7Args<T> A)
{
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned c_m = 0, c_nk = 0, c_nd = 0;
    float dmax2 = 0.f;
    if (s < A.n) sweep_agent<T, UIDMODE, ZSORTED, KS, FLUSH, true, LIST, KEY32, UNI, NT>(A, s, c_m, c_nk, c_nd, dmax2);
    warp_counters(A.slots, c_m, c_nk, c_nd);
    if (LIST || ZSORTED) warp_dmax(A.slots, dmax2);
}

// agents deferred by sweep7_kernel (more than KS survivors): grid-stride over
// the device-side list, further walks per agent
template <typename T, bool UIDMODE, bool ZSORTED, int KS, bool LIST = false, bool KEY32 = false>
__global__ void __launch_bounds__(kThreads) sweep7_overflow(Sweep7Args<T> A)
{
    unsigned c_m = 0, c_nk = 0, c_nd = 0;
    float dmax2 = 0.f;
    const unsigned cnt = *A.ovf_count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt; k += gridDim.x * blockDim.x)
        sweep_agent<T, UIDMODE, ZSORTED, KS, false, false, LIST, KEY32>(A, A.ovf[k], c_m, c_nk, c_nd, dmax2);
    warp_counters(A.slots, c_m, c_nk, c_nd);
    if (LIST || ZSORTED) warp_dmax(A.slots, dmax2);
}

}  // namespace cg
