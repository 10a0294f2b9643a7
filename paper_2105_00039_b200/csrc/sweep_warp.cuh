// sweep_warp.cuh -- warp-cooperative sweep for dense neighbourhoods.
//
// Same results as the reference force phase (kernels.py:148-277) + apply
// (engine.py:323-327).  When an agent has hundreds of stencil candidates
// (C2 / C3 at 27-100 neighbours: 170-600 candidates, 27-100 kept pairs),
// one thread per agent diverges badly; here one WARP takes one agent:
//   * lanes 0-8 fetch the 9 stencil column runs in one round; the runs are
//     flattened into one candidate index space that the warp walks 32
//     candidates at a time (independent proxy loads across columns);
//   * the fp32 prefilter survivors are ballot-compacted, in walk order, into
//     the warp's shared-memory queue;
//   * lanes evaluate the queued pairs in parallel (exact f64 predicate and
//     force, kernels.py:198-257, no FMA);
//   * stencil mode: lane partial sums in queue order, then a fixed butterfly
//     -- deterministic;  uid mode: the queue is bitonic-sorted by uid, the
//     pair forces are stored in that order and lane 0 adds them one by one --
//     the reference's summation, bit for bit;
//   * lane 0 runs the epilogue (gate, cap, apply, bbox shell, record).
// LIST (uid mode only): the list-building sweep of dense pools -- the reach
// grows by the skin, the walk covers the 5x5 columns (and z +-2) where the
// reach crosses a box face, and the uid-sorted queue is written out as the
// agent's neighbour list (partners within r_i + r_j + skin), ballot-compacted.
#pragma once

#include "common.cuh"
#include "grid.cuh"
#include "sweep7.cuh"

namespace cg {

#ifndef CG_WARP_MINB
#define CG_WARP_MINB 4       // stencil-mode blocks per SM (uid mode: 3, shared-memory bound)
#endif
constexpr int kWarpQ = 256;   // survivors queued per warp before a flush (stencil mode)

template <typename T, bool UIDMODE>
struct WarpSmem {
    int q[kThreads / 32][kWarpQ];
    uint64_t u[UIDMODE ? kThreads / 32 : 1][UIDMODE ? kWarpQ : 1];
    T f[UIDMODE ? kThreads / 32 : 1][UIDMODE ? kWarpQ : 1][3];
};

template <typename T>
__device__ __forceinline__ T warp_tree_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// exact pair force of kernels.py:198-257; returns false if the pair is not kept
template <typename T>
__device__ __forceinline__ bool pair_force(const Sweep7Args<T> &A, const Rec<T> &me, uint64_t ui, int j,
                                           T &fx, T &fy, T &fz, int &deg)
{
    const T half = T(0.5), zero = A.p.zero;
    const Rec<T> o = A.rec[j];
    const T dx = me.x - o.x, dy = me.y - o.y, dz = me.z - o.z;
    const T ri = me.d * half, rj = o.d * half;
    const T dist = tsqrt<T>(dx * dx + dy * dy + dz * dz);
    const T rsum = ri + rj;
    const T delta = rsum - dist;
    if (!(delta > zero)) return false;
    const T req = (ri * rj) / rsum;
    const T mag = A.p.kappa * delta - A.p.gamma * tsqrt<T>(req * delta);
    deg = 0;
    if (dist > zero) {
        const T sc = mag / dist;
        fx = sc * dx;
        fy = sc * dy;
        fz = sc * dz;
    } else {
        deg = 1;
        const uint64_t uj = A.uid[j];
        double ux, uy, uz;
        degenerate_dir(ui < uj ? ui : uj, ui < uj ? uj : ui, ux, uy, uz);
        const double sign = ui < uj ? 1.0 : -1.0;
        fx = (T)((double)mag * (sign * ux));
        fy = (T)((double)mag * (sign * uy));
        fz = (T)((double)mag * (sign * uz));
    }
    return true;
}

// pair_force plus list membership (superset test of dist <= rsum + skin)
template <typename T>
__device__ __forceinline__ bool pair_force_l(const Sweep7Args<T> &A, const Rec<T> &me, uint64_t ui, int j,
                                             T &fx, T &fy, T &fz, int &deg, bool &inl)
{
    const T half = T(0.5), zero = A.p.zero;
    const Rec<T> o = A.rec[j];
    const T dx = me.x - o.x, dy = me.y - o.y, dz = me.z - o.z;
    const T ri = me.d * half, rj = o.d * half;
    const T s2 = dx * dx + dy * dy + dz * dz;
    const T rsum = ri + rj;
    const T rs = rsum + A.skin;
    inl = s2 <= rs * rs * T(1.00001);
    deg = 0;
    if (s2 > rsum * rsum * T(1.0000000000009095)) return false;   // fl(sqrt(s2)) > rsum
    const T dist = tsqrt<T>(s2);
    const T delta = rsum - dist;
    if (!(delta > zero)) return false;
    const T req = (ri * rj) / rsum;
    const T mag = A.p.kappa * delta - A.p.gamma * tsqrt<T>(req * delta);
    if (dist > zero) {
        const T sc = mag / dist;
        fx = sc * dx;
        fy = sc * dy;
        fz = sc * dz;
    } else {
        deg = 1;
        const uint64_t uj = A.uid[j];
        double ux, uy, uz;
        degenerate_dir(ui < uj ? ui : uj, ui < uj ? uj : ui, ux, uy, uz);
        const double sign = ui < uj ? 1.0 : -1.0;
        fx = (T)((double)mag * (sign * ux));
        fy = (T)((double)mag * (sign * uy));
        fz = (T)((double)mag * (sign * uz));
    }
    return true;
}

// register bitonic sort of the warp's queue Q[0, qn) (qn <= 32 E) by packed
// (uid32 << 32 | slot) keys, uid32 from the slots' proxies; lane l holds
// elements [l E, l E + E); Q is rewritten in ascending uid order
template <int E>
__device__ __forceinline__ void sort_queue_packed(int *Q, int qn, int lane, const float *prox)
{
    constexpr int N = 32 * E;
    uint64_t a[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        a[e] = ~0ull;
        if (i < qn) {
            const int t = Q[i];
            a[e] = ((uint64_t)__float_as_uint(__ldg(prox + 8 * (t >> 1) + 6 + (t & 1))) << 32) | (unsigned)t;
        }
    }
#pragma unroll
    for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            if (jj >= E) {   // partner in lane ^ (jj / E), same register
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int i = lane * E + e;
                    const uint64_t o = __shfl_xor_sync(0xffffffffu, a[e], jj / E);
                    const bool lower = (i & jj) == 0, up = (i & k) == 0;
                    a[e] = (lower == up) ? (a[e] < o ? a[e] : o) : (a[e] < o ? o : a[e]);
                }
            } else {         // partner in the same lane
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const int f = e ^ jj;
                    if (f > e) {
                        const bool up = ((lane * E + e) & k) == 0;
                        const uint64_t x = a[e], y = a[f];
                        const bool sw = (x > y) == up;
                        a[e] = sw ? y : x;
                        a[f] = sw ? x : y;
                    }
                }
            }
        }
    }
    __syncwarp();
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        if (i < qn) Q[i] = (int)(unsigned)a[e];
    }
    __syncwarp();
}

// BIG: the second pass over the agents the first pass spilled (A.ovf): the
// same walk, sort and uid-order sum with the warp's queue in global memory
// (A.big_*, big_cap entries); agents beyond that go to A.ovf2.
template <typename T, bool UIDMODE, bool LIST = false, bool BIG = false>
__global__ void __launch_bounds__(kThreads, UIDMODE ? 3 : CG_WARP_MINB) sweep_warp_kernel(Sweep7Args<T> A)   // uid mode: 3 blocks by shared memory anyway
{
    static_assert(UIDMODE || !LIST, "lists are built in uid order");
    static_assert(UIDMODE || !BIG, "the global queue is for uid order");
    constexpr int R = LIST ? 2 : 1, W = 2 * R + 1, NC = W * W;
    extern __shared__ __align__(16) unsigned char wsm[];
    WarpSmem<T, UIDMODE> &S = *reinterpret_cast<WarpSmem<T, UIDMODE> *>(wsm);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int gw = blockIdx.x * (kThreads / 32) + wid;
    const int QC = BIG ? A.big_cap : kWarpQ;
    int *Q = BIG ? A.big_q + (size_t)gw * A.big_cap : S.q[wid];
    const unsigned lt = (1u << lane) - 1u;
    unsigned c_m = 0, c_nk = 0, c_nd = 0;
    float dmax2 = 0.f;
    const float Lf = (float)A.g.L;
    const T zero = A.p.zero;
    const int nunits = BIG ? (int)*A.ovf_count : A.n;
    for (int w = gw; w < nunits; w += gridDim.x * (kThreads / 32)) {
        const int s = BIG ? A.ovf[w] : w;
        const int a = storage_of(A, s);
        if ((unsigned)(a - A.own_lo) >= (unsigned)A.n_owned) continue;   // a ghost (uniform across the warp)
        int ix, iy, iz;
        decode_box(A.bd, __ldg(A.skey + s), ix, iy, iz);
        const float *myp = A.prox.p + 8 * (s >> 1) + (s & 1);
        const float mex = __ldg(myp), mey = __ldg(myp + 2), mez = __ldg(myp + 4);
        const Rec<T> me = A.rec[a];
        const uint64_t ui = A.uid[a];
        const float reach = (float)(me.d * T(0.5)) + A.rmax + A.margin + (LIST ? A.skin_f : 0.f);
        const float reach2 = reach * reach;
        const int z0m = max(iz - 1, 0), z1m = min(iz + 1, A.g.dimz - 1);
        int z0 = z0m, z1 = z1m;
        if (LIST) {   // the boxes two away in z only when the reach crosses the box face
            const float zl = mez - (float)iz * Lf;
            if (zl < reach - Lf) z0 = max(iz - 2, 0);
            if (Lf - zl < reach - Lf) z1 = min(iz + 2, A.g.dimz - 1);
        }
        int m = -1, qn = 0;
        T fx = zero, fy = zero, fz = zero;   // lane partials (stencil mode)
        int nk = 0, nd = 0;
        bool spill = false;                  // uid mode: more than kWarpQ survivors
        auto drain = [&](int cnt) {          // stencil mode: evaluate Q[0, cnt)
            for (int p = lane; p < cnt; p += 32) {
                T gx, gy, gz;
                int dg;
                const int t = Q[p];
                if (pair_force(A, me, ui, storage_of(A, t), gx, gy, gz, dg)) {
                    fx = fx + gx;
                    fy = fy + gy;
                    fz = fz + gz;
                    ++nk;
                    nd += dg;
                }
            }
            __syncwarp();
        };
        // lanes 0-8 fetch one stencil column each; the reachable runs are
        // flattened into one candidate index space walked 32 at a time
        int ct0 = 0, clen = 0;
        float cmx = 0.f, cmy = 0.f;
        if (lane < NC) {
            const int ox = lane / W - R, oy = lane % W - R;
            const int nx = ix + ox, ny = iy + oy;
            if ((unsigned)nx < (unsigned)A.g.dimx && (unsigned)ny < (unsigned)A.g.dimy) {
                const int base = (nx * A.g.dimy + ny) * A.g.dimz;
                ct0 = __ldg(A.off + base + z0);
                clen = __ldg(A.off + base + z1 + 1) - ct0;
                if (!LIST) {
                    m += clen;   // summed over lanes below
                } else if (abs(ox) <= 1 && abs(oy) <= 1) {   // m: the reference's 27 boxes
                    const int m1 = z1 == z1m ? ct0 + clen : __ldg(A.off + base + z1m + 1);
                    const int m0 = z0 == z0m ? ct0 : __ldg(A.off + base + z0m);
                    m += m1 - m0;
                }
                const float gx = ox == 0 ? 0.f
                                         : fmaxf(0.f, (ox < 0 ? mex : Lf - mex) + (float)(abs(ox) - 1) * Lf);
                const float gy = oy == 0 ? 0.f
                                         : fmaxf(0.f, (oy < 0 ? mey : Lf - mey) + (float)(abs(oy) - 1) * Lf);
                if (gx * gx + gy * gy > reach2) clen = 0;
                cmx = mex - (float)ox * Lf;
                cmy = mey - (float)oy * Lf;
            }
        }
        m = (int)__reduce_add_sync(0xffffffffu, (unsigned)(lane < NC ? m + 1 : 0)) - 1;
        int cpre = clen;   // inclusive prefix of run lengths over lanes 0..NC-1
#pragma unroll
        for (int o = 1; o < (LIST ? 32 : 16); o <<= 1) {
            const int v = __shfl_up_sync(0xffffffffu, cpre, o);
            if (lane >= o) cpre += v;
        }
        const int total = __shfl_sync(0xffffffffu, cpre, NC - 1);
        const int cex = cpre - clen;   // exclusive prefix
        for (int kb = 0; kb < total; kb += 32) {
            const int k = kb + lane;
            // column of candidate k: the last column whose run starts at or before k
            // (empty runs share the next run's start, so the last one is non-empty)
            // (binary search over the non-decreasing exclusive prefixes)
            int c = 0;
#pragma unroll
            for (int step = (NC > 16 ? 16 : 8); step > 0; step >>= 1) {
                const int q = c + step;
                const int v = __shfl_sync(0xffffffffu, cex, q < NC ? q : NC - 1);
                if (q < NC && v <= k) c = q;
            }
            const int c_t0 = __shfl_sync(0xffffffffu, ct0, c);
            const int c_ex = __shfl_sync(0xffffffffu, cex, c);
            const float mx = __shfl_sync(0xffffffffu, cmx, c), my = __shfl_sync(0xffffffffu, cmy, c);
            bool pass = false;
            const int t = c_t0 + (k - c_ex);
            if (k < total) {
                const float *cp = A.prox.p + 8 * (t >> 1) + (t & 1);
                const float cx = __ldg(cp), cy = __ldg(cp + 2), zc = __ldg(cp + 4);
                const float ddx = mx - cx, ddy = my - cy, ddz = mez - zc;
                pass = __fmaf_rn(ddx, ddx, __fmaf_rn(ddy, ddy, ddz * ddz)) <= reach2 && t != s;
            }
            const unsigned bal = __ballot_sync(0xffffffffu, pass);
            if (pass) {
                const int pos = qn + __popc(bal & lt);
                if (pos < QC) Q[pos] = t;
            }
            qn += __popc(bal);
            if (!UIDMODE && qn > kWarpQ - 32) {
                __syncwarp();
                drain(qn);
                qn = 0;
            }
        }
        __syncwarp();
        T sx, sy, sz;
        int snk, snd;
        if (!UIDMODE) {
            drain(qn);
            sx = warp_tree_sum(fx);
            sy = warp_tree_sum(fy);
            sz = warp_tree_sum(fz);
            snk = __reduce_add_sync(0xffffffffu, (unsigned)nk);
            snd = __reduce_add_sync(0xffffffffu, (unsigned)nd);
        } else {
            spill = qn > QC;
            if (spill) {   // more survivors than the queue holds: the next pass
                if (lane == 0) {
                    if (BIG) A.ovf2[atomicAdd(A.ovf2_count, 1u)] = s;
                    else A.ovf[atomicAdd(A.ovf_count, 1u)] = s;
                }
                __syncwarp();
                continue;
            }
            // bitonic sort of (uid, slot) by uid over the next power of two
            int np2 = 1;
            while (np2 < qn) np2 <<= 1;
            // every uid < 2^32: sort packed (uid32 << 32 | slot) keys, uid32 read from
            // the slot's proxy (no uid gather, no separate slot swaps) -- in
            // registers up to 256 survivors, else in shared memory
            uint64_t *U = BIG ? A.big_u + (size_t)gw * A.big_cap : S.u[wid];
            const bool packed = A.uid32;
            if (packed && qn <= 64) {
                sort_queue_packed<2>(Q, qn, lane, A.prox.p);
                np2 = 0;
            } else if (packed && qn <= 128) {
                sort_queue_packed<4>(Q, qn, lane, A.prox.p);
                np2 = 0;
            } else if (packed && qn <= 256) {
                sort_queue_packed<8>(Q, qn, lane, A.prox.p);
                np2 = 0;
            }
            for (int p = lane; p < np2; p += 32) {
                if (p < qn) {
                    const int t = Q[p];
                    U[p] = packed ? ((uint64_t)__float_as_uint(__ldg(A.prox.p + 8 * (t >> 1) + 6 + (t & 1))) << 32) |
                                        (unsigned)t
                                  : A.uid[storage_of(A, t)];
                } else {
                    U[p] = ~0ull;
                    Q[p] = -1;
                }
            }
            __syncwarp();
            for (int k = 2; k <= np2; k <<= 1)
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    for (int p = lane; p < np2; p += 32) {
                        const int r = p ^ jj;
                        if (r > p) {
                            const bool up = (p & k) == 0;
                            const uint64_t u0 = U[p], u1 = U[r];
                            if ((u0 > u1) == up) {
                                U[p] = u1;
                                U[r] = u0;
                                if (!packed) {
                                    const int tq = Q[p];
                                    Q[p] = Q[r];
                                    Q[r] = tq;
                                }
                            }
                        }
                    }
                    __syncwarp();
                }
            if (packed && np2) {
                for (int p = lane; p < qn; p += 32) Q[p] = (int)(unsigned)U[p];
                __syncwarp();
            }
            // pair forces in parallel, summed by lane 0 in uid order
            T(*F)[3] = BIG ? reinterpret_cast<T(*)[3]>(static_cast<T *>(A.big_f) + (size_t)gw * A.big_cap * 3)
                           : S.f[wid];
            if (!LIST) {
                for (int p = lane; p < qn; p += 32) {
                    T gx, gy, gz;
                    int dg = 0;
                    const int t = Q[p];
                    const bool kept = pair_force(A, me, ui, storage_of(A, t), gx, gy, gz, dg);
                    F[p][0] = kept ? gx : zero;
                    F[p][1] = kept ? gy : zero;
                    F[p][2] = kept ? gz : zero;
                    nk += kept;
                    nd += dg;
                }
            } else {
                // the queue in uid order is the neighbour list (members ballot-compacted)
                int nl = 0;
                for (int pb = 0; pb < qn; pb += 32) {
                    const int p = pb + lane;
                    bool inl = false;
                    int j = 0;
                    if (p < qn) {
                        T gx = zero, gy = zero, gz = zero;
                        int dg = 0;
                        j = storage_of(A, Q[p]);
                        const bool kept = pair_force_l(A, me, ui, j, gx, gy, gz, dg, inl);
                        F[p][0] = kept ? gx : zero;
                        F[p][1] = kept ? gy : zero;
                        F[p][2] = kept ? gz : zero;
                        nk += kept;
                        nd += dg;
                    }
                    const unsigned bal = __ballot_sync(0xffffffffu, inl);
                    const int pos = nl + __popc(bal & lt);
                    if (inl && pos < A.list_cap) A.nbr[(long long)pos * A.nbr_stride + a] = j;
                    nl += __popc(bal);
                }
                if (lane == 0) {
                    A.nbr_n[a] = nl;
                    if (nl > A.list_cap) atomicAdd(A.slots + (blockIdx.x % kSlots) * kSlotWords + 10, 1ull);
                }
            }
            __syncwarp();
            sx = zero, sy = zero, sz = zero;
            if (lane == 0)
                for (int p = 0; p < qn; ++p) {
                    sx = sx + F[p][0];
                    sy = sy + F[p][1];
                    sz = sz + F[p][2];
                }
            snk = __reduce_add_sync(0xffffffffu, (unsigned)nk);
            snd = __reduce_add_sync(0xffffffffu, (unsigned)nd);
            __syncwarp();
        }
        if (lane == 0) {
            // kernels.py:266-277, engine.py:325-327
            const T norm = tsqrt<T>(sx * sx + sy * sy + sz * sz);
            T ddx = zero, ddy = zero, ddz = zero;
            if (!(norm <= A.p.adh_scale * A.adh[a])) {
                T sc = A.p.timestep;
                if (norm * sc > A.p.max_disp) sc = A.p.max_disp / norm;
                ddx = sx * sc;
                ddy = sy * sc;
                ddz = sz * sc;
            }
            A.disp_x[a] = ddx;
            A.disp_y[a] = ddy;
            A.disp_z[a] = ddz;
            dmax2 = fmaxf(dmax2, (float)((double)ddx * ddx + (double)ddy * ddy + (double)ddz * ddz));
            if (A.new_rec) {
                Rec<T> nr;
                nr.x = me.x + ddx;
                nr.y = me.y + ddy;
                nr.z = me.z + ddz;
                nr.d = me.d;
                A.new_rec[a] = nr;
                const double p3[3] = {(double)nr.x, (double)nr.y, (double)nr.z};
                unsigned long long *slot = A.slots + (blockIdx.x % kSlots) * kSlotWords;
#pragma unroll
                for (int qq = 0; qq < 3; ++qq) {
                    if (p3[qq] <= A.shell_lo[qq]) atomicMin(slot + qq, enc_ordered(p3[qq]));
                    if (p3[qq] >= A.shell_hi[qq]) atomicMax(slot + 3 + qq, enc_ordered(p3[qq]));
                }
            }
            if (A.rec_m) {
                A.rec_m[a] = m;
                A.rec_nk[a] = snk;
            }
            c_m += (unsigned)m;
            c_nk += (unsigned)snk;
            c_nd += (unsigned)snd;
        }
        __syncwarp();
    }
    warp_counters(A.slots, c_m, c_nk, c_nd);
    warp_dmax(A.slots, dmax2);   // the step's largest displacement (list-build decision)
}

}  // namespace cg
