// list.cuh -- neighbour-list reuse between grid sweeps.
//
// The reference's force phase (kernels.py:148-277) keeps, for agent i, the
// stencil candidates j with delta = (ri + rj) - dist > 0 and sums their pair
// forces in ascending uid.  The result depends only on that SET of pairs (every
// overlapping pair lies inside the 27-box stencil, L >= ri + rj), so it may be
// enumerated from any superset.  A build sweep (sweep7 with LIST) records, per
// agent and in uid order, every partner within ri + rj + skin; while the
// agents have moved by at most D in total since the build, with 2 D <= skin,
// every pair that overlaps now is in those lists (triangle inequality).  The
// list sweep then runs the reference's exact pair expressions over the list --
// bit-identical displacements, positions and counters -- without the stencil
// walk.  The per-step grid (box ids, counts, offsets, occupancy stats, the
// presentation key) is still rebuilt every step: m (the candidates counter)
// and the statistics are the reference's, from this step's grid.
#pragma once

#include "common.cuh"
#include "grid.cuh"
#include "sweep7.cuh"

namespace cg {

template <typename T>
struct ListArgs {
    int n;                    // agents swept: indices [own_lo, own_lo + n)
    int own_lo;               // 0 on a single context; the lo-ghost count on a slab
    Geometry g;
    BoxDecode bd;
    const int2 *key_rank;     // this step's box of every storage index
    const int *off;           // this step's CSR offsets
    const Rec<T> *rec;
    const T *adh;
    const uint64_t *uid;
    Params<T> p;
    const int *nbr;           // [list width][nbr_stride]
    const int *nbr_n;
    long long nbr_stride;
    // rows swept: own_lo + t for t < skip_at, own_lo + t + skip beyond (a slab's
    // boundary rows around the interior range swept earlier); no skip by default
    int skip_at, skip;
    T *disp_x, *disp_y, *disp_z;
    Rec<T> *new_rec;          // nullptr when frozen
    int *rec_m, *rec_nk;      // nullptr unless recording
    int *pkey;                // this step's box (sort steps), nullptr otherwise
    int *count;               // FUSED: per-box counts accumulated here (zero on entry)
    int *count_own;           // unused (kept zero): a slab's ghost counts come from count_ghosts
    double invL;              // FUSED: 1 / box length
    unsigned long long *slots;
    double shell_lo[3], shell_hi[3];
    // UNI (every diameter equal): the pair constants, computed on the host in
    // the pool dtype with the kernel's expressions -- rsum = ri + ri,
    // req = (ri * ri) / rsum, bound = rsum * rsum * reject_factor
    T u_rsum, u_req, u_bound;
    // INNER: the sub-list written while sweeping the neighbour list -- every
    // entry with s2 <= (rsum + inner_delta)^2 (1 + 2^-20), in list order
    int *inner, *inner_n;
    T inner_delta, u_inner_bound;   // u_inner_bound: UNI
    // FUSED: agents whose operands leave the call-free range (or coincident
    // centres) are deferred here and finished by list_slow_kernel
    int *ovf;
    unsigned *ovf_count;
};

template <typename T>
struct AgentSum {
    T fx, fy, fz;
    int nk, nd;
};

// The whole pair sum of one agent with the library's sqrt and division and
// the coincident-centre branch (kernels.py:244-257).  The pair loops run a
// call-free fast path (common.cuh) and hand an agent here when an operand
// leaves its range or two centres coincide -- rare, so out of line.
template <typename T>
__device__ __noinline__ AgentSum<T> list_agent_slow(const Rec<T> *__restrict__ rec, const uint64_t *__restrict__ uid,
                                                     const int *__restrict__ L, long long stride, int cnt, int a,
                                                     T kappa, T gamma, T zero)
{
    const T half = T(0.5);
    const Rec<T> me = rec[a];
    const T ri = me.d * half;
    AgentSum<T> S{zero, zero, zero, 0, 0};
    for (int p = 0; p < cnt; ++p) {
        const int j = L[p * stride];
        const Rec<T> co = rec[j];
        const T dx = me.x - co.x, dy = me.y - co.y, dz = me.z - co.z;
        const T rj = co.d * half;
        const T dist = tsqrt<T>(dx * dx + dy * dy + dz * dz);
        const T rsum = ri + rj;
        const T delta = rsum - dist;
        if (!(delta > zero)) continue;
        ++S.nk;
        const T req = (ri * rj) / rsum;
        const T mag = kappa * delta - gamma * tsqrt<T>(req * delta);
        if (dist > zero) {
            const T sc = mag / dist;
            S.fx = S.fx + sc * dx;
            S.fy = S.fy + sc * dy;
            S.fz = S.fz + sc * dz;
        } else {
            const uint64_t ui = uid[a], uj = uid[j];
            double ux, uy, uz;
            degenerate_dir(ui < uj ? ui : uj, ui < uj ? uj : ui, ux, uy, uz);
            const double sign = ui < uj ? 1.0 : -1.0;
            S.fx = S.fx + (T)((double)mag * (sign * ux));
            S.fy = S.fy + (T)((double)mag * (sign * uy));
            S.fz = S.fz + (T)((double)mag * (sign * uz));
            ++S.nd;
        }
    }
    return S;
}

// 64-thread CTAs, 20 per SM: 48 registers, 40 resident warps (measured at
// C4: 256 x 4 = 64 registers 1.23 ms, 128 x 9 1.18 ms, 128 x 10 1.16 ms,
// 64 x 20 1.157 ms, 128 x 11 1.45 ms -- spills inside the pair loop)
#ifndef CG_LIST_THREADS
#define CG_LIST_THREADS 64
#endif
constexpr int kListThreads = CG_LIST_THREADS;
#ifndef CG_LIST_MINB
#define CG_LIST_MINB 20
#endif


// s2 > rsum^2 (1 + 2^-40) implies fl(sqrt(s2)) > rsum, i.e. delta <= 0: the
// pair cannot be kept and needs no sqrt.  The factor is representable in both
// dtypes only for fp64; fp32 uses 1 + 4 eps (both rely on a correctly rounded
// sqrt, the library's -prec-sqrt=true default).
template <typename T>
__device__ __forceinline__ T reject_factor();
template <>
__device__ __forceinline__ double reject_factor<double>() { return 1.0000000000009095; }
template <>
__device__ __forceinline__ float reject_factor<float>() { return 1.00000048f; }

// _write_displacement (kernels.py:266-277) and apply (engine.py:325-327) of
// one agent, the next step's bbox shell and the largest displacement.
// NOCALL: the norm and the cap division call-free (common.cuh); false = an
// operand left their range, nothing written (the agent is deferred).
template <typename T, bool NOCALL>
__device__ __forceinline__ bool list_finish(const ListArgs<T> &A, int a, T xi, T yi, T zi, T di, T fx, T fy, T fz,
                                            float &dmax2)
{
    const T zero = A.p.zero;
    bool ok = true;
    const T n2 = fx * fx + fy * fy + fz * fz;
    const T norm = NOCALL ? (n2 == zero ? zero : tsqrt_nocall(n2, ok)) : tsqrt<T>(n2);
    T ddx = zero, ddy = zero, ddz = zero;
    if (!(norm <= A.p.adh_scale * A.adh[a])) {
        T sc = A.p.timestep;
        if (norm * sc > A.p.max_disp) sc = NOCALL ? tdiv_nocall(A.p.max_disp, norm, ok) : A.p.max_disp / norm;
        ddx = fx * sc;
        ddy = fy * sc;
        ddz = fz * sc;
    }
    if (NOCALL && !ok) return false;
    A.disp_x[a] = ddx;
    A.disp_y[a] = ddy;
    A.disp_z[a] = ddz;
    dmax2 = fmaxf(dmax2, (float)((double)ddx * ddx + (double)ddy * ddy + (double)ddz * ddz));
    if (A.new_rec) {
        const T nxp = xi + ddx, nyp = yi + ddy, nzp = zi + ddz;
        Rec<T> nr;
        nr.x = nxp;
        nr.y = nyp;
        nr.z = nzp;
        nr.d = di;
        A.new_rec[a] = nr;
        const double p3[3] = {(double)nxp, (double)nyp, (double)nzp};
        unsigned long long *slot = A.slots + (blockIdx.x % kSlots) * kSlotWords;
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (p3[q] <= A.shell_lo[q]) atomicMin(slot + q, enc_ordered(p3[q]));
            if (p3[q] >= A.shell_hi[q]) atomicMax(slot + 3 + q, enc_ordered(p3[q]));
        }
    }
    return true;
}

// FUSED: the step's box counting is done here (box id of the current
// position, one atomic per run of equal keys in the warp) instead of in a
// separate box_keys pass; m and the grid statistics then come from the
// per-box pass box_stencil_pass (a step without CG_STEP_RECORD).
//
// The pair loop is call-free (sqrt_nocall / div_nocall, common.cuh): an agent
// whose operands leave the fast range, or with coincident centres, is redone
// by list_agent_slow.  Entries are consumed in list (uid) order, so the sums
// are the reference's.
//
// UNI: a uniform pool -- rj, rsum, the rejection bound and req are kernel
// constants (bitwise the values the per-pair expressions give), which frees
// the registers of the per-partner cache and three FP64 operations per entry.
//
// INNER: also write the sub-list of the entries within rsum + inner_delta (a
// superset test on s2): the next list steps sweep it instead of the whole
// list while twice the motion since stays below inner_delta (two-level
// Verlet list: fewer loop iterations per warp, same pairs, same order).
template <typename T>
__device__ __forceinline__ void prefetch_l1(const T *p)
{
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

template <typename T, bool FUSED = false, bool UNI = false, bool INNER = false>
__global__ void __launch_bounds__(kListThreads, CG_LIST_MINB) list_sweep_kernel(ListArgs<T> A)
{
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned c_m = 0, c_nk = 0, c_nd = 0;
    float dmax2 = 0.f;
    // the list's first loads go out before the box counting: the count and
    // the first two indices (every row holds the list width, so entries past
    // the count are in bounds and simply unused), the adherence into L1
    // (C4 list step 1.010 -> 0.975 ms; an L1 prefetch of the index line four
    // entries ahead measured 0.975 -> 0.993 ms, profiles/r2/ab_r2y.jsonl)
    const int a0 = A.own_lo + (t < A.skip_at ? t : t + A.skip);
    int cnt0 = 0, j0 = 0, j1 = 0;
    if (t < A.n) {
        cnt0 = A.nbr_n[a0];
        j0 = __ldg(A.nbr + a0);
        j1 = __ldg(A.nbr + a0 + A.nbr_stride);
        prefetch_l1(A.adh + a0);
    }
    Rec<T> me0;   // FUSED: the agent's record, loaded once for the box key and the sweep
    if (FUSED) {   // storage order: runs of equal box keys within the warp
        const int lane = threadIdx.x & 31;
        int flat = -1 - lane;   // distinct dummy keys past n
        if (t < A.n) {
            const int row = a0;
            me0 = A.rec[row];
            flat = flat_box_fast(A.g, A.invL, me0.x, me0.y, me0.z);
            if (A.pkey) A.pkey[row] = flat;
        }
        const int prev = __shfl_up_sync(0xffffffffu, flat, 1);
        const bool start = lane == 0 || prev != flat;
        const unsigned starts = __ballot_sync(0xffffffffu, start);
        const unsigned after = starts & ~(0xffffffffu >> (31 - lane));   // run starts above this lane
        const int run_end = after ? __ffs(after) - 1 : 32;
        if (start && t < A.n) atomicAdd(A.count + flat, run_end - lane);
    }
    if (t < A.n) {
        const int a = A.own_lo + (t < A.skip_at ? t : t + A.skip);
        int m = -1;
        if (!FUSED) {
        const int key = A.key_rank[a].x;
        if (A.pkey) A.pkey[a] = key;
        int ix, iy, iz;
        decode_box(A.bd, key, ix, iy, iz);
        // m: agents of the 27 clamped boxes minus self (_gather_stencil)
        {
            const int z0 = max(iz - 1, 0), z1 = min(iz + 1, A.g.dimz - 1);
#pragma unroll
            for (int ox = -1; ox <= 1; ++ox) {
                const int nx = ix + ox;
                if ((unsigned)nx >= (unsigned)A.g.dimx) continue;
#pragma unroll
                for (int oy = -1; oy <= 1; ++oy) {
                    const int ny = iy + oy;
                    if ((unsigned)ny >= (unsigned)A.g.dimy) continue;
                    const int base = (nx * A.g.dimy + ny) * A.g.dimz;
                    m += __ldg(A.off + base + z1 + 1) - __ldg(A.off + base + z0);
                }
            }
        }
        }
        const T half = T(0.5), zero = A.p.zero;
        const Rec<T> me = FUSED ? me0 : A.rec[a];
        const T xi = me.x, yi = me.y, zi = me.z;
        const T ri = me.d * half;
        const T kfac = reject_factor<T>();
        T fx = zero, fy = zero, fz = zero;
        int nk = 0, nd = 0;
        bool ok = true;
        T last_rj = T(-1), last_req = zero;
        const int cnt = cnt0;
        // two indices and one record ahead of the entry being tested
        const int *L = A.nbr + a;
        int jn = j0, jnn = j1;
        Rec<T> o;
        if (cnt > 0) o = A.rec[jn];
        int ni = 0;   // INNER: entries written
#pragma unroll 1
        for (int p = 0; p < cnt; ++p) {
            const Rec<T> co = o;
            const int jc = jn;
            jn = jnn;
            if (p + 1 < cnt) o = A.rec[jn];
            if (p + 2 < cnt) jnn = __ldg(L + (p + 2) * A.nbr_stride);
            const T dx = xi - co.x, dy = yi - co.y, dz = zi - co.z;
            const T rj = UNI ? zero : co.d * half;
            const T s2 = dx * dx + dy * dy + dz * dz;
            const T rsum = UNI ? A.u_rsum : ri + rj;
            if (INNER) {
                const T ro = rsum + A.inner_delta;
                if (!(s2 > (UNI ? A.u_inner_bound : ro * ro * T(1.00000095367431640625)))) {
                    A.inner[(long long)ni * A.nbr_stride + a] = jc;
                    ++ni;
                }
            }
            if (s2 > (UNI ? A.u_bound : rsum * rsum * kfac)) continue;
            T rs;
            const T dist = tsqrt_nocall_r(s2, ok, rs);
            const T delta = rsum - dist;
            if (!(delta > zero)) continue;
            ++nk;
            if (UNI) {
                last_req = A.u_req;
            } else if (rj != last_rj) {
                last_rj = rj;
                last_req = tdiv_nocall(ri * rj, rsum, ok);
            }
            const T mag = A.p.kappa * delta - A.p.gamma * tsqrt_nocall(last_req * delta, ok);
            const T sc = tdiv_seeded(mag, dist, rs, ok);   // dist == 0 (coincident centres): not ok
            fx = fx + sc * dx;
            fy = fy + sc * dy;
            fz = fz + sc * dz;
            if (!ok) break;   // (measured: without the break ptxas allocates worse, 1.25 vs 1.16 ms)
        }
        if (INNER) {
            if (!ok) {   // the loop stopped early: the rest of the list goes to the sub-list unfiltered
                for (int p = 0; p < cnt; ++p) A.inner[(long long)p * A.nbr_stride + a] = __ldg(L + p * A.nbr_stride);
                ni = cnt;
            }
            A.inner_n[a] = ni;
        }
        bool done = true;
        // fp64 FUSED: no call in the pair loop or the finish -- an agent off the
        // fast range is finished by list_slow_kernel (spills 32 -> 8 bytes, list
        // step 1.035 -> 1.010 ms at C4); fp32 keeps the inline slow path (its
        // fused kernel measured 0.947 -> 1.083 ms with the deferral)
        constexpr bool DEFER_SLOW = FUSED && sizeof(T) == 8;
        if (DEFER_SLOW) {
            done = ok && list_finish<T, true>(A, a, xi, yi, zi, me.d, fx, fy, fz, dmax2);
            if (!done) A.ovf[atomicAdd(A.ovf_count, 1u)] = a;
        } else {
            if (!ok) {
                const AgentSum<T> S = list_agent_slow<T>(A.rec, A.uid, L, A.nbr_stride, cnt, a, A.p.kappa,
                                                         A.p.gamma, zero);
                fx = S.fx;
                fy = S.fy;
                fz = S.fz;
                nk = S.nk;
                nd = S.nd;
            }
            list_finish<T, false>(A, a, xi, yi, zi, me.d, fx, fy, fz, dmax2);
            if (!FUSED && A.rec_m) {
                A.rec_m[a] = m;
                A.rec_nk[a] = nk;
            }
        }
        if (!done) nk = nd = 0;   // counted by list_slow_kernel
        c_m = FUSED ? 0u : (unsigned)m;
        c_nk = (unsigned)nk;
        c_nd = (unsigned)nd;
    }
    warp_counters(A.slots, c_m, c_nk, c_nd);
    warp_dmax(A.slots, dmax2);
}

// The agents a FUSED list sweep deferred (A.ovf): the whole pair sum with the
// library's sqrt and division and the coincident-centre branch, then the
// same finish -- rare (extreme operands, coincident centres), grid-stride.
template <typename T>
__global__ void __launch_bounds__(kThreads) list_slow_kernel(ListArgs<T> A)
{
    unsigned c_nk = 0, c_nd = 0;
    float dmax2 = 0.f;
    const unsigned cnt_ovf = *A.ovf_count;
    for (unsigned k = blockIdx.x * blockDim.x + threadIdx.x; k < cnt_ovf; k += gridDim.x * blockDim.x) {
        const int a = A.ovf[k];
        const Rec<T> me = A.rec[a];
        const AgentSum<T> S = list_agent_slow<T>(A.rec, A.uid, A.nbr + a, A.nbr_stride, A.nbr_n[a], a, A.p.kappa,
                                                 A.p.gamma, A.p.zero);
        list_finish<T, false>(A, a, me.x, me.y, me.z, me.d, S.fx, S.fy, S.fz, dmax2);
        c_nk += (unsigned)S.nk;
        c_nd += (unsigned)S.nd;
    }
    warp_counters(A.slots, 0u, c_nk, c_nd);
    warp_dmax(A.slots, dmax2);
}

// After a FUSED list sweep: per occupied box b, S_b = agents of its clamped
// 27-box stencil; candidates += count_b * (S_b - 1) (every agent of b has
// m = S_b - 1, _gather_stencil), occupied boxes and the largest occupancy
// (stat[0], stat[1]).  Separable: box_sum_yz writes the 3 x 3 (y, z) window
// sums, box_stencil_pass adds the three x planes (coalesced, z fastest) and
// resets the counts to zero for the next step.
__global__ void __launch_bounds__(kThreads) box_sum_yz(Geometry g, BoxDecode bd, const int *__restrict__ count,
                                                       int *__restrict__ syz)
{
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < g.nb; b += gridDim.x * blockDim.x) {
        int ix, iy, iz;
        decode_box(bd, b, ix, iy, iz);
        int v = 0;
#pragma unroll
        for (int dy = -1; dy <= 1; ++dy) {
            if ((unsigned)(iy + dy) >= (unsigned)g.dimy) continue;
#pragma unroll
            for (int dz = -1; dz <= 1; ++dz)
                if ((unsigned)(iz + dz) < (unsigned)g.dimz) v += __ldg(count + b + dy * g.dimz + dz);
        }
        syz[b] = v;
    }
}

__global__ void __launch_bounds__(kThreads) box_stencil_pass(Geometry g, BoxDecode bd, int *__restrict__ count,
                                                             int *__restrict__ ghosts, const int *__restrict__ syz,
                                                             unsigned long long *__restrict__ slots,
                                                             unsigned long long *__restrict__ stat)
{
    unsigned long long cand = 0, occ = 0, mx = 0;
    const int plane = g.dimy * g.dimz;
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < g.nb; b += gridDim.x * blockDim.x) {
        const int c = count[b];
        if (!c) continue;
        count[b] = 0;   // the counts start the next step at zero
        int own = c;    // agents of b whose m is counted: a slab's ghosts are not
        if (ghosts) {
            const int gh = ghosts[b];
            if (gh) {
                own -= gh;
                ghosts[b] = 0;
            }
        }
        const int ix = b / plane;
        int S = __ldg(syz + b);
        if (ix > 0) S += __ldg(syz + b - plane);
        if (ix + 1 < g.dimx) S += __ldg(syz + b + plane);
        cand += (unsigned long long)own * (unsigned long long)(S - 1);
        ++occ;
        mx = max(mx, (unsigned long long)c);
    }
    cand = warp_sum(cand);
    occ = warp_sum(occ);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    // one set of atomics per block: the occupancy words are two addresses
    // every block hits (same-address atomics serialise in L2)
    __shared__ unsigned long long red[3][kThreads / 32];
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        red[0][w] = cand;
        red[1][w] = occ;
        red[2][w] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int k = 1; k < kThreads / 32; ++k) {
            cand += red[0][k];
            occ += red[1][k];
            mx = max(mx, red[2][k]);
        }
        if (cand) atomicAdd(slots + (blockIdx.x % kSlots) * kSlotWords + 7, cand);
        if (occ) atomicAdd(stat + 0, occ);
        if (mx) atomicMax(stat + 1, mx);
    }
}

// slab list steps: the ghosts' boxes join the counts (owned agents are
// counted inside the fused list sweep); one atomic per run of equal keys
template <typename T>
__global__ void __launch_bounds__(kThreads) count_ghosts(int n_total, int lo, int n_owned, Geometry g, double invL,
                                                         const Rec<T> *__restrict__ rec, int *__restrict__ count,
                                                         int *__restrict__ ghosts)
{
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    const int ng = n_total - n_owned;
    int flat = -1 - lane;
    if (k < ng) {
        const int i = k < lo ? k : k + n_owned;
        const Rec<T> r = rec[i];
        flat = flat_box_fast(g, invL, r.x, r.y, r.z);
    }
    const int prev = __shfl_up_sync(0xffffffffu, flat, 1);
    const bool start = lane == 0 || prev != flat;
    const unsigned starts = __ballot_sync(0xffffffffu, start);
    const unsigned after = starts & ~(0xffffffffu >> (31 - lane));
    const int run_end = after ? __ffs(after) - 1 : 32;
    if (start && k < ng) {
        atomicAdd(count + flat, run_end - lane);
        atomicAdd(ghosts + flat, run_end - lane);
    }
}

}  // namespace cg
