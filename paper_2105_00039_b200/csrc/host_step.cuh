// host_step.cuh -- part of the cellgrid_b200.cu translation unit (host side):
// single-context step: grid rebuild, sweep launchers, neighbour-list reuse, step_impl (engine.py:279-341).
// Included once, in order, by cellgrid_b200.cu; not a standalone header.
#pragma once

// blocks per SM of the 27-box statistics passes of a list step (with the
// block-level reduction of box_stencil_pass: 8 -> 16 measured 1.0087 -> 1.0016 ms
// per list step, profiles/r2/ab_boxred.jsonl; 32 without it: +3 %)
// dense moving pools: a build (C2: 2.7 ms) pays off over a grid sweep
// (0.72 ms) only if its lists serve ~4 steps (0.23 ms each): no build while
// the last step's largest displacement exceeds skin / 12 (expected life < 6),
// and lists that served fewer than 5 steps back the next builds off
// (C2 over 100 steps 0.84 -> 0.67 ms, moving C3-27 1.64 -> 1.32 ms,
// profiles/r2/ab_dense.jsonl)
#ifndef CG_DENSE_LIFE
#define CG_DENSE_LIFE 12.0
#endif
#ifndef CG_DENSE_MIN_LIFE
#define CG_DENSE_MIN_LIFE 5
#endif
#ifndef CG_BOX_GRID
#define CG_BOX_GRID 16
#endif

// Grid rebuild on the current storage.  Leaves key_rank, offset, skey, prox and
// idx (or, when relayout, the records in slot order in the alternate buffers).
static int ensure_big(cg_context *c);
static int ensure_lists(cg_context *c, int width);
static int list_width_for(const cg_context *c, const Geometry &g, double skin);
template <typename T>
static int build_grid_geo(cg_context *c, const Geometry &g, bool relayout, bool sort, int rot = 0,
                          bool step_path = true);

template <typename T>
static int build_grid(cg_context *c, double ir, int64_t box_cap, bool relayout, bool sort,
                      double origin[3], int64_t dims64[3])
{
    cudaStream_t st = c->stream;
    int rc;
    if (!c->bbox_valid) {
        if ((rc = standalone_bbox<T>(c))) return rc;
    } else {
        CUDA_TRY(c, cudaStreamSynchronize(st));   // the previous step's bbox readback
    }
    Geometry g;
    if ((rc = host_geometry(c, c->bbox_host, ir, box_cap, g, dims64, origin))) return rc;
    return build_grid_geo<T>(c, g, relayout, sort, 0, false);   // a grid-only build (cg_build_grid)
}

// Grid rebuild for a given geometry (global, or a slab's sub-grid).  On the
// step path (not a grid-only cg_build_grid) a dense grid also allocates the
// warp sweep's queues and the lists a later build will need, so no build
// step pays a cudaMalloc.
template <typename T>
static int build_grid_geo(cg_context *c, const Geometry &g, bool relayout, bool sort, int rot, bool step_path)
{
    const int n = (int)c->n;
    cudaStream_t st = c->stream;
    int rc;
    const int slot = (int)(c->steps_done % kRing);
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][0], st));
    if ((rc = ensure_boxes(c, g.nb))) return rc;
    c->geo = g;
    c->bd = make_decode(g);
    unsigned long long *stat = c->stat_dev + slot * kStatSlots;
    CUDA_TRY(c, cudaMemsetAsync(stat, 0, sizeof(unsigned long long) * kStatSlots, st));
    const int nblk = cdiv(n, kThreads);
    const Rec<T> *rec = (const Rec<T> *)c->b.rec[c->cur_pos];
    box_keys<T><<<nblk, kThreads, 0, st>>>(n, g, 1.0 / g.L, rec, c->count, c->b.key_rank);
    LAUNCH_CHECK(c);
    c->launches += 1;
    if ((rc = launch_scan_rts(c, g.nb, stat))) return rc;
    // sparse pools (few agents per box): the scatter is the CSR; dense pools
    // also order each box by (z, uid) so column runs can be cut on z
    const double surv = 4.19 * (double)n / (double)g.nb;   // expected survivors per agent
    const bool dense = c->path == 2 || (c->path == 0 && surv > 10.0);
    const int a = c->cur_attr, o = 1 - c->cur_pos, oa = 1 - c->cur_attr;
    int *pk = sort ? c->b.pkey[a] : nullptr;
    if (!dense) {
        if (relayout) {
            // records move straight to their slots (storage becomes slot order);
            // pkey carries the last sort step's box (this step's on a sort step)
            place_relayout<T><<<nblk, kThreads, 0, st>>>(
                n, g, c->bd, c->b.key_rank, c->offset, rec, (T *)c->b.adh[a], c->b.uid[a], c->b.skey, c->b.P(),
                sort ? nullptr : c->b.pkey[a], rot ? nullptr : c->b.pkey[oa], (Rec<T> *)c->b.rec[o] - rot,
                (T *)c->b.adh[oa] - rot, c->b.uid[oa] - rot);
            LAUNCH_CHECK(c);
            c->launches += 1;
            CUDA_TRY(c, cudaEventRecord(c->ev[slot][1], st));
        } else {
            place_full<T><<<nblk, kThreads, 0, st>>>(n, g, c->bd, c->b.key_rank, c->offset, rec, c->b.idx,
                                                     c->b.skey, c->b.P(), pk, c->b.uid[a]);
            LAUNCH_CHECK(c);
            c->launches += 1;
            CUDA_TRY(c, cudaEventRecord(c->ev[slot][1], st));
        }
    } else {
        place<<<nblk, kThreads, 0, st>>>(n, c->b.key_rank, c->offset, c->b.tmp);
        LAUNCH_CHECK(c);
        c->launches += 1;
        CUDA_TRY(c, cudaEventRecord(c->ev[slot][1], st));
        if (relayout) {
            order_gather<T, true><<<nblk, kThreads, 0, st>>>(
                n, g, c->bd, c->b.tmp, c->b.key_rank, c->offset, rec, (T *)c->b.adh[a], c->b.uid[a],
                c->b.skey, c->b.P(), nullptr, (Rec<T> *)c->b.rec[o] - rot, (T *)c->b.adh[oa] - rot,
                c->b.uid[oa] - rot, sort ? c->b.pkey[oa] : nullptr);
        } else {
            order_gather<T, false><<<nblk, kThreads, 0, st>>>(
                n, g, c->bd, c->b.tmp, c->b.key_rank, c->offset, rec, (T *)c->b.adh[a], c->b.uid[a],
                c->b.skey, c->b.P(), c->b.idx, nullptr, nullptr, nullptr, pk);
        }
        LAUNCH_CHECK(c);
        c->launches += 1;
    }
    c->last_dense = dense;
    if (step_path && dense && (rc = ensure_big(c))) return rc;   // the warp sweep's second-pass queues
    if (step_path && dense && c->list_skin != 0.0 && c->sweep_impl == 1 && c->n > 1) {
        // the lists a later build will need, allocated now (outside the build step)
        const int w = list_width_for(c, g, c->list_skin < 0 ? auto_skin(c, g) : c->list_skin);
        if (w > 0 && (rc = ensure_lists(c, w))) return rc;
    }
    if (relayout) {
        c->cur_pos = o;
        c->cur_attr = oa;
        c->relaid = true;
    } else {
        c->relaid = false;
    }
    c->rot = relayout ? rot : 0;
    if (sort) c->geo_sort = g;
    c->have_grid = true;
    return CG_OK;
}

template <typename T, bool UID, bool ZS, int KS, bool FLUSH, int MINB, bool KEY32 = false, bool UNI = false>
static int launch_sweep7_k(cg_context *c, const Sweep7Args<T> &A)
{
    cudaStream_t st = c->stream;
    CUDA_TRY(c, cudaMemsetAsync(A.ovf_count, 0, sizeof(unsigned), st));
    sweep7_kernel<T, UID, ZS, KS, FLUSH, MINB, false, KEY32, UNI><<<cdiv(A.n, kThreads), kThreads, 0, st>>>(A);
    LAUNCH_CHECK(c);
    c->launches += 1;
    if (!FLUSH) {   // agents with more than KS survivors (none in most steps)
        sweep7_overflow<T, UID, ZS, KS, false, KEY32><<<std::min(cdiv(A.n, kThreads), c->sms * 2), kThreads, 0, st>>>(A);
        LAUNCH_CHECK(c);
        c->launches += 1;
    }
    return CG_OK;
}

constexpr int kBigCap = 1024;   // survivors per agent in the second warp pass
// dense thread sweep: survivors per agent in shared memory and 128-thread CTAs
// per SM (36 x 128 x 8 B = 36 KB: 6 CTAs; measured C2 sweep 44/5: 0.828 ms,
// 36/6: 0.776 ms, 32/7: 1.073 ms -- too many agents overflow to the warp pass)
#ifndef CG_DENSE_KS
#define CG_DENSE_KS 36
#endif
#ifndef CG_DENSE_MINB
#define CG_DENSE_MINB 6
#endif
constexpr int kDenseKS = CG_DENSE_KS;    // survivor list of the thread-per-agent dense sweep
constexpr double kDenseThreadSurv = 36.0;   // expected survivors up to which it is used (C3-50: 52, warp path)

// the second pass for dense uid-mode agents that spilled the warp's shared
// queue (A.ovf), then the thread-per-agent rounds for the few beyond kBigCap
static int ensure_big(cg_context *c)
{
    const int warps = c->sms * 4 * (kThreads / 32);
    if (c->big_warps < warps) {
        if (c->big) cudaFree(c->big);
        c->big = nullptr;
        c->big_warps = 0;
        CUDA_TRY(c, cudaMalloc(&c->big, (size_t)warps * kBigCap * (4 + 8 + 3 * 8)));
        c->big_warps = warps;
    }
    if (!c->ovf2_count) CUDA_TRY(c, cudaMalloc(&c->ovf2_count, sizeof(unsigned)));
    if (c->ovf2_cap < c->cap) {
        if (c->ovf2) cudaFree(c->ovf2);
        c->ovf2 = nullptr;
        c->ovf2_cap = 0;
        CUDA_TRY(c, cudaMalloc(&c->ovf2, sizeof(int) * (size_t)std::max<int64_t>(c->cap, 1)));
        c->ovf2_cap = c->cap;
    }
    return CG_OK;
}

template <typename T, bool LIST>
static int launch_sweep_warp_big(cg_context *c, const Sweep7Args<T> &A0)
{
    cudaStream_t st = c->stream;
    int rc = ensure_big(c);   // normally done when the grid turned dense
    if (rc) return rc;
    const int warps = c->big_warps;
    Sweep7Args<T> A = A0;
    char *base = (char *)c->big;
    A.big_cap = kBigCap;
    A.big_u = (uint64_t *)base;
    A.big_f = base + (size_t)warps * kBigCap * 8;
    A.big_q = (int *)(base + (size_t)warps * kBigCap * (8 + 3 * 8));
    A.ovf2 = c->ovf2;
    A.ovf2_count = c->ovf2_count;
    CUDA_TRY(c, cudaMemsetAsync(c->ovf2_count, 0, sizeof(unsigned), st));
    sweep_warp_kernel<T, true, LIST, true><<<c->sms * 4, kThreads, 0, st>>>(A);
    LAUNCH_CHECK(c);
    Sweep7Args<T> B = A;
    B.ovf = c->ovf2;
    B.ovf_count = c->ovf2_count;
    sweep7_overflow<T, true, true, 16, LIST><<<std::min(cdiv(A.n, kThreads), c->sms * 2), kThreads, 0, st>>>(B);
    LAUNCH_CHECK(c);
    c->launches += 2;
    return CG_OK;
}

// Uniform fp64 pool: the sweep's pair constants (sweep7.cuh UNI), host-computed
// with the kernel's expressions.  Sets them in a copy the caller launches with.
template <typename T>
static bool sweep_uniform(const cg_context *c, const Sweep7Args<T> &A0)
{
    Sweep7Args<T> &A = const_cast<Sweep7Args<T> &>(A0);
    if (sizeof(T) != 8 || !(c->min_diam == c->max_diam) || !std::isfinite(c->max_diam)) return false;
    const T ri = (T)c->max_diam * T(0.5);
    const T rsum = ri + ri;
    A.u_rsum = rsum;
    A.u_req = (ri * ri) / rsum;
    A.u_lim = rsum + A.skin;
    return std::isnormal(A.u_req) && std::isnormal(rsum);
}

template <typename T>
static int launch_sweep7(cg_context *c, const Sweep7Args<T> &A)
{
    if (A.nbr) {   // grid sweep that also builds the neighbour lists (uid order)
        cudaStream_t st = c->stream;
        CUDA_TRY(c, cudaMemsetAsync(A.ovf_count, 0, sizeof(unsigned), st));
        if (!c->last_dense) {
            const int g1 = cdiv(A.n, kThreads), g2 = std::min(cdiv(A.n, kThreads), c->sms * 2);
            if (A.uid32 && sweep_uniform(c, A)) {
                sweep7_kernel<T, true, false, CG_LIST_BUILD_KS, false, CG_LIST_BUILD_MINB, true, true, true>
                    <<<g1, kThreads, 0, st>>>(A);
                sweep7_overflow<T, true, false, CG_LIST_BUILD_KS, true, true><<<g2, kThreads, 0, st>>>(A);
            } else if (A.uid32) {
                sweep7_kernel<T, true, false, CG_LIST_BUILD_KS, false, CG_LIST_BUILD_MINB, true, true><<<g1, kThreads, 0, st>>>(A);
                sweep7_overflow<T, true, false, CG_LIST_BUILD_KS, true, true><<<g2, kThreads, 0, st>>>(A);
            } else {
                sweep7_kernel<T, true, false, 16, false, CG_LIST_BUILD_MINB, true><<<g1, kThreads, 0, st>>>(A);
                sweep7_overflow<T, true, false, 16, true><<<g2, kThreads, 0, st>>>(A);
            }
        } else if (4.19 * (double)A.n / (double)c->geo.nb <= 20.0) {
            // moderately dense: one thread per agent on z-sorted boxes
            sweep7_kernel<T, true, true, 16, false, 3, true><<<cdiv(A.n, kThreads), kThreads, 0, st>>>(A);
            sweep7_overflow<T, true, true, 16, true><<<cdiv(A.n, kThreads), kThreads, 0, st>>>(A);
        } else {
            // dense: one warp per agent, the uid-sorted survivor queue is the list;
            // agents with more than kWarpQ survivors take the second (global-queue) pass
            auto k = sweep_warp_kernel<T, true, true>;
            const size_t sm = sizeof(WarpSmem<T, true>);
            CUDA_TRY(c, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
            k<<<std::min(cdiv(A.n, kThreads / 32), c->sms * 12), kThreads, sm, st>>>(A);
            LAUNCH_CHECK(c);
            c->launches += 1;
            return launch_sweep_warp_big<T, true>(c, A);
        }
        LAUNCH_CHECK(c);
        c->launches += 2;
        return CG_OK;
    }
    if (!c->last_dense) {
        // sparse: survivors summed in uid order (deterministic and bit-identical to
        // the reference whatever the slot order in a box); agents with more than
        // 16 survivors go to the overflow kernel
        if (A.uid32 && sweep_uniform(c, A))
            return launch_sweep7_k<T, true, false, 16, false, CG_SPARSE_MINB, true, true>(c, A);
        if (A.uid32) return launch_sweep7_k<T, true, false, 16, false, CG_SPARSE_MINB, true>(c, A);
        return launch_sweep7_k<T, true, false, 16, false, CG_SPARSE_MINB>(c, A);
    }
    // moderately dense (<= 20 expected survivors): one thread per agent
    const double surv = 4.19 * (double)A.n / (double)c->geo.nb;
    if (surv <= 20.0) {
        if (c->summation == SUM_UID) return launch_sweep7_k<T, true, true, 16, false, 3>(c, A);
        return launch_sweep7_k<T, false, true, 32, true, 3>(c, A);   // list evaluated whenever it fills
    }
    // dense: one warp per agent (warp-cooperative walk, survivors compacted
    // into a per-warp queue); uid order bit-exact, stencil order deterministic
    cudaStream_t st = c->stream;
    const int blocks = std::min(cdiv(A.n, kThreads / 32), c->sms * 16);
    CUDA_TRY(c, cudaMemsetAsync(A.ovf_count, 0, sizeof(unsigned), st));
    if (A.uid32 && surv <= kDenseThreadSurv) {
        // moderately dense (C2: ~27 survivors): one thread per agent with a
        // kDenseKS-entry survivor list in shared memory; agents with more
        // survivors (or an operand outside the call-free range) go to the
        // warp kernel's global-queue pass.  Sums in uid order whatever the
        // requested summation: the reference's order, and faster here than the
        // stencil-order warp sweep (C2 0.76 vs 1.29 ms)
        constexpr int NT = 128;
        if (sweep_uniform(c, A))
            sweep7_kernel<T, true, true, kDenseKS, false, CG_DENSE_MINB, false, true, true, NT><<<cdiv(A.n, NT), NT, 0, st>>>(A);
        else
            sweep7_kernel<T, true, true, kDenseKS, false, CG_DENSE_MINB, false, true, false, NT><<<cdiv(A.n, NT), NT, 0, st>>>(A);
        LAUNCH_CHECK(c);
        c->launches += 1;
        return launch_sweep_warp_big<T, false>(c, A);
    }
    if (c->summation == SUM_UID) {
        auto k = sweep_warp_kernel<T, true>;
        const size_t sm = sizeof(WarpSmem<T, true>);
        CUDA_TRY(c, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k<<<blocks, kThreads, sm, st>>>(A);
        LAUNCH_CHECK(c);
        c->launches += 1;
        return launch_sweep_warp_big<T, false>(c, A);
    } else {
        auto k = sweep_warp_kernel<T, false>;
        const size_t sm = sizeof(WarpSmem<T, false>);
        CUDA_TRY(c, cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        k<<<blocks, kThreads, sm, st>>>(A);
        LAUNCH_CHECK(c);
        c->launches += 1;
    }
    return CG_OK;
}

// bbox shell (see sweep7.cuh): an agent can only become extreme if it ends
// within max_displacement (+ rounding slack) of the old bbox faces
static void bbox_shell(const cg_context *c, double md, double shell_lo[3], double shell_hi[3])
{
    const bool ok = std::isfinite(md) && md >= 0.0;
    for (int q = 0; q < 3; ++q) {
        const double lo = c->bbox_host[q], hi = c->bbox_host[3 + q];
        const double slack = 1e-6 * (std::fabs(lo) + std::fabs(hi) + 1.0);
        const double B = ok ? md * (1.0 + 1e-6) + slack : INFINITY;
        shell_lo[q] = lo + B;
        shell_hi[q] = hi - B;
    }
}

// After a list build (list_builds already counted): if the build also wrote
// both sub-lists (run_sweep), they hold its partners within their deltas
static void mark_build_sublists(cg_context *c)
{
    if (!c->sub_built) return;
    for (int k = 1; k <= 2; ++k) {
        c->lvl_delta[k] = c->lvl_frac[k] * c->list_skin_used;
        c->lvl_valid[k] = true;
        c->lvl_written[k] = true;
        c->lvl_epoch[k] = c->list_builds;
        c->lvl_parent[k] = k - 1;
    }
}

template <typename T>
static int run_sweep(cg_context *c, const double params[5], bool freeze, bool record, bool build_lists = false,
                     bool subs = false)
{
    const int n = (int)c->n;
    cudaStream_t st = c->stream;
    const int cp = c->cur_pos, ca = c->cur_attr;
    Rec<T> *nrec = freeze ? nullptr : (Rec<T> *)c->b.rec[1 - cp];
    const Params<T> P = make_params<T>(params);
    if (c->sweep_impl == 0) {
        // reference-order thread-per-agent sweep (sweep.cuh), then a standalone bbox next step
        const int nblk = cdiv(n, kThreads);
        if (nblk > kMaxCounterBlocks) return fail(c, CG_ERR_VALUE, "population too large for sweep 0");
        SweepArgs<T> A{};
        A.n = n;
        A.g = c->geo;
        A.rec = (const Rec<T> *)c->b.rec[cp];
        A.adh = (const T *)c->b.adh[ca];
        A.uid = c->b.uid[ca];
        A.idx = c->relaid ? nullptr : c->b.idx;
        A.slot_key = c->b.skey;
        A.off = c->offset;
        A.p = P;
        A.disp_x = (T *)c->b.disp[0];
        A.disp_y = (T *)c->b.disp[1];
        A.disp_z = (T *)c->b.disp[2];
        A.new_rec = nrec;
        A.rec_m = record ? c->b.rec_m : nullptr;
        A.rec_nk = record ? c->b.rec_nk : nullptr;
        A.block_counters = c->block_counters;
        if (c->relaid) {
            if (c->summation == SUM_UID) sweep_kernel<T, true, SUM_UID, 32><<<nblk, kThreads, 0, st>>>(A);
            else sweep_kernel<T, true, SUM_STENCIL, 1><<<nblk, kThreads, 0, st>>>(A);
        } else {
            if (c->summation == SUM_UID) sweep_kernel<T, false, SUM_UID, 32><<<nblk, kThreads, 0, st>>>(A);
            else sweep_kernel<T, false, SUM_STENCIL, 1><<<nblk, kThreads, 0, st>>>(A);
        }
        LAUNCH_CHECK(c);
        unsigned long long *stat = c->stat_dev + (c->steps_done % kRing) * kStatSlots;
        reduce_counters<<<1, kThreads, 0, st>>>(nblk, c->block_counters, stat);
        LAUNCH_CHECK(c);
        c->launches += 2;
        c->bbox_valid = freeze && c->bbox_valid;
        return CG_OK;
    }
    Sweep7Args<T> A{};
    A.n = n;
    A.g = c->geo;
    A.bd = c->bd;
    A.prox = c->b.P();
    A.skey = c->b.skey;
    A.idx = c->relaid ? nullptr : c->b.idx;
    A.off = c->offset;
    // relaid slab sub-grid: every storage-order column is addressed by slot
    // (shifted by rot; the writes land at [0, n_owned))
    const int rot = c->relaid ? c->rot : 0;
    A.rec = (const Rec<T> *)c->b.rec[cp] - rot;
    A.adh = (const T *)c->b.adh[ca] - rot;
    A.uid = c->b.uid[ca] - rot;
    A.p = P;
    A.rmax = nextafterf((float)(0.5 * c->max_diam), INFINITY);
    // fp32 prefilter margin: every stored / derived fp32 coordinate is within
    // a few ulp of E (box-local x/y, grid-relative z); 64 ulp(E) is used
    const double E = c->geo.L * (double)std::max(3, std::max(c->geo.dimz + 2, 3));
    A.margin = (float)(64.0 * E * 5.9604644775390625e-8);
    A.disp_x = (T *)c->b.disp[0] - rot;
    A.disp_y = (T *)c->b.disp[1] - rot;
    A.disp_z = (T *)c->b.disp[2] - rot;
    A.new_rec = nrec ? nrec - rot : nullptr;
    A.rec_m = record ? c->b.rec_m - rot : nullptr;
    A.rec_nk = record ? c->b.rec_nk - rot : nullptr;
    A.slots = c->slots;
    // bbox shell (see sweep7.cuh): an agent can only become extreme if it ends
    // within max_displacement (+ rounding slack) of the old bbox faces
    bbox_shell(c, (double)P.max_disp, A.shell_lo, A.shell_hi);
    A.ovf = c->b.ovf;
    A.ovf_count = c->ovf_count;
    A.n_owned = (int)c->n_owned;
    A.own_lo = c->rot;
    A.uid32 = c->uid32;
    if (build_lists) {
        A.nbr = c->nbr;
        A.nbr_n = c->nbr_n;
        A.nbr_stride = c->nbr_cap;
        A.list_cap = c->list_width;
        A.skin = (T)c->list_skin_used;
        A.skin_f = nextafterf((float)c->list_skin_used, INFINITY);
    }
    // the two sub-lists written with the list (single context, the sweep7
    // list builds; the dense warp build writes only the list)
    c->sub_built = false;
    if (build_lists && subs && c->lvl_nbr[1] && c->lvl_nbr[2] && c->lvl_frac[1] > 0.0 &&
        c->lvl_frac[2] > 0.0 && c->lvl_frac[2] < c->lvl_frac[1] && c->lvl_frac[1] < 1.0 &&
        (!c->last_dense || 4.19 * (double)n / (double)c->geo.nb <= 20.0)) {
        A.sub1 = c->lvl_nbr[1];
        A.sub1_n = c->lvl_n[1];
        A.sub2 = c->lvl_nbr[2];
        A.sub2_n = c->lvl_n[2];
        A.sub1_d = (T)(c->lvl_frac[1] * c->list_skin_used);
        A.sub2_d = (T)(c->lvl_frac[2] * c->list_skin_used);
        if (sizeof(T) == 8 && c->min_diam == c->max_diam && std::isfinite(c->max_diam)) {
            const T ri = (T)c->max_diam * T(0.5);
            const T rsum = ri + ri;
            A.u_sub1 = rsum + A.sub1_d;
            A.u_sub2 = rsum + A.sub2_d;
        }
        c->sub_built = true;
    }
    int rc = launch_sweep7<T>(c, A);
    if (rc) return rc;
    unsigned long long *stat = c->stat_dev + (c->steps_done % kRing) * kStatSlots;
    // frozen: positions (and so the bbox in bbox_host) are unchanged
    finish_step<<<1, kThreads, 0, st>>>(c->slots, c->max_diam, stat, c->bbox_dev,
                                         FINISH_COUNTERS | (freeze ? 0 : FINISH_BBOX));
    LAUNCH_CHECK(c);
    c->launches += 1;
    if (!freeze)
        CUDA_TRY(c, cudaMemcpyAsync(c->bbox_host, c->bbox_dev, 9 * sizeof(double), cudaMemcpyDeviceToHost, st));
    else   // frozen: the bbox is unchanged, but a list build's overflow count is new
        CUDA_TRY(c, cudaMemcpyAsync(c->bbox_host + 7, c->bbox_dev + 7, 2 * sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
    c->bbox_valid = true;
    return CG_OK;
}

// ---------------------------------------------------------------- neighbour-list reuse
static int ensure_lists(cg_context *c, int width)
{
    if (c->nbr && c->nbr_cap == c->cap && c->nbr_width >= width) return CG_OK;
    c->list_valid = false;   // new storage: whatever lists there were are gone
    if (c->nbr) cudaFree(c->nbr);
    if (c->nbr_n) cudaFree(c->nbr_n);
    c->nbr = c->nbr_n = nullptr;
    free_inner(c);
    c->nbr_cap = 0;
    c->nbr_width = 0;
    CUDA_TRY(c, cudaMalloc(&c->nbr, sizeof(int) * (size_t)width * (size_t)c->cap));
    CUDA_TRY(c, cudaMalloc(&c->nbr_n, sizeof(int) * (size_t)c->cap));
    // the sub-lists, same width, within the 16 GB list budget (the middle level
    // only when enabled)
    double used = (double)width * (double)c->cap * 4.0;
    for (int k = 2; k >= 1; --k) {
        if (c->lvl_frac[k] <= 0.0 || used + (double)width * (double)c->cap * 4.0 > 16e9) continue;
        CUDA_TRY(c, cudaMalloc(&c->lvl_nbr[k], sizeof(int) * (size_t)width * (size_t)c->cap));
        CUDA_TRY(c, cudaMalloc(&c->lvl_n[k], sizeof(int) * (size_t)c->cap));
        used += (double)width * (double)c->cap * 4.0;
    }
    c->nbr_cap = c->cap;
    c->nbr_width = width;
    return CG_OK;
}

// list width for the next build: kListCap on sparse pools; on dense pools
// (the same test as build_grid_geo) the expected partner count within
// max diameter + skin at the pool's mean density (bbox volume) plus a Poisson
// tail; 0 = too wide, no lists.  An agent with more partners than the width
// still makes the build's lists unusable (overflow count), never wrong.
static int list_width_for(const cg_context *c, const Geometry &g, double skin)
{
    const double surv = 4.19 * (double)c->n / (double)g.nb;
    const bool dense = c->path == 2 || (c->path == 0 && surv > 10.0);
    if (!dense) return kListCap;
    double vol = 1.0;
    for (int q = 0; q < 3; ++q) vol *= std::max(c->bbox_host[3 + q] - c->bbox_host[q], g.L);
    const double r = c->max_diam + skin;
    const double mu = 4.18879 * r * r * r * (double)c->n / vol;
    const int w = ((int)std::ceil(1.25 * mu + 6.0 * std::sqrt(mu) + 16.0) + 15) & ~15;
    if (w > 1024 || (double)w * (double)c->cap * 4.0 > 16e9) return 0;
    return std::max(w, kListCap);
}

// After the previous step's readback: lists built last step become valid if
// no agent overflowed; every step on valid lists adds its largest
// displacement (+ rounding of the position update) to the motion bound D.
template <typename T>
static void list_account(cg_context *c)
{
    if (c->last_kind == 1) {
        c->list_valid = c->bbox_host[8] == 0.0;
        c->list_D = 0.0;
        c->list_life = 0;
        if (!c->list_valid) {   // some agent has more than kListCap partners: back off
            c->list_backoff = c->list_backoff ? std::min(2 * c->list_backoff, 64) : 4;
            c->list_wait = c->list_backoff;
        }
    }
    for (int k = 1; k < 3; ++k)
        if (c->lvl_written[k]) {   // a sub-list reflects the positions before the last step's move
            c->lvl_D[k] = 0.0;
            c->lvl_written[k] = false;
        }
    if (c->list_valid && c->last_kind != 0 && !c->last_freeze) {
        double M = 0.0;
        for (int q = 0; q < 6; ++q) M = std::max(M, std::fabs(c->bbox_host[q]));
        const double ulp = M * (sizeof(T) == 8 ? 2.220446049250313e-16 : 1.1920928955078125e-07);
        const double dD = std::sqrt(std::max(c->bbox_host[7], 0.0)) * (1.0 + 1e-6) + 2.0 * ulp;
        c->list_D += dD;
        c->lvl_D[1] += dD;
        c->lvl_D[2] += dD;
    }
}

// Which list a fused list step sweeps and which sub-list it writes (list.cuh
// INNER): the shortest valid level -- level 2 if it and its parent chain are
// valid, else level 1, else the neighbour list -- and the next enabled level
// below the one swept.  A sub-list written from level r holds every partner of
// r within r_i + r_j + delta; a pair missing from it was either outside delta
// at the write (safe while 2 D < delta) or missing from r (safe while r is).
static void choose_levels(cg_context *c, bool fused, int &read, int &write)
{
    read = 0;
    write = -1;
    if (!fused) return;
    auto usable = [&](int k) {
        return c->lvl_nbr[k] && c->lvl_frac[k] > 0.0 && c->lvl_valid[k] && c->lvl_epoch[k] == c->list_builds &&
               2.0 * c->lvl_D[k] <= 0.999 * c->lvl_delta[k];
    };
    const bool ok1 = usable(1);
    const bool ok2 = usable(2) && (c->lvl_parent[2] == 0 || ok1);
    read = ok2 ? 2 : ok1 ? 1 : 0;
    for (int k = read + 1; k <= 2; ++k)
        if (c->lvl_nbr[k] && c->lvl_frac[k] > 0.0) {
            write = k;
            break;
        }
    if (read > 0) c->inner_steps++;
    if (write > 0) {
        c->lvl_delta[write] = c->lvl_frac[write] * c->list_skin_used;
        c->lvl_valid[write] = true;
        c->lvl_written[write] = true;
        c->lvl_epoch[write] = c->list_builds;
        c->lvl_parent[write] = read;
        if (write == 1) c->lvl_valid[2] = c->lvl_valid[2] && c->lvl_parent[2] == 0;   // its children go with it
    }
}

template <typename T>
static void apply_levels(const cg_context *c, ListArgs<T> &A, int read, int write)
{
    if (read > 0) {
        A.nbr = c->lvl_nbr[read];
        A.nbr_n = c->lvl_n[read];
    }
    if (write > 0) {
        A.inner = c->lvl_nbr[write];
        A.inner_n = c->lvl_n[write];
        A.inner_delta = (T)c->lvl_delta[write];
    }
}

// Uniform pool: the list sweep's pair constants (list.cuh UNI), in the pool
// dtype with the kernel's expression order (host: -ffp-contract=off, SSE).
// fp64 only (C4 list sweep 1.159 -> 1.040 ms, C3-27 0.465 -> 0.403 ms; the
// fp32 kernel measured 0.921 -> 0.940 ms, profiles/r2/ab_r2g.jsonl, and again
// 0.870 -> 0.892 ms after the early loads, ab_r2aa.jsonl).
template <typename T>
static bool list_uniform(const cg_context *c, ListArgs<T> &A)
{
    if (sizeof(T) != 8 || !(c->min_diam == c->max_diam) || !std::isfinite(c->max_diam)) return false;
    const T ri = (T)c->max_diam * T(0.5);
    const T rsum = ri + ri;
    A.u_rsum = rsum;
    A.u_req = (ri * ri) / rsum;
    A.u_bound = rsum * rsum * (sizeof(T) == 8 ? (T)1.0000000000009095 : (T)1.00000048f);
    return std::isnormal(A.u_req) && std::isnormal(rsum);
}

template <typename T>
static void launch_list_sweep(cg_context *c, ListArgs<T> &A, int n, bool fused, cudaStream_t st)
{
    const bool uni = list_uniform<T>(c, A);
    const int nblk = cdiv(n, kListThreads);
    if (fused) {   // agents off the call-free range are deferred to list_slow_kernel
        A.ovf = c->b.ovf;
        A.ovf_count = c->ovf_count;
        cudaMemsetAsync(c->ovf_count, 0, sizeof(unsigned), st);
    }
    if (fused && A.inner) {   // also write the sub-list (fused steps only)
        if (uni) {
            const T ro = A.u_rsum + A.inner_delta;
            A.u_inner_bound = ro * ro * (T)1.00000095367431640625;
            list_sweep_kernel<T, true, true, true><<<nblk, kListThreads, 0, st>>>(A);
        } else {
            list_sweep_kernel<T, true, false, true><<<nblk, kListThreads, 0, st>>>(A);
        }
    } else if (fused) {
        if (uni) list_sweep_kernel<T, true, true><<<nblk, kListThreads, 0, st>>>(A);
        else list_sweep_kernel<T, true><<<nblk, kListThreads, 0, st>>>(A);
    } else {
        if (uni) list_sweep_kernel<T, false, true><<<nblk, kListThreads, 0, st>>>(A);
        else list_sweep_kernel<T><<<nblk, kListThreads, 0, st>>>(A);
    }
    if (fused) {
        list_slow_kernel<T><<<c->sms, kThreads, 0, st>>>(A);
        c->launches += 1;
    }
}

template <typename T>
static int list_step_t(cg_context *c, const Geometry &g, const double params[5], bool sort, bool freeze,
                       bool record)
{
    const int n = (int)c->n;
    cudaStream_t st = c->stream;
    const int slot = (int)(c->steps_done % kRing);
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][0], st));
    int rc;
    if ((rc = ensure_boxes(c, g.nb))) return rc;
    c->geo = g;
    c->bd = make_decode(g);
    unsigned long long *stat = c->stat_dev + slot * kStatSlots;
    CUDA_TRY(c, cudaMemsetAsync(stat, 0, sizeof(unsigned long long) * kStatSlots, st));
    const int cp = c->cur_pos, ca = c->cur_attr;
    // a recorded step (per-agent m / nk, grid export) builds the CSR first;
    // otherwise the box counting runs inside the list sweep (FUSED) and the
    // candidates counter and grid statistics come from one pass over the boxes
    const bool fused = !record;
    if (!fused) {
        box_keys<T><<<cdiv(n, kThreads), kThreads, 0, st>>>(n, g, 1.0 / g.L, (const Rec<T> *)c->b.rec[cp], c->count,
                                                            c->b.key_rank);
        LAUNCH_CHECK(c);
        c->launches += 1;
        if ((rc = launch_scan_rts(c, g.nb, stat))) return rc;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][1], st));
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][2], st));
    ListArgs<T> A{};
    A.skip_at = INT_MAX;
    A.n = n;
    A.g = g;
    A.bd = c->bd;
    A.key_rank = c->b.key_rank;
    A.off = c->offset;
    A.rec = (const Rec<T> *)c->b.rec[cp];
    A.adh = (const T *)c->b.adh[ca];
    A.uid = c->b.uid[ca];
    A.p = make_params<T>(params);
    A.nbr = c->nbr;
    A.nbr_n = c->nbr_n;
    A.nbr_stride = c->nbr_cap;
    // the shortest valid sub-list is swept, the next one written (choose_levels)
    {
        int rd, wr;
        choose_levels(c, fused, rd, wr);
        apply_levels<T>(c, A, rd, wr);
    }
    A.disp_x = (T *)c->b.disp[0];
    A.disp_y = (T *)c->b.disp[1];
    A.disp_z = (T *)c->b.disp[2];
    A.new_rec = freeze ? nullptr : (Rec<T> *)c->b.rec[1 - cp];
    A.rec_m = record ? c->b.rec_m : nullptr;
    A.rec_nk = record ? c->b.rec_nk : nullptr;
    A.pkey = sort ? c->b.pkey[ca] : nullptr;
    A.count = c->count;
    A.invL = 1.0 / g.L;
    A.slots = c->slots;
    bbox_shell(c, (double)A.p.max_disp, A.shell_lo, A.shell_hi);
    if (fused) {
        launch_list_sweep<T>(c, A, n, true, st);
        const int gb = std::min(cdiv(g.nb, kThreads), c->sms * CG_BOX_GRID);
        box_sum_yz<<<gb, kThreads, 0, st>>>(g, c->bd, c->count, c->offset);   // offsets are unused on a fused step
        box_stencil_pass<<<gb, kThreads, 0, st>>>(g, c->bd, c->count, nullptr, c->offset, c->slots, stat);
        c->launches += 3;
    } else {
        launch_list_sweep<T>(c, A, n, false, st);
        c->launches += 1;
    }
    finish_step<<<1, kThreads, 0, st>>>(c->slots, c->max_diam, stat, c->bbox_dev,
                                         FINISH_COUNTERS | (freeze ? 0 : FINISH_BBOX));
    LAUNCH_CHECK(c);
    c->launches += 1;
    if (!freeze)
        CUDA_TRY(c, cudaMemcpyAsync(c->bbox_host, c->bbox_dev, 9 * sizeof(double), cudaMemcpyDeviceToHost, st));
    c->bbox_valid = true;
    c->have_grid = !fused;   // a fused step keeps no slot-level CSR to export
    c->relaid = false;       // slot arrays are not rebuilt: exports use key_rank
    c->last_dense = false;
    if (sort) c->geo_sort = g;
    c->list_life++;
    c->list_steps++;
    return CG_OK;
}

static int ensure_copy_stream(cg_context *c)
{
    if (c->copy_stream) return CG_OK;
    // highest priority: the reorder kernels of an early download go ahead of
    // the sweep's blocks, so the PCIe transfer starts while the sweep runs
    int lo = 0, hi = 0;
    CUDA_TRY(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CUDA_TRY(c, cudaStreamCreateWithPriority(&c->copy_stream, cudaStreamNonBlocking, hi));
    for (int k = 0; k < 9; ++k) {
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->dl_ready[k], cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->dl_done[k], cudaEventDisableTiming));
    }
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->dl_start, cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->early.grid_done, cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->early.ready, cudaEventDisableTiming));
    return CG_OK;
}

// cg_step_download, once the grid of the step is built: the reference order
// (pres) is materialised and the columns the sweep does not change --
// diameter, adherence, uid -- are reordered and copied to the host on the
// copy stream while the sweep runs on the context stream.
template <typename T>
static int early_download(cg_context *c)
{
    int rc;
    if ((rc = ensure_copy_stream(c))) return rc;
    const int64_t n = c->n;
    const size_t need = 2 * 8 * (size_t)n;
    if (need > c->early.bytes) {
        if (c->early.buf) cudaFree(c->early.buf);
        c->early.buf = nullptr;
        CUDA_TRY(c, cudaMalloc(&c->early.buf, need));
        c->early.bytes = need;
    }
    cudaStream_t st = c->stream, cs = c->copy_stream;
    CUDA_TRY(c, cudaEventRecord(c->early.grid_done, st));
    CUDA_TRY(c, cudaStreamWaitEvent(cs, c->early.grid_done, 0));
    if ((rc = materialize_presentation(c, cs))) return rc;
    const int *pres = c->pres_state == PRES_IDENTITY ? nullptr : c->b.pres;
    char *buf[3] = {c->early.buf, c->early.buf + 8 * (size_t)n, (char *)c->b.stage};
    const int nb = cdiv(n, kThreads);
    if (c->early.dst[0])
        unpack_component<T><<<nb, kThreads, 0, cs>>>((int)n, (const Rec<T> *)c->b.rec[c->cur_pos], 3, pres,
                                                     (T *)buf[0]);
    const void *src[3] = {nullptr, c->b.adh[c->cur_attr], c->b.uid[c->cur_attr]};
    for (int k = 1; k < 3; ++k) {
        if (!c->early.dst[k]) continue;
        if (!pres) {
            buf[k] = (char *)src[k];
        } else if (k == 2 || sizeof(T) == 8) {
            scatter_by<unsigned long long><<<nb, kThreads, 0, cs>>>((int)n, pres, (const unsigned long long *)src[k],
                                                                    (unsigned long long *)buf[k]);
        } else {
            scatter_by<unsigned><<<nb, kThreads, 0, cs>>>((int)n, pres, (const unsigned *)src[k], (unsigned *)buf[k]);
        }
    }
    LAUNCH_CHECK(c);
    c->launches += 3;
    for (int k = 0; k < 3; ++k)
        if (c->early.dst[k])
            CUDA_TRY(c, cudaMemcpyAsync(c->early.dst[k], buf[k], (k == 2 ? 8 : sizeof(T)) * (size_t)n,
                                        cudaMemcpyDeviceToHost, cs));
    CUDA_TRY(c, cudaEventRecord(c->early.ready, cs));
    c->early.done = true;
    return CG_OK;
}

template <typename T>
static int step_impl(cg_context *c, const double params[5], double ir, int64_t box_cap, int flags,
                     int64_t *step_id)
{
    const int slot = (int)(c->steps_done % kRing);
    cg_step_stats &S = c->ring[slot];
    std::memset(&S, 0, sizeof S);
    S.step_id = c->steps_done;
    S.agent_count = c->n;
    *step_id = c->steps_done;
    cudaStream_t st = c->stream;
    if (c->n == 0) {   // engine.py:291-298
        c->have_grid = false;
        CUDA_TRY(c, cudaMemsetAsync(c->stat_dev + slot * kStatSlots, 0, sizeof(unsigned long long) * kStatSlots, st));
        for (int e = 0; e < 5; ++e) CUDA_TRY(c, cudaEventRecord(c->ev[slot][e], st));
        CUDA_TRY(c, cudaMemcpyAsync(c->stat_host + slot * kStatSlots, c->stat_dev + slot * kStatSlots,
                                    sizeof(unsigned long long) * kStatSlots, cudaMemcpyDeviceToHost, st));
        c->steps_done++;
        return CG_OK;
    }
    const bool sort = (flags & CG_STEP_SORT) != 0;
    const bool relayout = sort && c->n > 1 && (c->sort_steps % c->relayout_every == 0);
    const bool freeze = (flags & CG_STEP_FREEZE) != 0;
    const bool record = (flags & CG_STEP_RECORD) != 0;
    double origin[3];
    int64_t dims64[3];
    int rc;
    // the previous step's readback (bbox, largest displacement, list
    // overflows), then the geometry; event 0 is recorded after it, so the
    // per-phase times are device times
    if (!c->bbox_valid) {
        c->list_valid = false;
        c->last_kind = 0;
        if ((rc = standalone_bbox<T>(c))) return rc;
    } else {
        CUDA_TRY(c, cudaStreamSynchronize(st));
    }
    list_account<T>(c);
    Geometry g;
    if ((rc = host_geometry(c, c->bbox_host, ir, box_cap, g, dims64, origin))) return rc;
    const bool lists_on = c->list_skin != 0.0 && c->sweep_impl == 1 && c->n > 1;
    bool use_list = false;
    if (lists_on && c->list_valid) {
        if (2.0 * c->list_D <= 0.999 * c->list_skin_used && c->nbr_cap == c->cap) {
            use_list = true;
        } else {   // expired: a list that served fewer than 2 steps makes the next builds wait
            c->list_valid = false;
            if (c->list_life < (c->list_width != kListCap ? CG_DENSE_MIN_LIFE : 2)) {
                c->list_backoff = c->list_backoff ? std::min(2 * c->list_backoff, 64) : 4;
                c->list_wait = c->list_backoff;
            } else {
                c->list_backoff = 0;
            }
        }
    }
    if (use_list) {
        if ((rc = list_step_t<T>(c, g, params, sort, freeze, record))) return rc;
        if (sort) {
            c->sort_steps++;
            c->pres_state = PRES_PENDING;
        }
        c->last_kind = 2;
        S.sweep_kind = 2;
    } else {
        bool build = lists_on && c->list_wait == 0;
        if (c->list_wait > 0) c->list_wait--;
        if (build) {
            c->list_skin_used = c->list_skin < 0 ? auto_skin(c, g) : c->list_skin;
            build = c->list_skin_used > 0 && c->list_skin_used <= g.L;
            c->list_width = build ? list_width_for(c, g, c->list_skin_used) : 0;
            build = build && c->list_width > 0;
            // dense pools: no build while the last moving step moved some agent by
            // more than skin / CG_DENSE_LIFE (the lists would not serve
            // CG_DENSE_LIFE / 2 steps)
            if (build && c->list_width != kListCap && !freeze && !c->last_freeze &&
                CG_DENSE_LIFE * std::sqrt(std::max(c->bbox_host[7], 0.0)) > c->list_skin_used)
                build = false;
            if (build && (rc = ensure_lists(c, c->list_width))) return rc;
        }
        if ((rc = build_grid_geo<T>(c, g, relayout, sort))) return rc;
        CUDA_TRY(c, cudaEventRecord(c->ev[slot][2], st));
        if (sort) {
            c->sort_steps++;
            c->pres_state = PRES_PENDING;   // the reference re-sorted its pool this step
        } else if (relayout) {
            c->pres_state = PRES_PENDING;
        }
        if (c->early.want && (rc = early_download<T>(c))) return rc;
        c->list_valid = false;
        if ((rc = run_sweep<T>(c, params, freeze, record, build, true))) return rc;
        c->last_kind = build ? 1 : 0;
        S.sweep_kind = build ? 1 : 0;
        if (build) c->list_builds++;
        if (build) mark_build_sublists(c);
    }
    c->last_freeze = freeze;
    if (!freeze) c->cur_pos = 1 - c->cur_pos;
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][3], st));
    CUDA_TRY(c, cudaMemcpyAsync(c->stat_host + slot * kStatSlots, c->stat_dev + slot * kStatSlots,
                                sizeof(unsigned long long) * kStatSlots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][4], st));
    for (int a = 0; a < 3; ++a) {
        S.grid_dims[a] = dims64[a];
        S.origin[a] = origin[a];
    }
    S.box_length = c->geo.L;
    c->last_record = record;
    c->steps_done++;
    return CG_OK;
}

static int collect(cg_context *c, int64_t step_id, cg_step_stats *out)
{
    if (step_id < 0 || step_id >= c->steps_done || step_id < c->steps_done - kRing)
        return fail(c, CG_ERR_STATE, "stats of step %lld are not available", (long long)step_id);
    const int slot = (int)(step_id % kRing);
    CUDA_TRY(c, cudaEventSynchronize(c->ev[slot][4]));
    cg_step_stats &S = c->ring[slot];
    const unsigned long long *h = c->stat_host + slot * kStatSlots;
    S.grid_occupied_boxes = (int64_t)h[0];
    S.grid_max_occupancy = (int64_t)h[1];
    S.force_evals = (int64_t)h[2];
    S.candidates = (int64_t)h[3];
    S.degenerate_pairs = (int64_t)h[4];
    if (S.agent_count > 0) {
        cudaEventElapsedTime(&S.t_grid_ms, c->ev[slot][0], c->ev[slot][1]);
        cudaEventElapsedTime(&S.t_sort_ms, c->ev[slot][1], c->ev[slot][2]);
        cudaEventElapsedTime(&S.t_force_ms, c->ev[slot][2], c->ev[slot][3]);
        cudaEventElapsedTime(&S.t_total_ms, c->ev[slot][0], c->ev[slot][3]);
    }
    *out = S;
    return CG_OK;
}

// Copy a storage-order device column to the host in the reference's order.
static int download_column(cg_context *c, const void *src, void *dst, size_t w)
{
    const int n = (int)c->n;
    cudaStream_t st = c->stream;
    if (c->pres_state == PRES_IDENTITY) {
        CUDA_TRY(c, cudaMemcpyAsync(dst, src, w * n, cudaMemcpyDeviceToHost, st));
        return CG_OK;
    }
    if (w == 8)
        scatter_by<unsigned long long><<<cdiv(n, kThreads), kThreads, 0, st>>>(
            n, c->b.pres, (const unsigned long long *)src, (unsigned long long *)c->b.stage);
    else
        scatter_by<unsigned><<<cdiv(n, kThreads), kThreads, 0, st>>>(n, c->b.pres, (const unsigned *)src,
                                                                      (unsigned *)c->b.stage);
    LAUNCH_CHECK(c);
    c->launches += 1;
    CUDA_TRY(c, cudaMemcpyAsync(dst, c->b.stage, w * n, cudaMemcpyDeviceToHost, st));
    return CG_OK;
}
