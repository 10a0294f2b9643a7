// host_slab.cuh -- part of the cellgrid_b200.cu translation unit (host side):
// x-slab (multi-GPU) plan / pack / unpack / step, see slab.cuh and distributed.py.
// Included once, in order, by cellgrid_b200.cu; not a standalone header.
#pragma once

// ---------------------------------------------------------------- x-slabs
static int slab_alloc(cg_context *c)
{
    auto &S = c->slab;
    if (S.cap >= c->cap && S.cnt) return CG_OK;
    void *ptrs[] = {S.dest, S.out, S.holes, S.movers, S.cnt, S.counts, S.seg_off, S.cursor};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    const size_t n = (size_t)std::max<int64_t>(c->cap, 1);
    CUDA_TRY(c, cudaMalloc(&S.dest, n));
    int **ints[] = {&S.out, &S.holes, &S.movers};
    for (int **p : ints) CUDA_TRY(c, cudaMalloc(p, sizeof(int) * n));
    CUDA_TRY(c, cudaMalloc(&S.cnt, sizeof(unsigned) * 8));
    CUDA_TRY(c, cudaMalloc(&S.counts, sizeof(unsigned long long) * kHist));
    CUDA_TRY(c, cudaMalloc(&S.seg_off, sizeof(unsigned long long) * kHist));
    CUDA_TRY(c, cudaMalloc(&S.cursor, sizeof(unsigned) * kHist));
    S.cap = c->cap;
    return CG_OK;
}

static int slab_list_alloc(cg_context *c)
{
    auto &S = c->slab;
    if (S.list_cap >= c->cap && S.ref_list) return CG_OK;
    void *ptrs[] = {S.ref_list, S.ref_off, S.r2g, S.mismatch};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    const size_t n = (size_t)std::max<int64_t>(c->cap, 1);
    CUDA_TRY(c, cudaMalloc(&S.ref_list, sizeof(int) * n));
    CUDA_TRY(c, cudaMalloc(&S.ref_off, sizeof(unsigned long long) * kHist));
    CUDA_TRY(c, cudaMalloc(&S.r2g, sizeof(int) * n));
    CUDA_TRY(c, cudaMalloc(&S.mismatch, sizeof(unsigned)));
    CUDA_TRY(c, cudaMemsetAsync(S.mismatch, 0, sizeof(unsigned), c->stream));
    S.list_cap = c->cap;
    return CG_OK;
}

// the ghost table's slots: a power of two >= 2 x ghosts
static int slab_hash_alloc(cg_context *c, int64_t ng)
{
    auto &S = c->slab;
    int64_t h = 1024;
    while (h < 2 * ng) h *= 2;
    if (h > S.hcap) {
        if (S.hkey) cudaFree(S.hkey);
        if (S.hval) cudaFree(S.hval);
        S.hkey = nullptr;
        S.hval = nullptr;
        S.hcap = 0;
        CUDA_TRY(c, cudaMalloc(&S.hkey, sizeof(uint64_t) * (size_t)h));
        CUDA_TRY(c, cudaMalloc(&S.hval, sizeof(int) * (size_t)h));
        S.hcap = h;
    }
    S.hmask = (unsigned)(h - 1);
    CUDA_TRY(c, cudaMemsetAsync(S.hval, 0xff, sizeof(int) * (size_t)h, c->stream));   // -1: empty
    return CG_OK;
}

// every slab index i lives at buffer position i - rot (lo ghosts in the headroom)
template <typename T>
static SlabCols<T> cols_at(cg_context *c, int rot)
{
    SlabCols<T> C;
    C.rec = (Rec<T> *)c->b.rec[c->cur_pos] - rot;
    C.adh = (T *)c->b.adh[c->cur_attr] - rot;
    C.uid = c->b.uid[c->cur_attr] - rot;
    C.dx = (T *)c->b.disp[0] - rot;
    C.dy = (T *)c->b.disp[1] - rot;
    C.dz = (T *)c->b.disp[2] - rot;
    return C;
}

// neighbour-list validity from the all-reduced largest displacement (bb[7],
// squared) and list overflows (bb[8]) of the previous step: every rank takes
// the same decision
template <typename T>
static void slab_list_account(cg_context *c, const double bb[9])
{
    double saved[9];
    for (int k = 0; k < 9; ++k) {
        saved[k] = c->bbox_host[k];
        c->bbox_host[k] = bb[k];
    }
    list_account<T>(c);
    for (int k = 0; k < 9; ++k) c->bbox_host[k] = saved[k];
}

template <typename T>
static SlabCols<T> cur_cols(cg_context *c)
{
    SlabCols<T> C;
    C.rec = (Rec<T> *)c->b.rec[c->cur_pos];
    C.adh = (T *)c->b.adh[c->cur_attr];
    C.uid = c->b.uid[c->cur_attr];
    C.dx = (T *)c->b.disp[0];
    C.dy = (T *)c->b.disp[1];
    C.dz = (T *)c->b.disp[2];
    return C;
}

template <typename T>
static int slab_plan_t(cg_context *c, const double bb[11], double ir, int64_t box_cap, int world, int rank,
                       int64_t *counts, int64_t planes[2])
{
    auto &S = c->slab;
    int rc;
    if ((rc = slab_alloc(c))) return rc;
    Geometry g;
    int64_t dims64[3];
    double origin[3];
    // the box cap bounds each rank's sub-grid (the reference's cap is a
    // per-process memory bound, spatial.py:111-116)
    if ((rc = host_geometry(c, bb, ir, INT64_MAX, g, dims64, origin))) return rc;
    if (g.dimx < world)
        return fail(c, CG_ERR_VALUE, "grid of %d x-planes is too narrow for %d slabs", g.dimx, world);
    const bool lists_on = c->list_skin != 0.0 && c->sweep_impl == 1 && world == S.world && rank == S.rank;
    if (lists_on) slab_list_account<T>(c, bb);
    S.list_mode = lists_on && c->list_valid && S.refresh_ready && c->nbr_cap == c->cap &&
                  2.0 * c->list_D <= 0.999 * c->list_skin_used;
    // the global diameter range: every agent a rank holds (owned, arrived or a
    // ghost) lies in it, so min == max is a uniform pool everywhere
    c->max_diam = std::max(c->max_diam, bb[6]);
    c->min_diam = std::isfinite(bb[9]) ? -bb[9] : -INFINITY;
    S.unpacked = false;
    S.g = g;
    if (S.list_mode) {
        // frozen partition: the owners refresh the ghosts they hold in other ranks' bands
        for (int k = 0; k < 3 * world; ++k) counts[k] = (k % 3 == 0) ? 0 : S.ref_counts[k];
        planes[0] = S.x0;
        planes[1] = S.x1;
        S.planned = true;
        S.packed = false;
        S.interior_done = false;
        return CG_OK;
    }
    if (c->list_valid && lists_on) {   // expired lists: the same backoff rule as a single context
        c->list_valid = false;
        if (c->list_life < 2) {
            c->list_backoff = c->list_backoff ? std::min(2 * c->list_backoff, 64) : 4;
            c->list_wait = c->list_backoff;
        } else {
            c->list_backoff = 0;
        }
    }
    // a rebuild: the ghosts kept by list steps are dropped
    c->n = c->n_owned;
    S.refresh_ready = false;
    c->list_valid = false;
    S.world = world;
    S.rank = rank;
    S.B.world = world;
    S.B.band = c->list_skin != 0.0 && c->sweep_impl == 1 ? 3 : 1;
    for (int k = 0; k <= world; ++k) S.B.x[k] = (int)(((int64_t)k * g.dimx) / world);
    S.x0 = S.B.x[rank];
    S.x1 = S.B.x[rank + 1];
    {
        const int64_t sub = (int64_t)(std::min(S.x1 + S.B.band, g.dimx) - std::max(S.x0 - S.B.band, 0)) * g.dimy *
                            g.dimz;
        if (sub > box_cap)
            return fail(c, CG_ERR_GRID_OVERFLOW, "slab sub-grid of %lld boxes exceeds cap %lld",
                        (long long)sub, (long long)box_cap);
    }
    // every candidate radius is bounded by the global largest diameter;
    // arrivals and ghosts bring uids this context has not seen
    // arrivals and ghosts bring uids this context has not seen: the global max
    c->uid32 = bb[10] < 4294967296.0;
    planes[0] = S.x0;
    planes[1] = S.x1;
    cudaStream_t st = c->stream;
    CUDA_TRY(c, cudaMemsetAsync(S.counts, 0, sizeof(unsigned long long) * kHist, st));
    const int n = (int)c->n_owned;
    if (n > 0) {
        slab_dest<T><<<std::min(cdiv(n, kThreads), c->sms * 8), kThreads, 0, st>>>(
            n, g, S.B, rank, (const Rec<T> *)c->b.rec[c->cur_pos], S.dest, S.counts);
        LAUNCH_CHECK(c);
        c->launches += 1;
    }
    unsigned long long h[kHist];
    CUDA_TRY(c, cudaMemcpyAsync(h, S.counts, sizeof(unsigned long long) * (3 * world + 1), cudaMemcpyDeviceToHost,
                                st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    for (int k = 0; k <= 3 * world; ++k) S.h_counts[k] = (int64_t)h[k];
    for (int k = 0; k < 3 * world; ++k) counts[k] = S.h_counts[k];
    S.planned = true;
    S.packed = false;
    S.interior_done = false;
    return CG_OK;
}

template <typename T>
static int slab_pack_t(cg_context *c, void *send)
{
    auto &S = c->slab;
    if (S.list_mode) {   // refresh records of the owned agents in other ranks' bands, in run order
        S.packed = true;
        if (S.ref_total > 0) {
            slab_refresh_pack<T><<<cdiv(S.ref_total, kThreads), kThreads, 0, c->stream>>>(
                (int)S.ref_total, S.ref_list, cols_at<T>(c, S.rot_build), (SlabRecord<T> *)send);
            LAUNCH_CHECK(c);
            c->launches += 1;
        }
        return CG_OK;   // the exchange is ordered after the pack on the context stream
    }
    const int n = (int)c->n_owned;
    const int W = S.world;
    const int n_keep = (int)S.h_counts[3 * W];
    unsigned long long off[kHist];
    unsigned long long acc = 0;
    for (int k = 0; k < 3 * W; ++k) {
        off[k] = acc;
        acc += (unsigned long long)S.h_counts[k];
    }
    S.packed = true;
    if (acc == 0 && n_keep == n) return CG_OK;
    cudaStream_t st = c->stream;
    CUDA_TRY(c, cudaMemcpyAsync(S.seg_off, off, sizeof(unsigned long long) * 3 * W, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemsetAsync(S.cursor, 0, sizeof(unsigned) * 3 * W, st));
    CUDA_TRY(c, cudaMemsetAsync(S.cnt, 0, sizeof(unsigned) * 8, st));
    slab_lists<<<cdiv(n, kThreads), kThreads, 0, st>>>(n, n_keep, S.rank, S.dest, S.out, S.holes, S.movers, S.cnt);
    unsigned hc[3];
    CUDA_TRY(c, cudaMemcpyAsync(hc, S.cnt, sizeof hc, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    const SlabCols<T> C = cur_cols<T>(c);
    if (hc[0])
        slab_pack_out<T><<<cdiv(hc[0], kThreads), kThreads, 0, st>>>((int)hc[0], S.rank, S.g, S.B, S.out, S.dest,
                                                                     S.seg_off, S.cursor, C, (SlabRecord<T> *)send);
    if (hc[1])
        slab_fill_holes<T><<<cdiv(hc[1], kThreads), kThreads, 0, st>>>((int)hc[1], S.holes, S.movers, C);
    LAUNCH_CHECK(c);
    c->launches += 3;
    c->n = c->n_owned = n_keep;   // the exchange is ordered after the pack on the context stream
    c->bbox_valid = false;
    return CG_OK;
}

template <typename T>
static int slab_unpack_t(cg_context *c, const void *recv, const int64_t *rc3)
{
    auto &S = c->slab;
    const int W = S.world;
    S.unpacked = true;
    if (S.list_mode) {
        int64_t got = 0;
        for (int k = 0; k < 3 * W; ++k) {
            if (rc3[k] < 0 || (k % 3 == 0 && rc3[k] != 0))
                return fail(c, CG_ERR_STATE, "unexpected migrants in a ghost-refresh step");
            got += rc3[k];
        }
        const int64_t ng = S.n_total - c->n_owned;
        if (got != ng)
            return fail(c, CG_ERR_STATE, "ghost refresh brought %lld records for %lld ghosts", (long long)got,
                        (long long)ng);
        if (ng == 0) return CG_OK;
        // the runs arrive in the same order all epoch: match by uid once, then
        // scatter through r2g; a record without its ghost counts in
        // S.mismatch, checked with the next bbox readback (no sync here)
        cudaStream_t st = c->stream;
        Rec<T> *rec = (Rec<T> *)c->b.rec[c->cur_pos] - S.rot_build;
        if (!S.r2g_valid) {
            slab_refresh_match<T><<<cdiv(ng, kThreads), kThreads, 0, st>>>(
                (int)ng, (const SlabRecord<T> *)recv, S.hkey, S.hval, S.hmask, S.r2g, rec, S.mismatch);
            S.r2g_valid = true;
        } else {
            slab_refresh_apply<T><<<cdiv(ng, kThreads), kThreads, 0, st>>>(
                (int)ng, (const SlabRecord<T> *)recv, S.r2g, cols_at<T>(c, S.rot_build).uid, rec, S.mismatch);
        }
        LAUNCH_CHECK(c);
        c->launches += 1;
        return CG_OK;
    }
    int64_t mig = 0, glo = 0, ghi = 0;
    for (int s = 0; s < W; ++s) {
        if (rc3[3 * s] < 0 || rc3[3 * s + 1] < 0 || rc3[3 * s + 2] < 0)
            return fail(c, CG_ERR_VALUE, "negative receive count");
        mig += rc3[3 * s];
        glo += rc3[3 * s + 1];
        ghi += rc3[3 * s + 2];
    }
    const int64_t base = c->n_owned, total = mig + glo + ghi;
    if (base + total > c->cap)
        return fail(c, CG_ERR_POOL_CAPACITY, "slab needs %lld agents, capacity %lld (cg_reserve)",
                    (long long)(base + total), (long long)c->cap);
    // destination of every run: migrants after the owned set, then lo ghosts, then hi ghosts
    SlabSegs G{};
    int64_t pos = 0, dm = base, dl = base + mig, dh = base + mig + glo;
    for (int s = 0; s < W; ++s)
        for (int kind = 0; kind < 3; ++kind) {
            const int k = 3 * s + kind;
            G.start[k] = pos;
            const int64_t cnt = rc3[k];
            int64_t &d = kind == 0 ? dm : kind == 1 ? dl : dh;
            G.dst[k] = (int)d;
            d += cnt;
            pos += cnt;
        }
    G.nseg = 3 * W;
    G.start[3 * W] = pos;
    if (total > 0) {
        cudaStream_t st = c->stream;
        slab_unpack_segs<T><<<cdiv(total, kThreads), kThreads, 0, st>>>((int)total, G, (const SlabRecord<T> *)recv,
                                                                        cur_cols<T>(c));
        LAUNCH_CHECK(c);
        c->launches += 1;
    }
    c->n_owned = base + mig;
    c->n = base + total;
    if (mig) c->bbox_valid = false;
    S.ghost_lo = glo;
    return CG_OK;
}

// After a rebuild step with lists: the ghost table (ghost indices sorted by
// uid) and the refresh lists (owned agents in other ranks' bands, by run).
template <typename T>
static int slab_list_tables(cg_context *c)
{
    auto &S = c->slab;
    int rc;
    if ((rc = slab_list_alloc(c))) return rc;
    cudaStream_t st = c->stream;
    const int W = S.world, lo = c->rot, no = (int)c->n_owned, nt = (int)c->n;
    const int ng = nt - no;
    const SlabCols<T> C = cols_at<T>(c, lo);   // the build positions (before this step's move)
    S.r2g_valid = false;
    if (ng > 0) {
        if ((rc = slab_hash_alloc(c, ng))) return rc;
        slab_ghost_hash<<<cdiv(ng, kThreads), kThreads, 0, st>>>(nt, lo, no, C.uid, S.hkey, S.hval, S.hmask);
    }
    CUDA_TRY(c, cudaMemsetAsync(S.counts, 0, sizeof(unsigned long long) * kHist, st));
    if (no > 0)
        slab_refresh_lists<T, false><<<cdiv(no, kThreads), kThreads, 0, st>>>(no, lo, S.g, S.B, C.rec, S.counts,
                                                                              nullptr, nullptr, nullptr);
    unsigned long long h[kHist];
    CUDA_TRY(c, cudaMemcpyAsync(h, S.counts, sizeof(unsigned long long) * 3 * W, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    unsigned long long off[kHist], acc = 0;
    for (int k = 0; k < 3 * W; ++k) {
        off[k] = acc;
        S.ref_counts[k] = (int64_t)h[k];
        acc += h[k];
    }
    S.ref_total = (int64_t)acc;
    if (acc > 0) {
        CUDA_TRY(c, cudaMemcpyAsync(S.ref_off, off, sizeof(unsigned long long) * 3 * W, cudaMemcpyHostToDevice, st));
        CUDA_TRY(c, cudaMemsetAsync(S.cursor, 0, sizeof(unsigned) * kHist, st));
        slab_refresh_lists<T, true><<<cdiv(no, kThreads), kThreads, 0, st>>>(no, lo, S.g, S.B, C.rec, nullptr,
                                                                             S.ref_off, S.cursor, S.ref_list);
    }
    LAUNCH_CHECK(c);
    c->launches += 3;
    S.n_total = nt;
    S.rot_build = lo;
    S.x_lo_abs = S.g.ox + (double)S.x0 * S.g.L;
    S.x_hi_abs = S.g.ox + (double)S.x1 * S.g.L;
    S.refresh_ready = true;
    // interior rows: with relaid storage the owned rows are the build's slots
    // in plane order, so the boundary rows (build planes within 3 of a slab
    // face -- list partners are within ri + rj + skin <= 2L) are the two ends
    S.split_ok = false;
    S.b_lo = no;
    S.b_hi = 0;
    const Geometry &gb = c->geo;
    if (c->relaid && no > 0 && S.x1 - S.x0 >= 7 && gb.xoff <= S.x0) {
        const int64_t P = (int64_t)gb.dimy * gb.dimz;
        const int64_t at[4] = {(S.x0 - gb.xoff) * P, (S.x0 + 3 - gb.xoff) * P, (S.x1 - 3 - gb.xoff) * P,
                               (S.x1 - gb.xoff) * P};
        int h[4];
        for (int k = 0; k < 4; ++k)
            CUDA_TRY(c, cudaMemcpyAsync(h + k, c->offset + at[k], sizeof(int), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(c, cudaStreamSynchronize(st));
        if (h[0] == lo && h[3] == lo + no && h[0] <= h[1] && h[1] <= h[2] && h[2] <= h[3]) {
            S.b_lo = h[1] - h[0];
            S.b_hi = h[3] - h[2];
            S.split_ok = true;
        }
    }
    return CG_OK;
}

// a list step on a slab: grid counts over owned + ghosts, list sweep of the
// owned agents (indices [rot, rot + n_owned), buffers at index - rot).
// part 1 (cg_slab_step_interior, before the ghost refresh is unpacked): set-up
// and the sweep of the interior rows; part 2 (cg_slab_step): the rest -- all
// rows, or only the boundary rows when part 1 ran.
template <typename T>
static int slab_list_step(cg_context *c, const double params[5], bool freeze, bool record, int part)
{
    auto &S = c->slab;
    const int slot = (int)(c->steps_done % kRing);
    cudaStream_t st = c->stream;
    const int rot = S.rot_build, nt = (int)S.n_total, no = (int)c->n_owned;
    const bool fused = !record;   // box counting inside the list sweep (owned) + count_ghosts
    int rc;
    if (part == 1 || !S.interior_done) {
        // sub-grid: every present agent lies within 3 box lengths (+ the motion
        // since the rebuild) of the owned slab's x range at the rebuild
        Geometry g = S.g;
        const auto plane = [&](double x) {
            return (int)std::min<double>(std::max<double>(std::floor((x - S.g.ox) / S.g.L), 0.0), S.g.dimx - 1.0);
        };
        const int xl = plane(S.x_lo_abs - 4.0 * S.g.L), xh = plane(S.x_hi_abs + 4.0 * S.g.L) + 1;
        g.xoff = xl;
        g.gdimx = S.g.dimx;
        g.dimx = std::max(xh - xl, 1);
        g.nb = g.dimx * g.dimy * g.dimz;
        CUDA_TRY(c, cudaEventRecord(c->ev[slot][0], st));
        if ((rc = ensure_boxes(c, g.nb))) return rc;
        c->geo = g;
        c->bd = make_decode(g);
        CUDA_TRY(c, cudaMemsetAsync(c->stat_dev + slot * kStatSlots, 0, sizeof(unsigned long long) * kStatSlots, st));
    }
    const Geometry g = c->geo;
    unsigned long long *stat = c->stat_dev + slot * kStatSlots;
    const int cp = c->cur_pos, ca = c->cur_attr;
    ListArgs<T> A{};
    A.skip_at = INT_MAX;
    A.g = g;
    A.bd = c->bd;
    A.key_rank = c->b.key_rank;
    A.off = c->offset;
    A.rec = (const Rec<T> *)c->b.rec[cp] - rot;
    A.adh = (const T *)c->b.adh[ca] - rot;
    A.uid = c->b.uid[ca] - rot;
    A.p = make_params<T>(params);
    A.nbr = c->nbr;
    A.nbr_n = c->nbr_n;
    A.nbr_stride = c->nbr_cap;
    // the sub-lists (choose_levels), chosen once per step for both parts
    if (part == 1 || !S.interior_done) choose_levels(c, fused, S.read_lvl, S.write_lvl);
    apply_levels<T>(c, A, S.read_lvl, S.write_lvl);
    A.disp_x = (T *)c->b.disp[0] - rot;
    A.disp_y = (T *)c->b.disp[1] - rot;
    A.disp_z = (T *)c->b.disp[2] - rot;
    A.new_rec = freeze ? nullptr : (Rec<T> *)c->b.rec[1 - cp] - rot;
    A.rec_m = record ? c->b.rec_m - rot : nullptr;
    A.rec_nk = record ? c->b.rec_nk - rot : nullptr;
    A.pkey = nullptr;
    A.count = c->count;
    A.count_own = nullptr;
    A.invL = 1.0 / g.L;
    A.slots = c->slots;
    bbox_shell(c, (double)A.p.max_disp, A.shell_lo, A.shell_hi);
    const int n_int = no - S.b_lo - S.b_hi;
    if (part == 1) {   // interior rows: their lists hold no ghost
        if (n_int > 0) {
            A.n = n_int;
            A.own_lo = rot + S.b_lo;
            launch_list_sweep<T>(c, A, n_int, true, st);
            LAUNCH_CHECK(c);
            c->launches += 1;
        }
        S.interior_done = true;
        c->overlapped_steps++;
        return CG_OK;
    }
    if (!fused) {
        box_keys<T><<<cdiv(nt, kThreads), kThreads, 0, st>>>(nt, g, 1.0 / g.L, (const Rec<T> *)c->b.rec[cp] - rot,
                                                             c->count, c->b.key_rank);
        LAUNCH_CHECK(c);
        c->launches += 1;
        if ((rc = launch_scan_rts(c, g.nb, stat))) return rc;
    } else if (nt > no) {
        count_ghosts<T><<<cdiv(nt - no, kThreads), kThreads, 0, st>>>(nt, rot, no, g, 1.0 / g.L,
                                                                       (const Rec<T> *)c->b.rec[cp] - rot, c->count,
                                                                       c->count_own);
        LAUNCH_CHECK(c);
        c->launches += 1;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][1], st));
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][2], st));
    A.own_lo = rot;
    A.n = no;
    if (S.interior_done) {   // the boundary rows: [0, b_lo) and [no - b_hi, no)
        A.n = S.b_lo + S.b_hi;
        A.skip_at = S.b_lo;
        A.skip = n_int;
    }
    if (A.n > 0) {
        launch_list_sweep<T>(c, A, A.n, fused, st);
        LAUNCH_CHECK(c);
        c->launches += 1;
    }
    if (fused) {
        const int gb = std::min(cdiv(g.nb, kThreads), c->sms * CG_BOX_GRID);
        box_sum_yz<<<gb, kThreads, 0, st>>>(g, c->bd, c->count, c->offset);
        box_stencil_pass<<<gb, kThreads, 0, st>>>(g, c->bd, c->count, c->count_own, c->offset, c->slots, stat);
        LAUNCH_CHECK(c);
        c->launches += 2;
    }
    finish_step<<<1, kThreads, 0, st>>>(c->slots, c->max_diam, stat, c->bbox_dev,
                                         FINISH_COUNTERS | (freeze ? 0 : FINISH_BBOX));
    LAUNCH_CHECK(c);
    c->launches += 1;
    if (!freeze)
        CUDA_TRY(c, cudaMemcpyAsync(c->bbox_host, c->bbox_dev, 9 * sizeof(double), cudaMemcpyDeviceToHost, st));
    c->bbox_valid = true;
    c->relaid = false;
    c->last_dense = false;
    c->list_life++;
    c->list_steps++;
    return CG_OK;
}

template <typename T>
static int slab_step_t(cg_context *c, const double params[5], int flags, int64_t *step_id)
{
    auto &S = c->slab;
    if (!S.planned || !S.packed) return fail(c, CG_ERR_STATE, "cg_slab_step without cg_slab_plan / cg_slab_pack");
    const int slot = (int)(c->steps_done % kRing);
    cg_step_stats &St = c->ring[slot];
    std::memset(&St, 0, sizeof St);
    St.step_id = c->steps_done;
    St.agent_count = c->n_owned;
    *step_id = c->steps_done;
    cudaStream_t st = c->stream;
    int rc;
    const bool freeze = (flags & CG_STEP_FREEZE) != 0;
    const bool record = (flags & CG_STEP_RECORD) != 0;
    if (S.list_mode) {
        if ((rc = slab_list_step<T>(c, params, freeze, record, 2))) return rc;
        S.interior_done = false;
        if (!freeze) c->cur_pos = 1 - c->cur_pos;
        c->last_kind = 2;
        St.sweep_kind = 2;
    } else {
        c->list_valid = false;
        // exact bbox of the owned set (the sweep's shell filter needs it)
        if (!c->bbox_valid && c->n_owned > 0 && (rc = standalone_bbox<T>(c))) return rc;
        // sub-grid: global planes [x0 - band, x1 + band) clipped to the grid
        Geometry g = S.g;
        const int xl = std::max(S.x0 - S.B.band, 0), xh = std::min(S.x1 + S.B.band, S.g.dimx);
        g.xoff = xl;
        g.gdimx = S.g.dimx;
        g.dimx = std::max(xh - xl, 1);
        g.nb = g.dimx * g.dimy * g.dimz;
        bool build = false;
        if (c->n > 0) {
            // relaid storage as in the single-context step; the owned planes are
            // the middle slot range, rotated to the front by the lo-ghost count
            const bool relayout = c->sweep_impl == 1 && c->n > 1 && (S.steps % c->relayout_every == 0);
            const int rot = (int)S.ghost_lo;
            if ((rc = build_grid_geo<T>(c, g, relayout && rot <= c->b.head, false, rot))) return rc;
            S.steps++;
            CUDA_TRY(c, cudaEventRecord(c->ev[slot][2], st));
            build = S.B.band == 3 && c->list_wait == 0 && !c->last_dense;
            if (c->list_wait > 0) c->list_wait--;
            if (build) {
                if ((rc = ensure_lists(c, kListCap))) return rc;
                c->list_width = kListCap;
                c->list_skin_used = c->list_skin < 0 ? 0.26 * S.g.L : c->list_skin;   // slab lists are 48 wide
                build = c->list_skin_used > 0 && c->list_skin_used <= S.g.L;
            }
            if ((rc = run_sweep<T>(c, params, freeze, record, build, true))) return rc;
            if (build) {
                if ((rc = slab_list_tables<T>(c))) return rc;
                c->list_builds++;
                mark_build_sublists(c);
            }
            if (!freeze) c->cur_pos = 1 - c->cur_pos;
        } else {
            CUDA_TRY(c, cudaMemsetAsync(c->stat_dev + slot * kStatSlots, 0, sizeof(unsigned long long) * kStatSlots,
                                        st));
            for (int e = 0; e < 3; ++e) CUDA_TRY(c, cudaEventRecord(c->ev[slot][e], st));
            c->bbox_valid = false;
        }
        if (!build) c->n = c->n_owned;   // this step's ghosts are dropped (list steps keep them)
        c->last_kind = build ? 1 : 0;
        St.sweep_kind = build ? 1 : 0;
    }
    c->last_freeze = freeze;
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][3], st));
    CUDA_TRY(c, cudaMemcpyAsync(c->stat_host + slot * kStatSlots, c->stat_dev + slot * kStatSlots,
                                sizeof(unsigned long long) * kStatSlots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][4], st));
    St.grid_dims[0] = S.g.dimx;
    St.grid_dims[1] = S.g.dimy;
    St.grid_dims[2] = S.g.dimz;
    St.origin[0] = S.g.ox;
    St.origin[1] = S.g.oy;
    St.origin[2] = S.g.oz;
    St.box_length = S.g.L;
    c->last_record = record;
    c->have_grid = false;   // the sub-grid is not exportable
    c->pres_state = PRES_IDENTITY;
    c->steps_done++;
    S.planned = S.packed = false;
    return CG_OK;
}
