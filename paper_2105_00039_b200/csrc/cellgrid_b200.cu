// cellgrid_b200.cu -- context, step orchestration and the C ABI
// (include/cellgrid_b200.h).
//
// One context = one agent population resident in the HBM of one B200.  A step
// (reference engine.py:279-341) is:
//   K1 bbox -> host geometry (spatial.py:99-116, bit-exact f64) -> [K5 Morton
//   table if dims changed] -> K2 box keys + warp-aggregated counts -> K3 scan ->
//   K4 place + uid order -> [K4b gather when the Z-order sort is due] ->
//   sweep (force, gate, cap, apply) -> counter reduction.
// The only host round trip is the 7-double bbox readback (needed to size the
// grid and to raise GridOverflowError before anything is modified, exactly
// where the reference raises).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/cellgrid_b200.h"
#include "common.cuh"
#include "grid.cuh"
#include "sweep.cuh"
#include "sweep_tile.cuh"
#include "sweep_proxy.cuh"

using namespace cg;

namespace {

constexpr int kStatSlots = 8;        // per step: occupied, maxocc, evals, cands, ndeg
constexpr int kRing = 64;            // pinned stats ring (steps in flight)
constexpr int kBboxBlocks = 148 * 4; // grid-stride bbox reduction: 4 CTAs per SM

struct Buffers {
    void *pos[2][3] = {{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
    void *dia[2] = {nullptr, nullptr};
    void *adh[2] = {nullptr, nullptr};
    uint64_t *uid[2] = {nullptr, nullptr};
    void *disp[3] = {nullptr, nullptr, nullptr};
    int *key = nullptr, *rnk = nullptr, *tmp = nullptr, *idx = nullptr, *skey = nullptr;
    float4 *prox = nullptr;
    int *rec_m = nullptr, *rec_nk = nullptr;
    unsigned long long *block_counters = nullptr;
};

}  // namespace

struct cg_context {
    int device = 0;
    int prec = CG_FP64;
    size_t esz = 8;
    cudaStream_t stream = nullptr;
    int64_t n = 0, cap = 0;
    Buffers b;
    int cur_pos = 0, cur_attr = 0;
    // grid
    int64_t box_cap = 0;                 // allocated box capacity
    int *count = nullptr, *offset = nullptr, *tile_sum = nullptr, *mrank = nullptr, *minv = nullptr;
    int table_dims[3] = {0, 0, 0};
    int64_t blockctr_cap = 0;
    double *bbox_partial = nullptr, *bbox_dev = nullptr;
    double *bbox_host = nullptr;         // pinned
    unsigned long long *stat_dev = nullptr;   // kRing * kStatSlots
    unsigned long long *stat_host = nullptr;  // pinned mirror
    cg_step_stats ring[kRing];
    cudaEvent_t ev[kRing][5];
    int64_t steps_done = 0;
    int64_t launches = 0;                // kernels launched by this context
    // last step
    bool have_grid = false, last_sorted = false, last_record = false;
    Geometry geo{};
    bool morton = true;
    int summation = SUM_UID;
    int sweep_impl = 2;                  // 0 = thread per agent, 1 = smem tiles, 2 = proxy (default)
    int tile_cap = 2048;                 // staged agents per CTA
    int debug_stop = 0;
    std::string err;
};

static int fail(cg_context *c, int code, const char *fmt, ...)
{
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CUDA_TRY(ctx, expr)                                                                      \
    do {                                                                                         \
        cudaError_t e_ = (expr);                                                                 \
        if (e_ != cudaSuccess)                                                                   \
            return fail(ctx, CG_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), \
                        __FILE__, __LINE__);                                                     \
    } while (0)

#define LAUNCH_CHECK(ctx) CUDA_TRY(ctx, cudaGetLastError())

static void free_agents(cg_context *c)
{
    Buffers &b = c->b;
    void *ptrs[] = {b.pos[0][0], b.pos[0][1], b.pos[0][2], b.pos[1][0], b.pos[1][1], b.pos[1][2],
                    b.dia[0], b.dia[1], b.adh[0], b.adh[1], b.uid[0], b.uid[1],
                    b.disp[0], b.disp[1], b.disp[2], b.key, b.rnk, b.tmp, b.idx, b.skey,
                    b.rec_m, b.rec_nk, b.prox};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    unsigned long long *bc = b.block_counters;   // sized by launch shape, not by n: keep
    c->b = Buffers{};
    c->b.block_counters = bc;
    c->cap = 0;
}

static int alloc_agents(cg_context *c, int64_t cap)
{
    free_agents(c);
    Buffers &b = c->b;
    const size_t fe = c->esz * (size_t)cap, ie = sizeof(int) * (size_t)cap;
    for (int k = 0; k < 2; ++k) {
        for (int a = 0; a < 3; ++a) CUDA_TRY(c, cudaMalloc(&b.pos[k][a], fe));
        CUDA_TRY(c, cudaMalloc(&b.dia[k], fe));
        CUDA_TRY(c, cudaMalloc(&b.adh[k], fe));
        CUDA_TRY(c, cudaMalloc(&b.uid[k], sizeof(uint64_t) * (size_t)cap));
    }
    for (int a = 0; a < 3; ++a) CUDA_TRY(c, cudaMalloc(&b.disp[a], fe));
    int **ints[] = {&b.key, &b.rnk, &b.tmp, &b.idx, &b.skey, &b.rec_m, &b.rec_nk};
    for (int **p : ints) CUDA_TRY(c, cudaMalloc(p, ie));
    CUDA_TRY(c, cudaMalloc(&b.prox, sizeof(float4) * (size_t)cap));
    c->cap = cap;
    return CG_OK;
}

static int ensure_boxes(cg_context *c, int64_t nb)
{
    if (nb <= c->box_cap) return CG_OK;
    int64_t want = nb + nb / 4 + 1024;
    int *ptrs[] = {c->count, c->offset, c->tile_sum, c->mrank, c->minv};
    for (int *p : ptrs)
        if (p) cudaFree(p);
    CUDA_TRY(c, cudaMalloc(&c->count, sizeof(int) * want));
    CUDA_TRY(c, cudaMalloc(&c->offset, sizeof(int) * (want + 1)));
    CUDA_TRY(c, cudaMalloc(&c->tile_sum, sizeof(int) * (cdiv(want, kScanTile) + 1)));
    CUDA_TRY(c, cudaMalloc(&c->mrank, sizeof(int) * want));
    CUDA_TRY(c, cudaMalloc(&c->minv, sizeof(int) * want));
    c->box_cap = want;
    c->table_dims[0] = c->table_dims[1] = c->table_dims[2] = 0;
    return CG_OK;
}

static int ensure_block_counters(cg_context *c, int64_t nblocks)
{
    if (nblocks <= c->blockctr_cap) return CG_OK;
    if (c->b.block_counters) cudaFree(c->b.block_counters);
    CUDA_TRY(c, cudaMalloc(&c->b.block_counters, sizeof(unsigned long long) * 3 * nblocks));
    c->blockctr_cap = nblocks;
    return CG_OK;
}

// spatial.py:99-116 on the host, from the device bbox (exact f64 arithmetic).
static int host_geometry(cg_context *c, const double bb[7], double ir, int64_t box_cap,
                         Geometry &g, int64_t dims64[3], double origin[3])
{
    double L = bb[6];
    if (!std::isnan(ir)) {
        if (!(ir > 0)) return fail(c, CG_ERR_VALUE, "interaction_radius must be positive, got %g", ir);
        if (ir > L) L = ir;
    }
    int64_t nb = 1;
    for (int a = 0; a < 3; ++a) {
        origin[a] = bb[a] - L;
        const double q = std::floor((bb[3 + a] - bb[a]) / L);
        dims64[a] = (int64_t)q + 3;
        nb *= dims64[a];
    }
    if (nb > box_cap)
        return fail(c, CG_ERR_GRID_OVERFLOW,
                    "grid of %lld x %lld x %lld = %lld boxes exceeds cap %lld; population too "
                    "sparse for box_length %g",
                    (long long)dims64[0], (long long)dims64[1], (long long)dims64[2],
                    (long long)nb, (long long)box_cap, L);
    if (nb >= (int64_t)INT32_MAX)
        return fail(c, CG_ERR_GRID_OVERFLOW, "grid of %lld boxes exceeds the int32 box index range",
                    (long long)nb);
    g.L = L;
    g.ox = origin[0];
    g.oy = origin[1];
    g.oz = origin[2];
    g.dimx = (int)dims64[0];
    g.dimy = (int)dims64[1];
    g.dimz = (int)dims64[2];
    g.nb = (int)nb;
    return CG_OK;
}

template <typename T>
static Params<T> make_params(const double p[5])
{
    Params<T> q;
    q.kappa = (T)p[0];
    q.gamma = (T)p[1];
    q.timestep = (T)p[2];
    q.max_disp = (T)p[3];
    q.adh_scale = (T)p[4];
    q.zero = (T)0;
    return q;
}

// Grid build (K1..K4) on the current storage: leaves count/offset/key/rnk/idx/skey.
template <typename T>
static int build_grid(cg_context *c, double ir, int64_t box_cap, double origin[3], int64_t dims64[3])
{
    const int n = (int)c->n;
    cudaStream_t st = c->stream;
    T *x = (T *)c->b.pos[c->cur_pos][0], *y = (T *)c->b.pos[c->cur_pos][1],
      *z = (T *)c->b.pos[c->cur_pos][2], *d = (T *)c->b.dia[c->cur_attr];
    const int nbb = std::min(kBboxBlocks, cdiv(n, kThreads));
    bbox_partial<T><<<nbb, kThreads, 0, st>>>(n, x, y, z, d, c->bbox_partial);
    bbox_final<<<1, 32, 0, st>>>(nbb, c->bbox_partial, c->bbox_dev);
    LAUNCH_CHECK(c);
    c->launches += 2;
    CUDA_TRY(c, cudaMemcpyAsync(c->bbox_host, c->bbox_dev, 7 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    Geometry g;
    int rc = host_geometry(c, c->bbox_host, ir, box_cap, g, dims64, origin);
    if (rc) return rc;
    if ((rc = ensure_boxes(c, g.nb))) return rc;
    c->geo = g;
    if (c->morton && (c->table_dims[0] != g.dimx || c->table_dims[1] != g.dimy ||
                      c->table_dims[2] != g.dimz)) {
        morton_table<<<std::min(cdiv(g.nb, kThreads), 148 * 16), kThreads, 0, st>>>(g, c->mrank, c->minv);
        LAUNCH_CHECK(c);
        c->launches += 1;
        c->table_dims[0] = g.dimx;
        c->table_dims[1] = g.dimy;
        c->table_dims[2] = g.dimz;
    }
    CUDA_TRY(c, cudaMemsetAsync(c->count, 0, sizeof(int) * g.nb, st));
    const int nblk = cdiv(n, kThreads);
    box_keys<T><<<nblk, kThreads, 0, st>>>(n, g, x, y, z, c->morton ? c->mrank : nullptr, c->count,
                                           c->b.key, c->b.rnk);
    const int ntiles = cdiv(g.nb, kScanTile);
    unsigned long long *stat = c->stat_dev + (c->steps_done % kRing) * kStatSlots;
    CUDA_TRY(c, cudaMemsetAsync(stat, 0, sizeof(unsigned long long) * kStatSlots, st));
    scan_tiles<<<ntiles, kThreads, 0, st>>>(g.nb, c->count, c->offset, c->tile_sum, stat);
    scan_tile_sums<<<1, kThreads, 0, st>>>(ntiles, c->tile_sum);
    scan_add<<<cdiv(g.nb, kThreads), kThreads, 0, st>>>(g.nb, n, c->tile_sum, c->offset);
    place<<<nblk, kThreads, 0, st>>>(n, c->b.key, c->b.rnk, c->offset, c->b.tmp);
    if (c->morton)
        order_in_box<T, false><<<nblk, kThreads, 0, st>>>(n, c->b.tmp, c->b.key, c->offset,
                                                          c->b.uid[c->cur_attr], z, c->b.idx, c->b.skey);
    else
        order_in_box<T, true><<<nblk, kThreads, 0, st>>>(n, c->b.tmp, c->b.key, c->offset,
                                                         c->b.uid[c->cur_attr], z, c->b.idx, c->b.skey);
    LAUNCH_CHECK(c);
    c->launches += 6;
    return CG_OK;
}

// Pick the tile shape: largest core block whose expected halo population fits
// comfortably in the staging capacity (overflowing tiles fall back to global
// reads, so this only affects speed).
static TileShape choose_tiles(const Geometry &g, int64_t n, int cap)
{
    const double rho = (double)n / (double)g.nb;
    const int menu_xy[][2] = {{1, 1}, {1, 2}, {2, 2}, {2, 4}, {4, 4}, {4, 8}, {8, 8}};
    const int menu_z[] = {4, 8, 16, 32};
    TileShape best{1, 1, 4, 0, 0, 0, cap, 0, 0};
    double best_core = -1.0;
    for (auto &xy : menu_xy)
        for (int tz : menu_z) {
            const int tx = xy[0], ty = xy[1];
            const int halo_boxes = (tx + 2) * (ty + 2) * (tz + 2);
            if (halo_boxes > 1200) continue;
            const double halo = rho * halo_boxes, core = rho * tx * ty * tz;
            if (halo > 0.45 * cap) continue;
            // prefer ~256-768 core agents; beyond that larger tiles add nothing
            const double score = std::min(core, 768.0) + 1e-3 * core / halo;
            if (score > best_core) {
                best_core = score;
                best = TileShape{tx, ty, tz, 0, 0, 0, cap, halo_boxes, 0};
            }
        }
    best.ntx = cdiv(g.dimx, best.tx);
    best.nty = cdiv(g.dimy, best.ty);
    best.ntz = cdiv(g.dimz, best.tz);
    best.max_halo_boxes = (best.tx + 2) * (best.ty + 2) * (best.tz + 2);
    return best;
}

template <typename T, bool SORTED, int SUM, bool ZS>
static cudaError_t launch_tile(cg_context *c, const TileArgs<T> &TA, int ntiles)
{
    const size_t smem = tile_smem_bytes<T>(TA.t);
    auto kern = sweep_tile_kernel<T, SORTED, SUM, ZS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<ntiles, kThreads, smem, c->stream>>>(TA);
    return cudaGetLastError();
}

template <typename T, bool SORTED, int SUM>
static cudaError_t launch_tile_z(cg_context *c, const TileArgs<T> &TA, int ntiles)
{
    // row-major boxes are (z, uid)-ordered inside (order_in_box): z-window on
    return TA.s.rank_of ? launch_tile<T, SORTED, SUM, false>(c, TA, ntiles)
                        : launch_tile<T, SORTED, SUM, true>(c, TA, ntiles);
}

template <typename T, bool SORTED, int SUM, bool RM>
static void launch_proxy_k(cg_context *c, const SweepArgs<T> &A, const ProxyArgs &P, int kscap)
{
    const int nblk = cdiv(A.n, kThreads);
    if (kscap <= 32) {
        auto k = sweep_proxy_kernel<T, SORTED, SUM, RM, 32>;
        const int sm = 32 * kThreads * sizeof(int);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        k<<<nblk, kThreads, sm, c->stream>>>(A, P);
    } else {
        auto k = sweep_proxy_kernel<T, SORTED, SUM, RM, 64>;
        const int sm = 64 * kThreads * sizeof(int);
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
        k<<<nblk, kThreads, sm, c->stream>>>(A, P);
    }
}

template <typename T, bool SORTED>
static void launch_proxy_s(cg_context *c, const SweepArgs<T> &A, const ProxyArgs &P, int kscap)
{
    const bool rm = A.rank_of == nullptr;
    if (c->summation == SUM_UID) {
        if (rm) launch_proxy_k<T, SORTED, SUM_UID, true>(c, A, P, kscap);
        else launch_proxy_k<T, SORTED, SUM_UID, false>(c, A, P, kscap);
    } else {
        if (rm) launch_proxy_k<T, SORTED, SUM_STENCIL, true>(c, A, P, kscap);
        else launch_proxy_k<T, SORTED, SUM_STENCIL, false>(c, A, P, kscap);
    }
}

template <typename T>
static int launch_sweep(cg_context *c, const SweepArgs<T> &A, bool sorted)
{
    if (c->sweep_impl == 2) {
        const int nblk = cdiv(A.n, kThreads);
        if (sorted)
            make_proxy<T, true><<<nblk, kThreads, 0, c->stream>>>(A.n, A.g, A.idx, A.slot_key, A.flat_of,
                                                                  A.x, A.y, A.z, A.d, c->b.prox);
        else
            make_proxy<T, false><<<nblk, kThreads, 0, c->stream>>>(A.n, A.g, A.idx, A.slot_key, A.flat_of,
                                                                   A.x, A.y, A.z, A.d, c->b.prox);
        LAUNCH_CHECK(c);
        ProxyArgs P;
        P.prox = c->b.prox;
        // fp32 prefilter margin: every stored / derived fp32 coordinate is within
        // a few ulp of E (box-local x/y, grid-relative z); 64 ulp(E) is used
        const double E = A.g.L * (double)std::max(3, A.g.dimz + 2);
        P.margin = (float)(64.0 * E * 5.9604644775390625e-8);
        // survivors per agent ~ 4.19 * density (contact ball / box volume)
        const double rho = (double)A.n / (double)A.g.nb;
        const int kscap = 4.19 * rho <= 20.0 ? 32 : 64;
        CUDA_TRY(c, cudaMemsetAsync(A.block_counters, 0, sizeof(unsigned long long) * 3 * kCounterSlots,
                                    c->stream));
        if (sorted) launch_proxy_s<T, true>(c, A, P, kscap);
        else launch_proxy_s<T, false>(c, A, P, kscap);
        LAUNCH_CHECK(c);
        c->launches += 1;   // make_proxy (the sweep itself is counted by the caller)
        return CG_OK;
    }
    if (c->sweep_impl == 1) {
        TileArgs<T> TA;
        TA.s = A;
        TA.t = choose_tiles(A.g, A.n, c->tile_cap);
        TA.t.debug_stop = c->debug_stop;
        const long long nt = (long long)TA.t.ntx * TA.t.nty * TA.t.ntz;
        if (nt >= INT32_MAX) return fail(c, CG_ERR_VALUE, "too many tiles");
        CUDA_TRY(c, cudaMemsetAsync(A.block_counters, 0, sizeof(unsigned long long) * 3 * kCounterSlots,
                                    c->stream));
        cudaError_t e;
        if (c->summation == SUM_UID)
            e = sorted ? launch_tile_z<T, true, SUM_UID>(c, TA, (int)nt)
                       : launch_tile_z<T, false, SUM_UID>(c, TA, (int)nt);
        else
            e = sorted ? launch_tile_z<T, true, SUM_STENCIL>(c, TA, (int)nt)
                       : launch_tile_z<T, false, SUM_STENCIL>(c, TA, (int)nt);
        CUDA_TRY(c, e);
        return CG_OK;
    }
    const int nblk = cdiv(A.n, kThreads);
    constexpr int KC = sizeof(T) == 8 ? 32 : 32;
    if (c->summation == SUM_UID) {
        if (sorted) sweep_kernel<T, true, SUM_UID, KC><<<nblk, kThreads, 0, c->stream>>>(A);
        else sweep_kernel<T, false, SUM_UID, KC><<<nblk, kThreads, 0, c->stream>>>(A);
    } else {
        if (sorted) sweep_kernel<T, true, SUM_STENCIL, 1><<<nblk, kThreads, 0, c->stream>>>(A);
        else sweep_kernel<T, false, SUM_STENCIL, 1><<<nblk, kThreads, 0, c->stream>>>(A);
    }
    LAUNCH_CHECK(c);
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
    const int n = (int)c->n;
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][0], st));
    double origin[3];
    int64_t dims64[3];
    int rc = build_grid<T>(c, ir, box_cap, origin, dims64);
    if (rc) return rc;
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][1], st));
    const bool sort = (flags & CG_STEP_SORT) && n > 1;
    if (sort) {   // storage re-sort into (box rank, uid) order == lexsort((uid, code))
        const int o = 1 - c->cur_pos, oa = 1 - c->cur_attr;
        gather_records<T><<<cdiv(n, kThreads), kThreads, 0, st>>>(
            n, c->b.idx, (T *)c->b.pos[c->cur_pos][0], (T *)c->b.pos[c->cur_pos][1],
            (T *)c->b.pos[c->cur_pos][2], (T *)c->b.dia[c->cur_attr], (T *)c->b.adh[c->cur_attr],
            c->b.uid[c->cur_attr], (T *)c->b.pos[o][0], (T *)c->b.pos[o][1], (T *)c->b.pos[o][2],
            (T *)c->b.dia[oa], (T *)c->b.adh[oa], c->b.uid[oa]);
        LAUNCH_CHECK(c);
        c->launches += 1;
        c->cur_pos = o;
        c->cur_attr = oa;
    }
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][2], st));
    const int nblk = cdiv(n, kThreads);
    if ((rc = ensure_block_counters(c, std::max(nblk, kCounterSlots)))) return rc;
    SweepArgs<T> A;
    A.n = n;
    A.g = c->geo;
    const int cp = c->cur_pos, ca = c->cur_attr;
    A.x = (const T *)c->b.pos[cp][0];
    A.y = (const T *)c->b.pos[cp][1];
    A.z = (const T *)c->b.pos[cp][2];
    A.d = (const T *)c->b.dia[ca];
    A.adh = (const T *)c->b.adh[ca];
    A.uid = c->b.uid[ca];
    A.idx = c->b.idx;
    A.slot_key = c->b.skey;
    A.off = c->offset;
    A.rank_of = c->morton ? c->mrank : nullptr;
    A.flat_of = c->morton ? c->minv : nullptr;
    A.p = make_params<T>(params);
    A.disp_x = (T *)c->b.disp[0];
    A.disp_y = (T *)c->b.disp[1];
    A.disp_z = (T *)c->b.disp[2];
    const bool freeze = flags & CG_STEP_FREEZE;
    A.new_x = freeze ? nullptr : (T *)c->b.pos[1 - cp][0];
    A.new_y = freeze ? nullptr : (T *)c->b.pos[1 - cp][1];
    A.new_z = freeze ? nullptr : (T *)c->b.pos[1 - cp][2];
    const bool record = flags & CG_STEP_RECORD;
    A.rec_m = record ? c->b.rec_m : nullptr;
    A.rec_nk = record ? c->b.rec_nk : nullptr;
    A.block_counters = c->b.block_counters;
    if ((rc = launch_sweep<T>(c, A, sort))) return rc;
    unsigned long long *stat = c->stat_dev + slot * kStatSlots;
    reduce_counters<<<1, kThreads, 0, st>>>(c->sweep_impl >= 1 ? kCounterSlots : nblk,
                                            c->b.block_counters, stat);
    LAUNCH_CHECK(c);
    c->launches += 2;
    if (!freeze) c->cur_pos = 1 - cp;
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][3], st));
    CUDA_TRY(c, cudaMemcpyAsync(c->stat_host + slot * kStatSlots, stat,
                                sizeof(unsigned long long) * kStatSlots, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaEventRecord(c->ev[slot][4], st));
    for (int a = 0; a < 3; ++a) {
        S.grid_dims[a] = dims64[a];
        S.origin[a] = origin[a];
    }
    S.box_length = c->geo.L;
    c->have_grid = true;
    c->last_sorted = sort;
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

// --------------------------------------------------------------------------- C ABI
extern "C" {

int cg_abi_version(void) { return CG_ABI_VERSION; }

int cg_device_count(int *count)
{
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return CG_ERR_NO_DEVICE;
    }
    return CG_OK;
}

int cg_create(int device, int precision, cg_context **out)
{
    *out = nullptr;
    if (precision != CG_FP64 && precision != CG_FP32) return CG_ERR_VALUE;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
        return CG_ERR_NO_DEVICE;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
        return CG_ERR_NO_DEVICE;   // built for sm_100a only
    if (cudaSetDevice(device) != cudaSuccess) return CG_ERR_NO_DEVICE;
    cg_context *c = new cg_context();
    c->device = device;
    c->prec = precision;
    c->esz = precision == CG_FP64 ? 8 : 4;
    int rc = CG_OK;
    auto chk = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == CG_OK) rc = fail(c, CG_ERR_CUDA, "%s", cudaGetErrorString(e));
    };
    chk(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    chk(cudaMalloc(&c->bbox_partial, sizeof(double) * 7 * kBboxBlocks));
    chk(cudaMalloc(&c->bbox_dev, sizeof(double) * 8));
    chk(cudaMallocHost(&c->bbox_host, sizeof(double) * 8));
    chk(cudaMalloc(&c->stat_dev, sizeof(unsigned long long) * kStatSlots * kRing));
    chk(cudaMallocHost(&c->stat_host, sizeof(unsigned long long) * kStatSlots * kRing));
    for (int r = 0; r < kRing; ++r)
        for (int e = 0; e < 5; ++e) chk(cudaEventCreate(&c->ev[r][e]));
    if (rc != CG_OK) {
        cg_destroy(c);
        return rc;
    }
    *out = c;
    return CG_OK;
}

void cg_destroy(cg_context *c)
{
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    free_agents(c);
    int *ptrs[] = {c->count, c->offset, c->tile_sum, c->mrank, c->minv};
    for (int *p : ptrs)
        if (p) cudaFree(p);
    if (c->b.block_counters) cudaFree(c->b.block_counters);
    if (c->bbox_partial) cudaFree(c->bbox_partial);
    if (c->bbox_dev) cudaFree(c->bbox_dev);
    if (c->bbox_host) cudaFreeHost(c->bbox_host);
    if (c->stat_dev) cudaFree(c->stat_dev);
    if (c->stat_host) cudaFreeHost(c->stat_host);
    for (int r = 0; r < kRing; ++r)
        for (int e = 0; e < 5; ++e)
            if (c->ev[r][e]) cudaEventDestroy(c->ev[r][e]);
    if (c->stream) cudaStreamDestroy(c->stream);
    delete c;
}

const char *cg_last_error(const cg_context *c) { return c ? c->err.c_str() : "null context"; }

void *cg_stream(cg_context *c) { return c ? (void *)c->stream : nullptr; }

int64_t cg_count(const cg_context *c) { return c ? c->n : -1; }

int64_t cg_launch_count(const cg_context *c) { return c ? c->launches : -1; }

void *cg_host_alloc(int64_t bytes)
{
    void *p = nullptr;
    if (bytes <= 0 || cudaMallocHost(&p, (size_t)bytes) != cudaSuccess) return nullptr;
    return p;
}

void cg_host_free(void *p)
{
    if (p) cudaFreeHost(p);
}

int cg_set_option(cg_context *c, int key, int value)
{
    if (!c) return CG_ERR_VALUE;
    if (key == CG_OPT_SUMMATION && (value == SUM_UID || value == SUM_STENCIL)) {
        c->summation = value;
        return CG_OK;
    }
    if (key == CG_OPT_SWEEP && value >= 0 && value <= 2) {
        c->sweep_impl = value;
        return CG_OK;
    }
    if (key == 99 && value >= 0 && value <= 2) {   // profiling aid (not in the header)
        c->debug_stop = value;
        return CG_OK;
    }
    if (key == CG_OPT_TILE_CAP && value >= 256 && value <= 8192) {
        c->tile_cap = value;
        return CG_OK;
    }
    if (key == CG_OPT_BOX_ORDER && (value == 0 || value == 1)) {
        c->morton = value == 0;
        c->table_dims[0] = 0;
        return CG_OK;
    }
    return fail(c, CG_ERR_VALUE, "bad option %d=%d", key, value);
}

int cg_upload(cg_context *c, int64_t n, const void *px, const void *py, const void *pz,
              const void *diameter, const void *adherence, const uint64_t *uid)
{
    if (!c) return CG_ERR_VALUE;
    if (n < 0) return fail(c, CG_ERR_VALUE, "negative agent count");
    if (n >= (int64_t)INT32_MAX / 2) return fail(c, CG_ERR_POOL_CAPACITY, "%lld agents exceeds the device cap", (long long)n);
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (n > c->cap) {
        int rc = alloc_agents(c, n);
        if (rc) return rc;
    }
    c->n = n;
    c->cur_pos = c->cur_attr = 0;
    c->have_grid = false;
    if (n == 0) return CG_OK;
    const size_t fe = c->esz * (size_t)n;
    cudaStream_t st = c->stream;
    const void *src[3] = {px, py, pz};
    for (int a = 0; a < 3; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(c->b.pos[0][a], src[a], fe, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.dia[0], diameter, fe, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.adh[0], adherence, fe, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.uid[0], uid, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
    for (int a = 0; a < 3; ++a) CUDA_TRY(c, cudaMemsetAsync(c->b.disp[a], 0, fe, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));   // host buffers are only borrowed
    return CG_OK;
}

int cg_download(cg_context *c, void *px, void *py, void *pz, void *diameter, void *adherence,
                uint64_t *uid, void *dx, void *dy, void *dz)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    const int64_t n = c->n;
    if (n == 0) return CG_OK;
    const size_t fe = c->esz * (size_t)n;
    cudaStream_t st = c->stream;
    void *dst[9] = {px, py, pz, diameter, adherence, uid, dx, dy, dz};
    const void *src[9] = {c->b.pos[c->cur_pos][0], c->b.pos[c->cur_pos][1], c->b.pos[c->cur_pos][2],
                          c->b.dia[c->cur_attr], c->b.adh[c->cur_attr], c->b.uid[c->cur_attr],
                          c->b.disp[0], c->b.disp[1], c->b.disp[2]};
    for (int k = 0; k < 9; ++k)
        if (dst[k])
            CUDA_TRY(c, cudaMemcpyAsync(dst[k], src[k], k == 5 ? sizeof(uint64_t) * n : fe,
                                        cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    return CG_OK;
}

int cg_step(cg_context *c, const double params[5], double interaction_radius, int64_t box_cap,
            int flags, cg_step_stats *stats)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    int64_t id = -1;
    const int rc = c->prec == CG_FP64
                       ? step_impl<double>(c, params, interaction_radius, box_cap, flags, &id)
                       : step_impl<float>(c, params, interaction_radius, box_cap, flags, &id);
    if (rc) return rc;
    if (stats) return collect(c, id, stats);
    return CG_OK;
}

int cg_build_grid(cg_context *c, double interaction_radius, int64_t box_cap, cg_step_stats *stats)
{
    if (!c) return CG_ERR_VALUE;
    if (c->n == 0) return fail(c, CG_ERR_VALUE, "cannot build a grid over an empty pool");
    CUDA_TRY(c, cudaSetDevice(c->device));
    double origin[3];
    int64_t dims64[3];
    const int slot = (int)(c->steps_done % kRing);
    const int rc = c->prec == CG_FP64
                       ? build_grid<double>(c, interaction_radius, box_cap, origin, dims64)
                       : build_grid<float>(c, interaction_radius, box_cap, origin, dims64);
    if (rc) return rc;
    c->have_grid = true;
    c->last_sorted = false;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (stats) {
        std::memset(stats, 0, sizeof *stats);
        stats->step_id = -1;
        stats->agent_count = c->n;
        unsigned long long h[kStatSlots];
        CUDA_TRY(c, cudaMemcpy(h, c->stat_dev + slot * kStatSlots, sizeof h, cudaMemcpyDeviceToHost));
        stats->grid_occupied_boxes = (int64_t)h[0];
        stats->grid_max_occupancy = (int64_t)h[1];
        for (int a = 0; a < 3; ++a) {
            stats->grid_dims[a] = dims64[a];
            stats->origin[a] = origin[a];
        }
        stats->box_length = c->geo.L;
    }
    return CG_OK;
}

int cg_fetch_stats(cg_context *c, int64_t step_id, cg_step_stats *stats)
{
    if (!c || !stats) return CG_ERR_VALUE;
    return collect(c, step_id, stats);
}

int cg_synchronize(cg_context *c)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return CG_OK;
}

int cg_grid_export(cg_context *c, int64_t *box_index, int64_t *box_count)
{
    if (!c) return CG_ERR_VALUE;
    if (!c->have_grid) return fail(c, CG_ERR_STATE, "no grid: run a step first");
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const int n = (int)c->n, nb = c->geo.nb;
    std::vector<int> skey(n), key(n), cnt(nb), minv;
    if (c->morton) {
        minv.resize(nb);
        CUDA_TRY(c, cudaMemcpy(minv.data(), c->minv, sizeof(int) * nb, cudaMemcpyDeviceToHost));
    }
    auto flat = [&](int k) { return c->morton ? minv[k] : k; };
    if (box_index) {
        // sorted: storage slot s holds slot s of the CSR; else key[] is per storage index
        if (c->last_sorted) {
            CUDA_TRY(c, cudaMemcpy(skey.data(), c->b.skey, sizeof(int) * n, cudaMemcpyDeviceToHost));
            for (int s = 0; s < n; ++s) box_index[s] = flat(skey[s]);
        } else {
            CUDA_TRY(c, cudaMemcpy(key.data(), c->b.key, sizeof(int) * n, cudaMemcpyDeviceToHost));
            for (int i = 0; i < n; ++i) box_index[i] = flat(key[i]);
        }
    }
    if (box_count) {
        CUDA_TRY(c, cudaMemcpy(cnt.data(), c->count, sizeof(int) * nb, cudaMemcpyDeviceToHost));
        for (int k = 0; k < nb; ++k) box_count[flat(k)] = cnt[k];
    }
    return CG_OK;
}

int cg_record_export(cg_context *c, int32_t *m, int32_t *nk)
{
    if (!c) return CG_ERR_VALUE;
    if (!c->last_record) return fail(c, CG_ERR_STATE, "last step did not run with CG_STEP_RECORD");
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (m) CUDA_TRY(c, cudaMemcpy(m, c->b.rec_m, sizeof(int) * c->n, cudaMemcpyDeviceToHost));
    if (nk) CUDA_TRY(c, cudaMemcpy(nk, c->b.rec_nk, sizeof(int) * c->n, cudaMemcpyDeviceToHost));
    return CG_OK;
}

int cg_box_ids(cg_context *c, int64_t n, const void *px, const void *py, const void *pz, double ox,
               double oy, double oz, double box_length, int64_t dimx, int64_t dimy, int64_t dimz,
               int64_t *out)
{
    if (!c) return CG_ERR_VALUE;
    if (n == 0) return CG_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    int rc = CG_OK;
    if (n > c->cap && (rc = alloc_agents(c, n))) return rc;
    c->n = 0;   // the resident pool is overwritten by this call
    c->have_grid = false;
    Geometry g{box_length, ox, oy, oz, (int)dimx, (int)dimy, (int)dimz, (int)(dimx * dimy * dimz)};
    const size_t fe = c->esz * (size_t)n;
    const void *src[3] = {px, py, pz};
    for (int a = 0; a < 3; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(c->b.pos[0][a], src[a], fe, cudaMemcpyHostToDevice, c->stream));
    void *tmp = nullptr;
    CUDA_TRY(c, cudaMallocAsync(&tmp, sizeof(long long) * n, c->stream));
    long long *dout = (long long *)tmp;
    if (c->prec == CG_FP64)
        box_ids_only<double><<<cdiv(n, kThreads), kThreads, 0, c->stream>>>(
            (int)n, g, (double *)c->b.pos[0][0], (double *)c->b.pos[0][1], (double *)c->b.pos[0][2], dout);
    else
        box_ids_only<float><<<cdiv(n, kThreads), kThreads, 0, c->stream>>>(
            (int)n, g, (float *)c->b.pos[0][0], (float *)c->b.pos[0][1], (float *)c->b.pos[0][2], dout);
    LAUNCH_CHECK(c);
    CUDA_TRY(c, cudaMemcpyAsync(out, dout, sizeof(long long) * n, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaFreeAsync(tmp, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return CG_OK;
}

int cg_force_phase(cg_context *c, int64_t n, const void *px, const void *py, const void *pz,
                   const void *radii, const void *adherence, const uint64_t *uid,
                   const int64_t *box_index, int64_t dimx, int64_t dimy, int64_t dimz,
                   const void *params7, void *out_dx, void *out_dy, void *out_dz,
                   int64_t counters[3])
{
    if (!c) return CG_ERR_VALUE;
    counters[0] = counters[1] = counters[2] = 0;
    if (n == 0) return CG_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    // upload the pool with radii in the diameter column (doubled on device: exact)
    int rc = cg_upload(c, n, px, py, pz, radii, adherence, uid);
    if (rc) return rc;
    const int nn = (int)n;
    cudaStream_t st = c->stream;
    const int64_t nb64 = dimx * dimy * dimz;
    if (nb64 >= (int64_t)INT32_MAX) return fail(c, CG_ERR_GRID_OVERFLOW, "too many boxes");
    if ((rc = ensure_boxes(c, nb64))) return rc;
    Geometry g{0.0, 0.0, 0.0, 0.0, (int)dimx, (int)dimy, (int)dimz, (int)nb64};
    c->geo = g;
    c->morton = false;   // kernel-level call: row-major keys taken from box_index
    c->table_dims[0] = 0;
    // no box_length is given at this level, so use the thread-per-agent sweep
    // (the tiled sweep's prefilter needs L)
    struct Restore {
        cg_context *c;
        int v;
        ~Restore() { c->sweep_impl = v; }
    } restore{c, c->sweep_impl};
    c->sweep_impl = 0;
    long long *dbox = nullptr;
    CUDA_TRY(c, cudaMallocAsync(&dbox, sizeof(long long) * n, st));
    CUDA_TRY(c, cudaMemcpyAsync(dbox, box_index, sizeof(long long) * n, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemsetAsync(c->count, 0, sizeof(int) * g.nb, st));
    const int nblk = cdiv(nn, kThreads);
    if (c->prec == CG_FP64) double_column<double><<<nblk, kThreads, 0, st>>>(nn, (double *)c->b.dia[0]);
    else double_column<float><<<nblk, kThreads, 0, st>>>(nn, (float *)c->b.dia[0]);
    keys_from_flat<<<nblk, kThreads, 0, st>>>(nn, dbox, c->count, c->b.key, c->b.rnk);
    const int ntiles = cdiv(g.nb, kScanTile);
    const int slot = (int)(c->steps_done % kRing);
    unsigned long long *stat = c->stat_dev + slot * kStatSlots;
    CUDA_TRY(c, cudaMemsetAsync(stat, 0, sizeof(unsigned long long) * kStatSlots, st));
    scan_tiles<<<ntiles, kThreads, 0, st>>>(g.nb, c->count, c->offset, c->tile_sum, stat);
    scan_tile_sums<<<1, kThreads, 0, st>>>(ntiles, c->tile_sum);
    scan_add<<<cdiv(g.nb, kThreads), kThreads, 0, st>>>(g.nb, nn, c->tile_sum, c->offset);
    place<<<nblk, kThreads, 0, st>>>(nn, c->b.key, c->b.rnk, c->offset, c->b.tmp);
    order_in_box<double, false><<<nblk, kThreads, 0, st>>>(nn, c->b.tmp, c->b.key, c->offset,
                                                           c->b.uid[0], nullptr, c->b.idx, c->b.skey);
    LAUNCH_CHECK(c);
    if ((rc = ensure_block_counters(c, std::max(nblk, kCounterSlots)))) return rc;
    double p5[5];
    for (int k = 0; k < 5; ++k)
        p5[k] = c->prec == CG_FP64 ? ((const double *)params7)[k] : (double)((const float *)params7)[k];
    if (c->prec == CG_FP64) {
        SweepArgs<double> A{};
        A.n = nn; A.g = g;
        A.x = (double *)c->b.pos[0][0]; A.y = (double *)c->b.pos[0][1]; A.z = (double *)c->b.pos[0][2];
        A.d = (double *)c->b.dia[0]; A.adh = (double *)c->b.adh[0]; A.uid = c->b.uid[0];
        A.idx = c->b.idx; A.slot_key = c->b.skey; A.off = c->offset;
        A.p = make_params<double>(p5);
        A.disp_x = (double *)c->b.disp[0]; A.disp_y = (double *)c->b.disp[1]; A.disp_z = (double *)c->b.disp[2];
        A.block_counters = c->b.block_counters;
        if ((rc = launch_sweep<double>(c, A, false))) return rc;
    } else {
        SweepArgs<float> A{};
        A.n = nn; A.g = g;
        A.x = (float *)c->b.pos[0][0]; A.y = (float *)c->b.pos[0][1]; A.z = (float *)c->b.pos[0][2];
        A.d = (float *)c->b.dia[0]; A.adh = (float *)c->b.adh[0]; A.uid = c->b.uid[0];
        A.idx = c->b.idx; A.slot_key = c->b.skey; A.off = c->offset;
        A.p = make_params<float>(p5);
        A.disp_x = (float *)c->b.disp[0]; A.disp_y = (float *)c->b.disp[1]; A.disp_z = (float *)c->b.disp[2];
        A.block_counters = c->b.block_counters;
        if ((rc = launch_sweep<float>(c, A, false))) return rc;
    }
    reduce_counters<<<1, kThreads, 0, st>>>(c->sweep_impl >= 1 ? kCounterSlots : nblk,
                                            c->b.block_counters, stat);
    LAUNCH_CHECK(c);
    unsigned long long h[kStatSlots];
    CUDA_TRY(c, cudaMemcpyAsync(h, stat, sizeof h, cudaMemcpyDeviceToHost, st));
    const size_t fe = c->esz * (size_t)n;
    void *dst[3] = {out_dx, out_dy, out_dz};
    for (int a = 0; a < 3; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(dst[a], c->b.disp[a], fe, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaFreeAsync(dbox, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    counters[0] = (int64_t)h[2];
    counters[1] = (int64_t)h[3];
    counters[2] = (int64_t)h[4];
    c->n = 0;   // the resident buffers no longer hold a consistent pool
    c->have_grid = false;
    return CG_OK;
}

}  // extern "C"
