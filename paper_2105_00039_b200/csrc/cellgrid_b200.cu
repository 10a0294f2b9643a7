// cellgrid_b200.cu -- context, step orchestration and the C ABI
// (include/cellgrid_b200.h).
//
// One context = one agent population resident in the HBM of one B200.  A step
// (reference engine.py:279-341) is:
//   bbox (from the previous sweep's reduction slots; a standalone pass only
//   after an upload) -> host geometry (spatial.py:99-116, exact f64) ->
//   box_keys (+ warp-aggregated counts) -> reduce-then-scan -> then either
//   * a grid sweep: place (CSR slots + fp32 proxies; on a relayout step the
//     records themselves move into slot order) -> sweep7 (force, gate, cap,
//     apply, counters, next bbox; optionally also the neighbour lists), or
//   * a list sweep (list.cuh) while the neighbour lists are valid
//   -> finish_step (fold the slots).
// The only host round trip is the 9-double readback (bbox, largest
// displacement, list overflows): it sizes the grid and raises
// GridOverflowError before anything is modified, exactly where the reference
// raises, and decides whether the lists still cover every pair.
//
// Storage order.  The reference re-sorts its pool into (Morton code, uid)
// order on every sort step (engine.py:305-309, morton.py:67-74); only the
// pool's storage order observes that.  Here the records move into the
// device's slot order on relayout steps (every `relayout_every`-th sort step)
// and the reference's order is kept as a permutation `pres` (storage index
// -> reference storage position), materialised only when the host downloads
// or exports -- so every download returns exactly the reference's pool.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>


#include "../../include/cellgrid_b200.h"

#ifndef CG_LIST_BUILD_MINB
#define CG_LIST_BUILD_MINB 4   // the same sweep building neighbour lists
#endif
#ifndef CG_LIST_BUILD_KS
#define CG_LIST_BUILD_KS 24    // survivors per agent held by the (uniform, 32-bit key) list build (48 KB smem; 16: build 4.44 -> 4.32 ms at skin 1.2)
#endif
#ifndef CG_SPARSE_MINB
#define CG_SPARSE_MINB 4   // resident 256-thread CTAs per SM for the sparse sweep (measured)
#endif
#include "common.cuh"
#include "grid.cuh"
#include "sweep.cuh"
#include "sweep7.cuh"
#include "slab.cuh"
#include "sweep_warp.cuh"
#include "query.cuh"
#include "list.cuh"
#include "behavior.cuh"

using namespace cg;

namespace {

constexpr int kStatSlots = 8;        // per step: occupied, maxocc, evals, cands, ndeg
constexpr int kRing = 64;            // pinned stats ring (steps in flight)
// grid-stride launches are sized in multiples of the SM count (cg_create
// reads it; 148 on a B200)
constexpr int kMaxCounterBlocks = 1 << 20;

enum { PRES_IDENTITY = 0, PRES_VALID = 1, PRES_PENDING = 2 };

struct Buffers {
    void *rec[2] = {nullptr, nullptr};   // Rec<T>: x, y, z, diameter (double-buffered)
    void *adh[2] = {nullptr, nullptr};
    uint64_t *uid[2] = {nullptr, nullptr};
    void *disp[3] = {nullptr, nullptr, nullptr};
    int2 *key_rank = nullptr;
    int *tmp = nullptr, *idx = nullptr, *skey = nullptr, *pres = nullptr;
    int *pkey[2] = {nullptr, nullptr};   // box at the last sort step (travels with the records)
    int *ovf = nullptr;              // sweep overflow list
    void *pscratch = nullptr;        // lazy presentation sort scratch
    size_t pscratch_bytes = 0;
    int *rec_m = nullptr, *rec_nk = nullptr;
    float *prox = nullptr;           // Proxies: 8 floats per slot pair
    Proxies P() const { return Proxies{prox}; }
    int64_t pairs = 0;
    void *stage = nullptr;           // download staging (n x 8 B)
    int64_t head = 0;                // front headroom (elements) of rec / adh / uid
};

}  // namespace

struct cg_context {
    int device = 0;
    int sms = 148;                // streaming multiprocessors of the device
    int prec = CG_FP64;
    size_t esz = 8;
    cudaStream_t stream = nullptr;
    int64_t n = 0, cap = 0;
    int64_t n_owned = 0;          // agents this context owns; [n_owned, n) are this step's ghosts
    Buffers b;
    int cur_pos = 0, cur_attr = 0;
    // boxes
    int64_t box_cap = 0;
    int *count = nullptr, *offset = nullptr, *mrank = nullptr, *minv = nullptr;
    int *count_own = nullptr;   // slab list steps: per-box ghost counts (zero between steps)
    unsigned long long *scan_status = nullptr;   // (tiles + 2) words; the last two are tickets
    int64_t scan_tiles_cap = 0;
    int table_dims[3] = {0, 0, 0};
    // per-step reductions
    unsigned long long *slots = nullptr;
    unsigned long long *maxd_enc = nullptr;
    unsigned *ovf_count = nullptr;
    // dense uid-mode second pass (sweep_warp BIG): per-warp global queues
    void *big = nullptr;
    int big_warps = 0;
    int *ovf2 = nullptr;
    unsigned *ovf2_count = nullptr;
    int64_t ovf2_cap = 0;
    unsigned long long *block_counters = nullptr;   // reference-order sweep only
    double *bbox_dev = nullptr, *bbox_host = nullptr;
    bool bbox_valid = false;
    double max_diam = 0.0;
    double min_diam = -INFINITY;   // == max_diam: a uniform pool (list sweep pair constants from the host)
    unsigned long long *stat_dev = nullptr, *stat_host = nullptr;
    cg_step_stats ring[kRing];
    cudaEvent_t ev[kRing][5];
    cudaStream_t copy_stream = nullptr;       // download: D2H overlapped with the unpack kernels
    // cg_step_download: diameter / adherence / uid leave during the sweep
    struct Early {
        bool want = false, done = false;
        void *dst[3] = {nullptr, nullptr, nullptr};   // diameter, adherence, uid (host)
        char *buf = nullptr;
        size_t bytes = 0;
        cudaEvent_t grid_done = nullptr, ready = nullptr;
    } early;
    cudaEvent_t dl_ready[9] = {}, dl_done[9] = {}, dl_start = nullptr;
    int64_t steps_done = 0;
    int64_t launches = 0;
    // grid / layout state
    Geometry geo{};
    BoxDecode bd{};
    bool have_grid = false;
    bool relaid = false;          // storage == slot order of the current grid
    int pres_state = PRES_IDENTITY;
    bool last_record = false;
    bool last_dense = false;
    bool grid_current = false;    // the grid indexes the stored positions (cg_build_grid)
    // neighbour-list reuse (list.cuh): skin < 0 = auto (auto_skin), 0 = off
    double list_skin = -1.0;
    int *nbr = nullptr, *nbr_n = nullptr;
    // sub-lists (list.cuh INNER): level k in {1, 2} holds the partners within
    // r_i + r_j + delta_k, written by a sweep of a longer list (its parent:
    // level 0 = the neighbour list, or level 1) and swept while twice the
    // motion since it was written stays below delta_k and its parent is still
    // valid.  Level 2 is the short list most steps sweep (CG_OPT_INNER_LIST),
    // level 1 an optional middle list (CG_OPT_MID_LIST) that refreshes it.
    int *lvl_nbr[3] = {nullptr, nullptr, nullptr}, *lvl_n[3] = {nullptr, nullptr, nullptr};
    double lvl_frac[3] = {1.0, 0.385, 0.173};   // delta_k = frac_k x skin (C4: 1.0 and 0.45 at skin 2.6)
    bool lvl_valid[3] = {}, lvl_written[3] = {};
    int64_t lvl_epoch[3] = {-1, -1, -1};     // list_builds when written
    double lvl_D[3] = {}, lvl_delta[3] = {};
    int lvl_parent[3] = {};
    int64_t inner_steps = 0;      // list steps that swept a sub-list
    int64_t nbr_cap = 0;
    int nbr_width = 0;            // entries per agent allocated
    int list_width = kListCap;    // entries per agent of the current lists
    bool list_valid = false;      // lists cover every pair that can overlap now
    int last_kind = 0;            // previous step: 0 other, 1 list build, 2 list step
    bool last_freeze = false;
    double list_D = 0.0;          // bound on any agent's motion since the build
    double list_skin_used = 0.0;
    int list_life = 0, list_backoff = 0, list_wait = 0;
    int64_t list_builds = 0, list_steps = 0;
    int64_t overlapped_steps = 0;   // slab list steps whose interior sweep ran before the ghost refresh
    bool uid32 = false;           // every stored uid < 2^32 (upload, behaviour phase; slabs: the global max uid)
    uint64_t max_uid = 0;         // largest stored uid (upload, behaviour phase)
    void *beh = nullptr;          // behaviour phase scratch (ripe list, sort buffers), beh_bytes
    size_t beh_bytes = 0;
    unsigned long long *maxuid_dev = nullptr;
    int rot = 0;                  // relaid slab sub-grid: slot s lives at storage s - rot (lo ghosts in
                                  // the buffers' front headroom, owned agents at [0, n_owned))
    int64_t sort_steps = 0;
    Geometry geo_sort{};          // geometry of the last sort step (presentation order)
    // options
    int summation = SUM_UID;
    int sweep_impl = 1;           // 0 = reference-order thread per agent, 1 = sweep7 (production)
    int relayout_every = 1;       // relayout on every k-th sort step (1 = every sort step)
    int path = 0;                 // 0 = auto, 1 = sparse (uid-sorted lists), 2 = dense (z-sorted boxes)
    // x-slab decomposition (multi-GPU)
    struct Slab {
        bool planned = false;
        Geometry g{};            // global geometry of this step
        SlabBounds B{};
        int rank = 0, world = 1, x0 = 0, x1 = 0;
        bool packed = false;
        unsigned char *dest = nullptr;           // owner rank | ghost flags (slab.cuh)
        int *out = nullptr, *holes = nullptr, *movers = nullptr;
        unsigned *cnt = nullptr;                 // 8 counters
        unsigned long long *counts = nullptr;    // kHist bins (slab.cuh)
        unsigned long long *seg_off = nullptr;   // send-buffer run starts, 3 per destination
        unsigned *cursor = nullptr;
        int64_t cap = 0;
        int64_t h_counts[kHist] = {};
        int64_t steps = 0;
        int64_t ghost_lo = 0;    // ghosts from rank - 1 (in front of the ghost buffer)
        // neighbour lists across slabs (list mode: frozen partition, ghost refresh)
        bool list_mode = false;    // this step refreshes ghosts and runs the list sweep
        bool refresh_ready = false;
        bool unpacked = false;
        int64_t n_total = 0;       // owned + ghosts kept between rebuilds
        int rot_build = 0;         // index of the first owned agent (the lo-ghost count)
        // list steps: owned rows [rot_build + b_lo, rot_build + n_owned - b_hi)
        // hold no ghost in their lists (build planes >= 3 from either slab face)
        // and may be swept before the ghost refresh lands (cg_slab_step_interior)
        bool split_ok = false;
        int b_lo = 0, b_hi = 0;
        bool interior_done = false;
        int read_lvl = 0, write_lvl = -1;   // this list step's sub-list choice (both parts)
        double x_lo_abs = 0, x_hi_abs = 0;   // the owned slab's x range at the rebuild
        int64_t ref_counts[kHist] = {};      // refresh records per (destination, kind)
        int64_t ref_total = 0;
        int *ref_list = nullptr;             // owned indices, grouped by (destination, kind)
        unsigned long long *ref_off = nullptr;
        uint64_t *hkey = nullptr;    // ghost table: uid -> ghost index (slab.cuh), per list epoch
        int *hval = nullptr;
        int64_t hcap = 0;            // slots (power of two)
        unsigned hmask = 0;
        int *r2g = nullptr;          // receive position -> ghost index (valid after the epoch's first refresh)
        bool r2g_valid = false;
        unsigned *mismatch = nullptr;   // refresh records without a ghost (read back with the next bbox)
        int64_t list_cap = 0;
    } slab;
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

static void free_inner(cg_context *c)
{
    for (int k = 1; k < 3; ++k) {
        if (c->lvl_nbr[k]) cudaFree(c->lvl_nbr[k]);
        if (c->lvl_n[k]) cudaFree(c->lvl_n[k]);
        c->lvl_nbr[k] = c->lvl_n[k] = nullptr;
        c->lvl_valid[k] = false;
    }
}

static void free_agents(cg_context *c)
{
    Buffers &b = c->b;
    for (int k = 0; k < 2; ++k) {
        if (b.rec[k]) cudaFree((char *)b.rec[k] - 4 * c->esz * b.head);
        if (b.adh[k]) cudaFree((char *)b.adh[k] - c->esz * b.head);
        if (b.uid[k]) cudaFree(b.uid[k] - b.head);
    }
    void *ptrs[] = {b.disp[0], b.disp[1], b.disp[2], b.key_rank, b.tmp, b.idx, b.skey, b.pres,
                    b.rec_m, b.rec_nk, b.prox, b.stage, b.pkey[0], b.pkey[1], b.pscratch, b.ovf};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    c->b = Buffers{};
    c->cap = 0;
    if (c->nbr) cudaFree(c->nbr);
    if (c->nbr_n) cudaFree(c->nbr_n);
    c->nbr = c->nbr_n = nullptr;
    free_inner(c);
    c->nbr_cap = 0;
    c->list_valid = false;
    c->last_kind = 0;
}

static int alloc_agents(cg_context *c, int64_t cap)
{
    free_agents(c);
    Buffers &b = c->b;
    const size_t fe = c->esz * (size_t)cap, ie = sizeof(int) * (size_t)cap;
    // front headroom: a relaid slab step stores its lo ghosts before element 0
    const int64_t H = cap / 16 + 1024;
    for (int k = 0; k < 2; ++k) {
        void *p;
        CUDA_TRY(c, cudaMalloc(&p, 4 * c->esz * (size_t)(cap + H)));
        b.rec[k] = (char *)p + 4 * c->esz * H;
        CUDA_TRY(c, cudaMalloc(&p, c->esz * (size_t)(cap + H)));
        b.adh[k] = (char *)p + c->esz * H;
        CUDA_TRY(c, cudaMalloc(&p, sizeof(uint64_t) * (size_t)(cap + H)));
        b.uid[k] = (uint64_t *)p + H;
        b.head = H;
    }
    for (int a = 0; a < 3; ++a) CUDA_TRY(c, cudaMalloc(&b.disp[a], fe));
    CUDA_TRY(c, cudaMalloc(&b.key_rank, sizeof(int2) * (size_t)cap));
    int **ints[] = {&b.tmp, &b.idx, &b.skey, &b.pres, &b.rec_m, &b.rec_nk, &b.pkey[0], &b.pkey[1], &b.ovf};
    for (int **p : ints) CUDA_TRY(c, cudaMalloc(p, ie));
    b.pairs = cap / 2 + 8;   // the sweep may read a few pairs past n
    CUDA_TRY(c, cudaMalloc(&b.prox, sizeof(float) * 8 * (size_t)b.pairs));
    CUDA_TRY(c, cudaMemset(b.prox, 0, sizeof(float) * 8 * (size_t)b.pairs));
    CUDA_TRY(c, cudaMalloc(&b.stage, 8 * (size_t)cap));
    c->cap = cap;
    return CG_OK;
}

// More agent capacity with the resident pool kept: the live columns (records,
// adherence, uid, displacements, the presentation order) move to buffers of
// the new capacity; per-step scratch is reallocated, neighbour lists dropped.
static int grow_agents(cg_context *c, int64_t cap)
{
    const Buffers old = c->b;
    const int64_t n = c->n;
    const int cp = c->cur_pos, ca = c->cur_attr;
    c->b = Buffers{};   // alloc_agents frees c->b: keep the old set alive until copied
    const int64_t oldcap = c->cap;
    c->cap = 0;
    int *nbr = c->nbr, *nbr_n = c->nbr_n;
    c->nbr = c->nbr_n = nullptr;
    free_inner(c);
    int rc = alloc_agents(c, cap);
    if (nbr) cudaFree(nbr);
    if (nbr_n) cudaFree(nbr_n);
    if (rc) return rc;
    cudaStream_t st = c->stream;
    const size_t es = c->esz;
    CUDA_TRY(c, cudaMemcpyAsync(c->b.rec[0], old.rec[cp], 4 * es * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.adh[0], old.adh[ca], es * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.uid[0], old.uid[ca], 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    for (int a = 0; a < 3; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(c->b.disp[a], old.disp[a], es * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.pres, old.pres, 4 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.pkey[0], old.pkey[ca], 4 * (size_t)n, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    for (int k = 0; k < 2; ++k) {
        if (old.rec[k]) cudaFree((char *)old.rec[k] - 4 * es * old.head);
        if (old.adh[k]) cudaFree((char *)old.adh[k] - es * old.head);
        if (old.uid[k]) cudaFree(old.uid[k] - old.head);
    }
    void *ptrs[] = {old.disp[0], old.disp[1], old.disp[2], old.key_rank, old.tmp, old.idx, old.skey, old.pres,
                    old.rec_m, old.rec_nk, old.prox, old.stage, old.pkey[0], old.pkey[1], old.pscratch, old.ovf};
    for (void *p : ptrs)
        if (p) cudaFree(p);
    (void)oldcap;
    c->cur_pos = c->cur_attr = 0;
    c->have_grid = false;
    c->relaid = false;
    return CG_OK;
}

static int ensure_boxes(cg_context *c, int64_t nb)
{
    if (nb <= c->box_cap) return CG_OK;
    const int64_t want = nb + nb / 4 + 1024;
    int *ptrs[] = {c->count, c->offset, c->mrank, c->minv, c->count_own};
    for (int *p : ptrs)
        if (p) cudaFree(p);
    if (c->scan_status) cudaFree(c->scan_status);
    CUDA_TRY(c, cudaMalloc(&c->count, sizeof(int) * want));
    CUDA_TRY(c, cudaMemsetAsync(c->count, 0, sizeof(int) * want, c->stream));   // the scan keeps it zero
    CUDA_TRY(c, cudaMalloc(&c->offset, sizeof(int) * (want + 1)));
    CUDA_TRY(c, cudaMalloc(&c->mrank, sizeof(int) * want));
    CUDA_TRY(c, cudaMalloc(&c->minv, sizeof(int) * want));
    CUDA_TRY(c, cudaMalloc(&c->count_own, sizeof(int) * want));
    CUDA_TRY(c, cudaMemsetAsync(c->count_own, 0, sizeof(int) * want, c->stream));
    c->scan_tiles_cap = cdiv(want, kScanTile) + 1;
    CUDA_TRY(c, cudaMalloc(&c->scan_status, sizeof(unsigned long long) * (c->scan_tiles_cap + 2)));
    c->box_cap = want;
    c->table_dims[0] = c->table_dims[1] = c->table_dims[2] = 0;
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
    if (nb >= (int64_t)INT32_MAX / 2)
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
    g.xoff = 0;
    g.gdimx = g.dimx;
    return CG_OK;
}

static BoxDecode make_decode(const Geometry &g)
{
    BoxDecode bd;
    bd.by_z = FastDiv((unsigned)g.dimz);
    bd.by_y = FastDiv((unsigned)g.dimy);
    bd.dimz = g.dimz;
    bd.dimy = g.dimy;
    return bd;
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

// Exclusive scan of the per-box counts (decoupled look-back, one pass).  stat
// may be null.
static int launch_scan(cg_context *c, int nb, int *out, unsigned long long *stat)
{
    const int ntiles = cdiv(nb, kScanTile);
    CUDA_TRY(c, cudaMemsetAsync(c->scan_status, 0, sizeof(unsigned long long) * ntiles, c->stream));
    unsigned *ticket = reinterpret_cast<unsigned *>(c->scan_status + c->scan_tiles_cap);
    CUDA_TRY(c, cudaMemsetAsync(ticket, 0, sizeof(unsigned), c->stream));
    ScanState S{c->scan_status, ticket};
    scan_lookback<false><<<ntiles, kThreads, 0, c->stream>>>(nb, c->count, nullptr, nullptr, out, S, stat);
    LAUNCH_CHECK(c);
    c->launches += 1;
    return CG_OK;
}

// Reduce-then-scan of the per-box counts into offsets (zeroes the counts).
static int launch_scan_rts(cg_context *c, int nb, unsigned long long *stat)
{
    const int ntiles = cdiv(nb, kScanTile);
    cudaStream_t st = c->stream;
    int *tile_sum = reinterpret_cast<int *>(c->scan_status);   // >= ntiles ints
    scan_reduce<<<ntiles, kThreads, 0, st>>>(nb, c->count, tile_sum);
    scan_tilesums<<<1, 1024, 0, st>>>(ntiles, tile_sum);
    scan_down<<<ntiles, kThreads, 0, st>>>(nb, c->count, tile_sum, c->offset, stat);
    LAUNCH_CHECK(c);
    c->launches += 3;
    return CG_OK;
}

// Standalone bbox of the stored positions into bbox_host (synchronous).
template <typename T>
static int standalone_bbox(cg_context *c)
{
    const int n = (int)c->n_owned;
    cudaStream_t st = c->stream;
    bbox_slots<T><<<std::min(c->sms * 4, cdiv(n, kThreads)), kThreads, 0, st>>>(
        n, (const Rec<T> *)c->b.rec[c->cur_pos], c->slots);
    finish_step<<<1, kThreads, 0, st>>>(c->slots, c->max_diam, nullptr, c->bbox_dev, FINISH_BBOX);
    LAUNCH_CHECK(c);
    c->launches += 2;
    CUDA_TRY(c, cudaMemcpyAsync(c->bbox_host, c->bbox_dev, 9 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    c->bbox_valid = true;
    return CG_OK;
}

// The reference's storage order (see header comment): sort storage indices
// by uid, then stably by the Morton rank of their box at the last sort step.
static int materialize_presentation(cg_context *c, cudaStream_t st = nullptr)
{
    if (c->pres_state != PRES_PENDING) return CG_OK;
    const Geometry &g = c->geo_sort;
    if (!st) st = c->stream;
    const int n = (int)c->n;
    if (c->table_dims[0] != g.dimx || c->table_dims[1] != g.dimy || c->table_dims[2] != g.dimz) {
        int rc = ensure_boxes(c, g.nb);
        if (rc) return rc;
        morton_table<<<std::min(cdiv(g.nb, kThreads), c->sms * 16), kThreads, 0, st>>>(g, c->mrank, c->minv);
        LAUNCH_CHECK(c);
        c->launches += 1;
        c->table_dims[0] = g.dimx;
        c->table_dims[1] = g.dimy;
        c->table_dims[2] = g.dimz;
    }
    // scratch: per agent box rank, slot in box, segment entry; per Morton rank
    // counts and offsets; the scan's tile sums; the crowded-box list
    const int nb = g.nb;
    const int ntiles = cdiv(nb, kScanTile);
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    const size_t need = 3 * al(sizeof(int) * (size_t)n) + 2 * al(sizeof(int) * ((size_t)nb + 1)) +
                        al(sizeof(int) * (size_t)ntiles) + al(sizeof(int) * (size_t)n) + 256;
    if (need > c->b.pscratch_bytes) {
        if (c->b.pscratch) cudaFree(c->b.pscratch);
        c->b.pscratch = nullptr;
        CUDA_TRY(c, cudaMalloc(&c->b.pscratch, need));
        c->b.pscratch_bytes = need;
    }
    char *p = (char *)c->b.pscratch;
    auto take = [&](size_t bytes) { char *q = p; p += al(bytes); return (int *)q; };
    int *rkey = take(sizeof(int) * (size_t)n), *slot = take(sizeof(int) * (size_t)n);
    int *seg = take(sizeof(int) * (size_t)n);
    int *cnt = take(sizeof(int) * ((size_t)nb + 1)), *off = take(sizeof(int) * ((size_t)nb + 1));
    int *tsum = take(sizeof(int) * (size_t)ntiles), *big = take(sizeof(int) * (size_t)n);
    unsigned *nbig = (unsigned *)take(256);
    const int blk = cdiv(n, kThreads);
    CUDA_TRY(c, cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)nb + 1), st));
    CUDA_TRY(c, cudaMemsetAsync(nbig, 0, sizeof(unsigned), st));
    pres_count<<<blk, kThreads, 0, st>>>(n, c->b.pkey[c->cur_attr], c->mrank, cnt, rkey, slot);
    scan_reduce<<<ntiles, kThreads, 0, st>>>(nb, cnt, tsum);
    scan_tilesums<<<1, 1024, 0, st>>>(ntiles, tsum);
    scan_down<<<ntiles, kThreads, 0, st>>>(nb, cnt, tsum, off, nullptr);
    pres_scatter<<<blk, kThreads, 0, st>>>(n, rkey, slot, off, seg);
    pres_rank<<<blk, kThreads, 0, st>>>(n, rkey, slot, off, seg, c->b.uid[c->cur_attr], c->b.pres, big, nbig);
    pres_rank_big<<<c->sms, 1024, 0, st>>>(big, nbig, off, seg, c->b.uid[c->cur_attr], c->b.pres);
    LAUNCH_CHECK(c);
    c->launches += 7;
    c->pres_state = PRES_VALID;
    return CG_OK;
}

// Automatic skin: sparse pools (48-wide lists) 0.26 L -- builds every ~45
// C4 steps, the middle and short sub-lists keep the swept lists short; dense
// pools 0.07 L (their list width grows with (d + skin)^3).  Measured at C4
// over 180 steps (profiles/r2/ab_r2ac.jsonl, ab_r2aj.jsonl): two levels at
// skin 1.2 / 1.8 / 2.6 -> 1.216 / 1.188 / 1.179 ms per step; three levels at
// 2.6 (middle 1.0, short 0.45) -> 1.165 ms.
static double auto_skin(const cg_context *c, const Geometry &g)
{
    const double surv = 4.19 * (double)c->n / (double)g.nb;
    const bool dense = c->path == 2 || (c->path == 0 && surv > 10.0);
    return (dense ? 0.07 : 0.26) * g.L;
}

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
                sweep7_kernel<T, true, false, 16, false, CG_LIST_BUILD_MINB, true, true><<<g1, kThreads, 0, st>>>(A);
                sweep7_overflow<T, true, false, 16, true, true><<<g2, kThreads, 0, st>>>(A);
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

template <typename T>
static int run_sweep(cg_context *c, const double params[5], bool freeze, bool record, bool build_lists = false)
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
        const int gb = std::min(cdiv(g.nb, kThreads), c->sms * 8);
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
            if (c->list_life < 2) {
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
            // more than skin / 4 (the lists would not serve 2 steps)
            if (build && c->list_width != kListCap && !freeze && !c->last_freeze &&
                4.0 * std::sqrt(std::max(c->bbox_host[7], 0.0)) > c->list_skin_used)
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
        if ((rc = run_sweep<T>(c, params, freeze, record, build))) return rc;
        c->last_kind = build ? 1 : 0;
        S.sweep_kind = build ? 1 : 0;
        if (build) c->list_builds++;
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
        const int gb = std::min(cdiv(g.nb, kThreads), c->sms * 8);
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
            if ((rc = run_sweep<T>(c, params, freeze, record, build))) return rc;
            if (build) {
                if ((rc = slab_list_tables<T>(c))) return rc;
                c->list_builds++;
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

// --------------------------------------------------------------------------- C ABI
// ---------------------------------------------------------------- behaviour phase
template <typename T>
static int behavior_t(cg_context *c, int64_t step_index, double rate, double div_d, bool divide, uint64_t next_uid,
                      int64_t *divisions)
{
    *divisions = 0;
    const int64_t n = c->n;
    if (n == 0) return CG_OK;
    cudaStream_t st = c->stream;
    int rc;
    // daughters take reference positions n, n + 1, ...: the order must be explicit
    if ((rc = materialize_presentation(c))) return rc;
    const int ntiles = cdiv(n, kSortTile);
    auto al = [](size_t v) { return (v + 255) & ~size_t(255); };
    const size_t need = 2 * al(8 * (size_t)n) + 2 * al(4 * (size_t)n) + 2 * al(4 * 256 * (size_t)ntiles + 4) +
                        al(4 * (size_t)cdiv(256 * ntiles, kScanTile)) + 256;
    if (need > c->beh_bytes) {
        if (c->beh) cudaFree(c->beh);
        c->beh = nullptr;
        c->beh_bytes = 0;
        CUDA_TRY(c, cudaMalloc(&c->beh, need));
        c->beh_bytes = need;
    }
    char *p = (char *)c->beh;
    auto take = [&](size_t b) { char *q = p; p += al(b); return (void *)q; };
    uint64_t *key0 = (uint64_t *)take(8 * (size_t)n), *key1 = (uint64_t *)take(8 * (size_t)n);
    int *idx0 = (int *)take(4 * (size_t)n), *idx1 = (int *)take(4 * (size_t)n);
    int *hist = (int *)take(4 * 256 * (size_t)ntiles + 4), *offs = (int *)take(4 * 256 * (size_t)ntiles + 4);
    int *tsum = (int *)take(4 * (size_t)cdiv(256 * ntiles, kScanTile));
    unsigned *nripe = (unsigned *)take(256);
    CUDA_TRY(c, cudaMemsetAsync(nripe, 0, sizeof(unsigned), st));
    Rec<T> *rec = (Rec<T> *)c->b.rec[c->cur_pos];
    grow_kernel<T><<<cdiv(n, kThreads), kThreads, 0, st>>>((int)n, rec, c->b.uid[c->cur_attr], (T)rate, (T)div_d, divide,
                                                           key0, idx0, nripe);
    LAUNCH_CHECK(c);
    c->launches += 1;
    unsigned k = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&k, nripe, sizeof k, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    if (k > 0) {
        if (n + (int64_t)k >= (int64_t)INT32_MAX / 4)
            return fail(c, CG_ERR_POOL_CAPACITY, "%lld agents exceeds the device cap", (long long)(n + k));
        // mothers by uid (the order daughters take uids and places in): LSD radix
        // passes over the bytes in which the ripe uids differ
        unsigned long long oa[2] = {0ull, ~0ull};
        unsigned long long *doa = (unsigned long long *)(nripe + 2);
        CUDA_TRY(c, cudaMemcpyAsync(doa, oa, sizeof oa, cudaMemcpyHostToDevice, st));
        key_or_and<<<std::min(cdiv(k, kThreads), c->sms * 4), kThreads, 0, st>>>((int)k, key0, doa);
        CUDA_TRY(c, cudaMemcpyAsync(oa, doa, sizeof oa, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(c, cudaStreamSynchronize(st));
        const uint64_t vary = oa[0] ^ oa[1];
        const int kt = cdiv(k, kSortTile);
        const int nh = 256 * kt;
        for (int sh = 0; sh < 64; sh += 8) {
            if (!((vary >> sh) & 0xff)) continue;
            radix_hist<<<kt, kThreads, 0, st>>>((int)k, key0, sh, hist, kt);
            const int nt = cdiv(nh, kScanTile);
            scan_reduce<<<nt, kThreads, 0, st>>>(nh, hist, tsum);
            scan_tilesums<<<1, 1024, 0, st>>>(nt, tsum);
            scan_down<<<nt, kThreads, 0, st>>>(nh, hist, tsum, offs, nullptr);
            radix_scatter<<<kt, kThreads, 0, st>>>((int)k, key0, idx0, key1, idx1, sh, offs, kt);
            LAUNCH_CHECK(c);
            c->launches += 5;
            std::swap(key0, key1);
            std::swap(idx0, idx1);
        }
        if (n + (int64_t)k > c->cap) {   // room for the daughters (the pool at most doubles per step)
            const int64_t want = std::max<int64_t>(n + k, std::min<int64_t>(2 * n, (int64_t)INT32_MAX / 4 - 1));
            // the ripe list lives in c->beh, which grow_agents leaves alone
            if ((rc = grow_agents(c, want))) return rc;
            rec = (Rec<T> *)c->b.rec[c->cur_pos];
        }
        divide_kernel<T><<<cdiv(k, kThreads), kThreads, 0, st>>>(
            (int)k, (int)n, key0, idx0, rec, (T *)c->b.adh[c->cur_attr], c->b.uid[c->cur_attr], (T *)c->b.disp[0],
            (T *)c->b.disp[1], (T *)c->b.disp[2], c->pres_state == PRES_VALID ? c->b.pres : nullptr, next_uid,
            (uint64_t)step_index);
        LAUNCH_CHECK(c);
        c->launches += 1;
        c->n = c->n_owned = n + k;
        const uint64_t last = next_uid + k - 1;
        c->uid32 = c->uid32 && last < (1ull << 32);
        c->max_uid = std::max<uint64_t>(c->max_uid, last);
    }
    // new diameters (and daughters): the largest diameter and the bbox are recomputed
    CUDA_TRY(c, cudaMemsetAsync(c->maxd_enc, 0, 2 * sizeof(unsigned long long), st));
    max_diam_kernel<T><<<std::min(c->sms * 4, cdiv(c->n, kThreads)), kThreads, 0, st>>>((int)c->n, rec, c->maxd_enc);
    LAUNCH_CHECK(c);
    c->launches += 1;
    unsigned long long enc[2] = {0, 0};
    CUDA_TRY(c, cudaMemcpyAsync(enc, c->maxd_enc, sizeof enc, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    c->max_diam = dec_ordered(enc[0]);
    c->min_diam = c->n ? -dec_ordered(enc[1]) : -INFINITY;
    c->bbox_valid = false;
    c->list_valid = false;      // lists were built for the old radii
    c->last_kind = 0;
    c->have_grid = false;
    c->grid_current = false;
    c->relaid = false;
    *divisions = k;
    return CG_OK;
}

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
    c->sms = prop.multiProcessorCount;
    c->prec = precision;
    c->esz = precision == CG_FP64 ? 8 : 4;
    int rc = CG_OK;
    // test hook: CG_LIST_SKIN_DEFAULT sets the initial neighbour-list skin of
    // every new context, in LENGTH units ("auto" or a negative value = auto,
    // 0 = lists off); anything else is refused rather than guessed
    if (const char *e = std::getenv("CG_LIST_SKIN_DEFAULT")) {
        char *end = nullptr;
        const double v = std::strtod(e, &end);
        if (std::strcmp(e, "auto") == 0) {
            c->list_skin = -1.0;
        } else if (end == e || *end != '\0' || !std::isfinite(v)) {
            rc = fail(c, CG_ERR_VALUE, "CG_LIST_SKIN_DEFAULT='%s' is not a length (e.g. 0.7, 0, auto)", e);
            std::fprintf(stderr, "cellgrid_b200: %s\n", c->err.c_str());
        } else {
            c->list_skin = v < 0 ? -1.0 : v;
        }
    }
    auto chk = [&](cudaError_t e) {
        if (e != cudaSuccess && rc == CG_OK) rc = fail(c, CG_ERR_CUDA, "%s", cudaGetErrorString(e));
    };
    chk(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    chk(cudaMalloc(&c->slots, sizeof(unsigned long long) * kSlots * kSlotWords));
    chk(cudaMalloc(&c->maxd_enc, 2 * sizeof(unsigned long long)));
    chk(cudaMalloc(&c->ovf_count, sizeof(unsigned)));
    chk(cudaMalloc(&c->block_counters, sizeof(unsigned long long) * 3 * kMaxCounterBlocks));
    chk(cudaMalloc(&c->bbox_dev, sizeof(double) * 16));
    chk(cudaMallocHost(&c->bbox_host, sizeof(double) * 16));
    chk(cudaMalloc(&c->stat_dev, sizeof(unsigned long long) * kStatSlots * kRing));
    chk(cudaMallocHost(&c->stat_host, sizeof(unsigned long long) * kStatSlots * kRing));
    for (int r = 0; r < kRing; ++r)
        for (int e = 0; e < 5; ++e) chk(cudaEventCreate(&c->ev[r][e]));
    if (rc == CG_OK) {
        init_slots<<<16, kThreads, 0, c->stream>>>(c->slots);
        chk(cudaGetLastError());
        chk(cudaStreamSynchronize(c->stream));
    }
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
    {
        auto &S = c->slab;
        void *sp[] = {S.dest, S.out, S.holes, S.movers, S.cnt, S.counts, S.seg_off, S.cursor,
                      S.ref_list, S.ref_off, S.r2g, S.mismatch, S.hkey, S.hval};
        for (void *p : sp)
            if (p) cudaFree(p);
    }
    int *ptrs[] = {c->count, c->offset, c->mrank, c->minv, c->count_own};
    for (int *p : ptrs)
        if (p) cudaFree(p);
    void *vptrs[] = {c->scan_status, c->slots, c->maxd_enc, c->ovf_count, c->block_counters, c->bbox_dev, c->stat_dev,
                     c->maxuid_dev, c->big, c->ovf2, c->ovf2_count, c->beh};
    for (void *p : vptrs)
        if (p) cudaFree(p);
    if (c->bbox_host) cudaFreeHost(c->bbox_host);
    if (c->stat_host) cudaFreeHost(c->stat_host);
    for (int r = 0; r < kRing; ++r)
        for (int e = 0; e < 5; ++e)
            if (c->ev[r][e]) cudaEventDestroy(c->ev[r][e]);
    if (c->stream) cudaStreamDestroy(c->stream);
    if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
    if (c->early.buf) cudaFree(c->early.buf);
    if (c->early.grid_done) cudaEventDestroy(c->early.grid_done);
    if (c->early.ready) cudaEventDestroy(c->early.ready);
    for (int k = 0; k < 9; ++k) {
        if (c->dl_ready[k]) cudaEventDestroy(c->dl_ready[k]);
        if (c->dl_done[k]) cudaEventDestroy(c->dl_done[k]);
    }
    if (c->dl_start) cudaEventDestroy(c->dl_start);
    delete c;
}

const char *cg_last_error(const cg_context *c) { return c ? c->err.c_str() : "null context"; }

void *cg_stream(cg_context *c) { return c ? (void *)c->stream : nullptr; }

int64_t cg_count(const cg_context *c) { return c ? c->n_owned : -1; }   // agents owned (a slab also holds ghosts)

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
    if (key == CG_OPT_SWEEP && value >= 0 && value <= 1) {
        c->sweep_impl = value;
        return CG_OK;
    }
    if (key == CG_OPT_RELAYOUT_EVERY && value >= 1) {
        c->relayout_every = value;
        return CG_OK;
    }
    if (key == CG_OPT_PATH && value >= 0 && value <= 2) {
        c->path = value;
        return CG_OK;
    }
    if (key == CG_OPT_MID_LIST && value >= 0) {
        c->lvl_frac[1] = value * 1e-3;
        c->lvl_valid[1] = c->lvl_valid[2] = false;
        c->list_valid = false;
        c->nbr_width = 0;   // the list buffers are reallocated (with or without this level) at the next build
        return CG_OK;
    }
    if (key == CG_OPT_INNER_LIST && value >= 0) {
        c->lvl_frac[2] = value * 1e-3;
        c->lvl_valid[2] = false;
        c->list_valid = false;
        c->nbr_width = 0;   // the list buffers are reallocated at the next build
        return CG_OK;
    }
    if (key == CG_OPT_LIST_SKIN && value >= -1) {
        c->list_skin = value < 0 ? -1.0 : value * 1e-3;
        c->list_valid = false;
        c->last_kind = 0;
        return CG_OK;
    }
    return fail(c, CG_ERR_VALUE, "bad option %d=%d", key, value);
}

int cg_upload(cg_context *c, int64_t n, const void *px, const void *py, const void *pz,
              const void *diameter, const void *adherence, const uint64_t *uid)
{
    if (!c) return CG_ERR_VALUE;
    if (n < 0) return fail(c, CG_ERR_VALUE, "negative agent count");
    if (n >= (int64_t)INT32_MAX / 4)
        return fail(c, CG_ERR_POOL_CAPACITY, "%lld agents exceeds the device cap", (long long)n);
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (n > c->cap) {
        int rc = alloc_agents(c, n);
        if (rc) return rc;
    }
    c->n = n;
    c->n_owned = n;
    c->list_valid = false;
    c->last_kind = 0;
    // lists pay off only over consecutive resident steps: none on the first
    // step after an upload (a caller that uploads before every step, like
    // engine.step, never pays for a build)
    c->list_wait = std::max(c->list_wait, 1);
    c->grid_current = false;
    c->slab.planned = false;
    c->cur_pos = c->cur_attr = 0;
    c->have_grid = false;
    c->relaid = false;
    c->bbox_valid = false;
    c->pres_state = PRES_IDENTITY;
    c->sort_steps = 0;
    if (n == 0) return CG_OK;
    const size_t fe = c->esz * (size_t)n;
    cudaStream_t st = c->stream;
    // SoA columns land in scratch (the displacement columns and the staging
    // buffer) and are packed into records
    const void *src[4] = {px, py, pz, diameter};
    void *tmp4[4] = {c->b.disp[0], c->b.disp[1], c->b.disp[2], c->b.stage};
    for (int a = 0; a < 4; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(tmp4[a], src[a], fe, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.adh[0], adherence, fe, cudaMemcpyHostToDevice, st));
    CUDA_TRY(c, cudaMemcpyAsync(c->b.uid[0], uid, sizeof(uint64_t) * n, cudaMemcpyHostToDevice, st));
    const int nblk = cdiv(n, kThreads);
    if (c->prec == CG_FP64)
        pack_records<double><<<nblk, kThreads, 0, st>>>((int)n, (const double *)tmp4[0], (const double *)tmp4[1],
                                                        (const double *)tmp4[2], (const double *)tmp4[3],
                                                        (Rec<double> *)c->b.rec[0]);
    else
        pack_records<float><<<nblk, kThreads, 0, st>>>((int)n, (const float *)tmp4[0], (const float *)tmp4[1],
                                                       (const float *)tmp4[2], (const float *)tmp4[3],
                                                       (Rec<float> *)c->b.rec[0]);
    for (int a = 0; a < 3; ++a) CUDA_TRY(c, cudaMemsetAsync(c->b.disp[a], 0, fe, st));
    CUDA_TRY(c, cudaMemsetAsync(c->maxd_enc, 0, 2 * sizeof(unsigned long long), st));
    if (!c->maxuid_dev) CUDA_TRY(c, cudaMalloc(&c->maxuid_dev, sizeof(unsigned long long)));
    CUDA_TRY(c, cudaMemsetAsync(c->maxuid_dev, 0, sizeof(unsigned long long), st));
    max_uid_kernel<<<std::min(c->sms * 4, nblk), kThreads, 0, st>>>((int)n, c->b.uid[0], c->maxuid_dev);
    if (c->prec == CG_FP64)
        max_diam_kernel<double><<<std::min(c->sms * 4, nblk), kThreads, 0, st>>>(
            (int)n, (const Rec<double> *)c->b.rec[0], c->maxd_enc);
    else
        max_diam_kernel<float><<<std::min(c->sms * 4, nblk), kThreads, 0, st>>>(
            (int)n, (const Rec<float> *)c->b.rec[0], c->maxd_enc);
    LAUNCH_CHECK(c);
    c->launches += 3;
    unsigned long long enc[2] = {0, 0}, mu = 0;
    CUDA_TRY(c, cudaMemcpyAsync(enc, c->maxd_enc, sizeof enc, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaMemcpyAsync(&mu, c->maxuid_dev, sizeof mu, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));   // host buffers are only borrowed
    c->max_diam = dec_ordered(enc[0]);
    c->min_diam = n ? -dec_ordered(enc[1]) : -INFINITY;
    c->uid32 = mu < (1ull << 32);
    c->max_uid = mu;
    return CG_OK;
}

static int download_cols(cg_context *c, void *const dst_in[9])
{
    const int64_t n = c->n_owned;   // a slab keeps its ghosts after the owned agents
    if (n == 0) return CG_OK;
    int rc = materialize_presentation(c);
    if (rc) return rc;
    if ((rc = ensure_copy_stream(c))) return rc;
    void *dst[9];
    for (int k = 0; k < 9; ++k) dst[k] = dst_in[k];
    const void *src[9] = {nullptr, nullptr, nullptr, nullptr, c->b.adh[c->cur_attr], c->b.uid[c->cur_attr],
                          c->b.disp[0], c->b.disp[1], c->b.disp[2]};
    cudaStream_t st = c->stream, cs = c->copy_stream;
    const int *pres = c->pres_state == PRES_IDENTITY ? nullptr : c->b.pres;
    // staging ring (8 n bytes each): the download buffer and the idle record
    // buffer (the next step's output); column k is produced on the context
    // stream into ring[k % R] and copied on the copy stream, so the unpack /
    // reorder kernels run under the PCIe transfers
    char *ring[5];
    int R = 0;
    ring[R++] = (char *)c->b.stage;
    const size_t colb = 8 * (size_t)n;
    for (size_t off = 0; off + colb <= 4 * c->esz * (size_t)c->cap && R < 5; off += colb)
        ring[R++] = (char *)c->b.rec[1 - c->cur_pos] + off;
    CUDA_TRY(c, cudaEventRecord(c->dl_start, st));
    CUDA_TRY(c, cudaStreamWaitEvent(cs, c->dl_start, 0));
    int used = 0;
    for (int k = 0; k < 9; ++k) {
        if (!dst[k]) continue;
        const size_t w = k == 5 ? 8 : c->esz;
        if (k >= 4 && !pres) {   // storage order is the reference's: straight copy
            CUDA_TRY(c, cudaMemcpyAsync(dst[k], src[k], w * n, cudaMemcpyDeviceToHost, cs));
            continue;
        }
        const int slot = used % R;
        if (used >= R) CUDA_TRY(c, cudaStreamWaitEvent(st, c->dl_done[used - R], 0));
        void *buf = ring[slot];
        if (k < 4) {   // record components
            if (c->prec == CG_FP64)
                unpack_component<double><<<cdiv(n, kThreads), kThreads, 0, st>>>(
                    (int)n, (const Rec<double> *)c->b.rec[c->cur_pos], k, pres, (double *)buf);
            else
                unpack_component<float><<<cdiv(n, kThreads), kThreads, 0, st>>>(
                    (int)n, (const Rec<float> *)c->b.rec[c->cur_pos], k, pres, (float *)buf);
        } else if (w == 8) {
            scatter_by<unsigned long long><<<cdiv(n, kThreads), kThreads, 0, st>>>(
                (int)n, pres, (const unsigned long long *)src[k], (unsigned long long *)buf);
        } else {
            scatter_by<unsigned><<<cdiv(n, kThreads), kThreads, 0, st>>>((int)n, pres, (const unsigned *)src[k],
                                                                          (unsigned *)buf);
        }
        LAUNCH_CHECK(c);
        c->launches += 1;
        CUDA_TRY(c, cudaEventRecord(c->dl_ready[used], st));
        CUDA_TRY(c, cudaStreamWaitEvent(cs, c->dl_ready[used], 0));
        CUDA_TRY(c, cudaMemcpyAsync(dst[k], buf, w * n, cudaMemcpyDeviceToHost, cs));
        CUDA_TRY(c, cudaEventRecord(c->dl_done[used], cs));
        ++used;
    }
    CUDA_TRY(c, cudaStreamSynchronize(cs));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    return CG_OK;
}

int cg_download(cg_context *c, void *px, void *py, void *pz, void *diameter, void *adherence,
                uint64_t *uid, void *dx, void *dy, void *dz)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    void *dst[9] = {px, py, pz, diameter, adherence, uid, dx, dy, dz};
    return download_cols(c, dst);
}

int cg_step_download(cg_context *c, const double params[5], double interaction_radius, int64_t box_cap, int flags,
                     cg_step_stats *stats, void *px, void *py, void *pz, void *diameter, void *adherence,
                     uint64_t *uid, void *dx, void *dy, void *dz)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    c->early = cg_context::Early{false, false, {diameter, adherence, uid}, c->early.buf, c->early.bytes,
                                 c->early.grid_done, c->early.ready};
    c->early.want = c->n == c->n_owned && c->n > 0;
    int rc = cg_step(c, params, interaction_radius, box_cap, flags, stats);
    const bool early = c->early.done;
    c->early.want = c->early.done = false;
    if (rc) {
        if (early) cudaStreamSynchronize(c->copy_stream);
        return rc;
    }
    void *dst[9] = {px, py, pz, early ? nullptr : diameter, early ? nullptr : adherence, early ? nullptr : (void *)uid,
                    dx, dy, dz};
    if (early) CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->early.ready, 0));   // pres + early buffers
    return download_cols(c, dst);
}

int cg_step(cg_context *c, const double params[5], double interaction_radius, int64_t box_cap,
            int flags, cg_step_stats *stats)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    int64_t id = -1;
    c->grid_current = false;
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
                       ? build_grid<double>(c, interaction_radius, box_cap, false, false, origin, dims64)
                       : build_grid<float>(c, interaction_radius, box_cap, false, false, origin, dims64);
    if (rc) return rc;
    c->grid_current = true;
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
    int rc = materialize_presentation(c);
    if (rc) return rc;
    const int n = (int)c->n, nb = c->geo.nb;
    cudaStream_t st = c->stream;
    if (box_index) {
        // after a relayout the storage index is the slot: its box is skey
        const int *keys = c->b.skey;
        if (!c->relaid) {
            key_of_storage<<<cdiv(n, kThreads), kThreads, 0, st>>>(n, c->b.key_rank, c->b.tmp);
            LAUNCH_CHECK(c);
            keys = c->b.tmp;
        }
        std::vector<int> k(n);
        if ((rc = download_column(c, keys, k.data(), 4))) return rc;
        CUDA_TRY(c, cudaStreamSynchronize(st));
        for (int i = 0; i < n; ++i) box_index[i] = k[i];
    }
    if (box_count) {
        std::vector<int> off(nb + 1);
        CUDA_TRY(c, cudaMemcpyAsync(off.data(), c->offset, sizeof(int) * (nb + 1), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(c, cudaStreamSynchronize(st));
        for (int b = 0; b < nb; ++b) box_count[b] = off[b + 1] - off[b];
    }
    return CG_OK;
}

int cg_record_export(cg_context *c, int32_t *m, int32_t *nk)
{
    if (!c) return CG_ERR_VALUE;
    if (!c->last_record) return fail(c, CG_ERR_STATE, "last step did not run with CG_STEP_RECORD");
    CUDA_TRY(c, cudaSetDevice(c->device));
    int rc = materialize_presentation(c);
    if (rc) return rc;
    if (m && (rc = download_column(c, c->b.rec_m, m, 4))) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (nk && (rc = download_column(c, c->b.rec_nk, nk, 4))) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
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
    c->n = c->n_owned = 0;   // the resident pool is overwritten by this call
    c->have_grid = false;
    c->bbox_valid = false;
    c->pres_state = PRES_IDENTITY;
    Geometry g{box_length, ox, oy, oz, (int)dimx, (int)dimy, (int)dimz, (int)(dimx * dimy * dimz), 0, (int)dimx};
    const size_t fe = c->esz * (size_t)n;
    const void *src[3] = {px, py, pz};
    for (int a = 0; a < 3; ++a)   // the displacement columns serve as scratch
        CUDA_TRY(c, cudaMemcpyAsync(c->b.disp[a], src[a], fe, cudaMemcpyHostToDevice, c->stream));
    long long *dout = (long long *)c->b.stage;
    if (c->prec == CG_FP64)
        box_ids_only<double><<<cdiv(n, kThreads), kThreads, 0, c->stream>>>(
            (int)n, g, (double *)c->b.disp[0], (double *)c->b.disp[1], (double *)c->b.disp[2], dout);
    else
        box_ids_only<float><<<cdiv(n, kThreads), kThreads, 0, c->stream>>>(
            (int)n, g, (float *)c->b.disp[0], (float *)c->b.disp[1], (float *)c->b.disp[2], dout);
    LAUNCH_CHECK(c);
    c->launches += 1;
    CUDA_TRY(c, cudaMemcpyAsync(out, dout, sizeof(long long) * n, cudaMemcpyDeviceToHost, c->stream));
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
    if (nb64 >= (int64_t)INT32_MAX / 2) return fail(c, CG_ERR_GRID_OVERFLOW, "too many boxes");
    if ((rc = ensure_boxes(c, nb64))) return rc;
    Geometry g{1.0, 0.0, 0.0, 0.0, (int)dimx, (int)dimy, (int)dimz, (int)nb64, 0, (int)dimx};
    c->geo = g;
    c->bd = make_decode(g);
    const int nblk = cdiv(nn, kThreads);
    if (nblk > kMaxCounterBlocks) return fail(c, CG_ERR_VALUE, "population too large");
    // radii were uploaded in the diameter slot: double them (exact)
    if (c->prec == CG_FP64) double_diameter<double><<<nblk, kThreads, 0, st>>>(nn, (Rec<double> *)c->b.rec[0]);
    else double_diameter<float><<<nblk, kThreads, 0, st>>>(nn, (Rec<float> *)c->b.rec[0]);
    c->min_diam = -INFINITY;
    long long *dbox = (long long *)c->b.stage;
    CUDA_TRY(c, cudaMemcpyAsync(dbox, box_index, sizeof(long long) * n, cudaMemcpyHostToDevice, st));
    keys_from_flat<<<nblk, kThreads, 0, st>>>(nn, dbox, c->count, c->b.key_rank);
    LAUNCH_CHECK(c);
    const int slot = (int)(c->steps_done % kRing);
    unsigned long long *stat = c->stat_dev + slot * kStatSlots;
    CUDA_TRY(c, cudaMemsetAsync(stat, 0, sizeof(unsigned long long) * kStatSlots, st));
    if ((rc = launch_scan(c, g.nb, c->offset, stat))) return rc;
    place<<<nblk, kThreads, 0, st>>>(nn, c->b.key_rank, c->offset, c->b.tmp);
    if (c->prec == CG_FP64)
        order_gather<double, false><<<nblk, kThreads, 0, st>>>(
            nn, g, c->bd, c->b.tmp, c->b.key_rank, c->offset, (const Rec<double> *)c->b.rec[0],
            (double *)c->b.adh[0], c->b.uid[0], c->b.skey, c->b.P(), c->b.idx, nullptr, nullptr, nullptr, nullptr);
    else
        order_gather<float, false><<<nblk, kThreads, 0, st>>>(
            nn, g, c->bd, c->b.tmp, c->b.key_rank, c->offset, (const Rec<float> *)c->b.rec[0],
            (float *)c->b.adh[0], c->b.uid[0], c->b.skey, c->b.P(), c->b.idx, nullptr, nullptr, nullptr, nullptr);
    LAUNCH_CHECK(c);
    c->launches += 5;
    c->relaid = false;
    // the kernel-level call has no box_length: use the reference-order sweep
    const int saved = c->sweep_impl;
    c->sweep_impl = 0;
    double p5[5];
    for (int k = 0; k < 5; ++k)
        p5[k] = c->prec == CG_FP64 ? ((const double *)params7)[k] : (double)((const float *)params7)[k];
    rc = c->prec == CG_FP64 ? run_sweep<double>(c, p5, true, false) : run_sweep<float>(c, p5, true, false);
    c->sweep_impl = saved;
    if (rc) return rc;
    unsigned long long h[kStatSlots];
    CUDA_TRY(c, cudaMemcpyAsync(h, stat, sizeof h, cudaMemcpyDeviceToHost, st));
    const size_t fe = c->esz * (size_t)n;
    void *dst[3] = {out_dx, out_dy, out_dz};
    for (int a = 0; a < 3; ++a)
        CUDA_TRY(c, cudaMemcpyAsync(dst[a], c->b.disp[a], fe, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    counters[0] = (int64_t)h[2];
    counters[1] = (int64_t)h[3];
    counters[2] = (int64_t)h[4];
    c->n = c->n_owned = 0;   // the resident buffers no longer hold a consistent pool
    c->have_grid = false;
    c->bbox_valid = false;
    return CG_OK;
}

int64_t cg_record_bytes(const cg_context *c)
{
    if (!c) return -1;
    return (int64_t)(c->esz == 8 ? sizeof(SlabRecord<double>) : sizeof(SlabRecord<float>));
}

int cg_reserve(cg_context *c, int64_t capacity)
{
    if (!c) return CG_ERR_VALUE;
    if (c->n > 0) return fail(c, CG_ERR_STATE, "cg_reserve must precede cg_upload");
    if (capacity >= (int64_t)INT32_MAX / 4) return fail(c, CG_ERR_POOL_CAPACITY, "capacity too large");
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (capacity > c->cap) return alloc_agents(c, capacity);
    return CG_OK;
}

int cg_local_bbox(cg_context *c, double out[11])
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (c->n_owned == 0) {
        out[0] = out[1] = out[2] = INFINITY;
        out[3] = out[4] = out[5] = -INFINITY;
        out[6] = c->max_diam;
        out[7] = 0.0;
        out[8] = c->last_kind == 2 ? 0.0 : 1.0;   // no lists of its own: veto list steps
        out[9] = -INFINITY;                       // no diameters of its own
        out[10] = 0.0;
        return CG_OK;
    }
    int rc = CG_OK;
    unsigned bad = 0;
    if (c->slab.mismatch)   // ghost refreshes of the last step (slab_unpack_t)
        CUDA_TRY(c, cudaMemcpyAsync(&bad, c->slab.mismatch, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    if (!c->bbox_valid)
        rc = c->prec == CG_FP64 ? standalone_bbox<double>(c) : standalone_bbox<float>(c);
    else
        CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (rc) return rc;
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (bad) return fail(c, CG_ERR_STATE, "ghost refresh: %u records did not match the ghost set", bad);
    for (int k = 0; k < 6; ++k) out[k] = c->bbox_host[k];
    out[6] = c->max_diam;
    // the last step's largest squared displacement and neighbour-list
    // overflows (all-reduced with the bbox for the list decision)
    out[7] = c->last_kind != 0 && !c->last_freeze ? c->bbox_host[7] : 0.0;
    // list veto: overflows of a build, or 1 when this rank neither built lists
    // nor ran a list step last (every rank must take the same decision)
    out[8] = c->last_kind == 1 ? c->bbox_host[8] : (c->last_kind == 2 ? 0.0 : 1.0);
    // -min diameter of the owned agents: the slab's own minimum until ghosts
    // or arrivals widened the range (min_diam is then the global one)
    out[9] = std::isfinite(c->min_diam) ? -c->min_diam : -INFINITY;
    // the largest uid (all-reduced: 32-bit survivor sort keys when every uid
    // of the global pool is below 2^32); rounded up to a double
    out[10] = c->max_uid < (1ull << 53) ? (double)c->max_uid : 1.8446744073709552e19;
    return CG_OK;
}

int cg_slab_plan(cg_context *c, const double bbox[11], double interaction_radius, int64_t box_cap, int world,
                 int rank, int64_t *counts, int64_t planes[2])
{
    if (!c) return CG_ERR_VALUE;
    if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world) return fail(c, CG_ERR_VALUE, "bad world/rank");
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (c->slab.planned) return fail(c, CG_ERR_STATE, "cg_slab_plan twice without cg_slab_step");
    return c->prec == CG_FP64 ? slab_plan_t<double>(c, bbox, interaction_radius, box_cap, world, rank, counts, planes)
                              : slab_plan_t<float>(c, bbox, interaction_radius, box_cap, world, rank, counts, planes);
}

int cg_slab_pack(cg_context *c, void *send)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (!c->slab.planned || c->slab.packed) return fail(c, CG_ERR_STATE, "cg_slab_pack needs a fresh cg_slab_plan");
    return c->prec == CG_FP64 ? slab_pack_t<double>(c, send) : slab_pack_t<float>(c, send);
}

int cg_slab_unpack(cg_context *c, const void *recv, const int64_t *recv_counts)
{
    if (!c || !recv_counts) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (!c->slab.packed) return fail(c, CG_ERR_STATE, "cg_slab_unpack without cg_slab_pack");
    if (c->slab.unpacked) return fail(c, CG_ERR_STATE, "cg_slab_unpack called twice");
    return c->prec == CG_FP64 ? slab_unpack_t<double>(c, recv, recv_counts)
                              : slab_unpack_t<float>(c, recv, recv_counts);
}

int cg_slab_step_interior(cg_context *c, const double params[5], int flags)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    auto &S = c->slab;
    if (!S.planned || !S.packed || S.unpacked)
        return fail(c, CG_ERR_STATE, "cg_slab_step_interior belongs between cg_slab_pack and cg_slab_unpack");
    // nothing to overlap: a rebuild step, no interior, a recorded step, or twice
    if (!S.list_mode || !S.split_ok || (flags & CG_STEP_RECORD) || S.interior_done) return CG_OK;
    const bool freeze = (flags & CG_STEP_FREEZE) != 0;
    return c->prec == CG_FP64 ? slab_list_step<double>(c, params, freeze, false, 1)
                              : slab_list_step<float>(c, params, freeze, false, 1);
}

int cg_slab_step(cg_context *c, const double params[5], int flags, cg_step_stats *stats)
{
    if (!c) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    int64_t id = -1;
    const int rc = c->prec == CG_FP64 ? slab_step_t<double>(c, params, flags, &id)
                                      : slab_step_t<float>(c, params, flags, &id);
    if (rc) return rc;
    if (stats) return collect(c, id, stats);
    return CG_OK;
}

// ---------------------------------------------------------------- radius queries
}  // extern "C"

template <typename T>
static int neighbor_query_t(cg_context *c, double radius, int64_t *counts, const int64_t *indptr,
                            int64_t *indices)
{
    const int n = (int)c->n;
    cudaStream_t st = c->stream;
    int rc = materialize_presentation(c);
    if (rc) return rc;
    QueryArgs<T> Q{};
    Q.n = n;
    Q.g = c->geo;
    Q.bd = c->bd;
    Q.skey = c->b.skey;
    Q.idx = c->relaid ? nullptr : c->b.idx;
    Q.off = c->offset;
    Q.rec = (const Rec<T> *)c->b.rec[c->cur_pos];
    Q.uid = c->b.uid[c->cur_attr];
    Q.pres = c->pres_state == PRES_IDENTITY ? nullptr : c->b.pres;
    Q.r2 = radius * radius;
    if (counts) {
        Q.counts = (long long *)c->b.stage;
        neighbor_kernel<T, false><<<cdiv(n, kThreads), kThreads, 0, st>>>(Q);
        LAUNCH_CHECK(c);
        c->launches += 1;
        CUDA_TRY(c, cudaMemcpyAsync(counts, c->b.stage, sizeof(int64_t) * n, cudaMemcpyDeviceToHost, st));
        CUDA_TRY(c, cudaStreamSynchronize(st));
        return CG_OK;
    }
    const int64_t total = indptr[n];
    long long *dptr = nullptr, *dind = nullptr;
    int *inv = nullptr;
    CUDA_TRY(c, cudaMallocAsync(&dptr, sizeof(long long) * (n + 1), st));
    CUDA_TRY(c, cudaMallocAsync(&dind, sizeof(long long) * std::max<int64_t>(total, 1), st));
    CUDA_TRY(c, cudaMemcpyAsync(dptr, indptr, sizeof(long long) * (n + 1), cudaMemcpyHostToDevice, st));
    Q.indptr = dptr;
    Q.indices = dind;
    neighbor_kernel<T, true><<<cdiv(n, kThreads), kThreads, 0, st>>>(Q);
    if (Q.pres) {   // reference position -> storage index, for the uids of row entries
        CUDA_TRY(c, cudaMallocAsync(&inv, sizeof(int) * n, st));
        invert_perm<<<cdiv(n, kThreads), kThreads, 0, st>>>(n, Q.pres, inv);
    }
    sort_rows_by_uid<<<cdiv(n, kThreads), kThreads, 0, st>>>(n, dptr, dind, inv, Q.uid);
    LAUNCH_CHECK(c);
    c->launches += Q.pres ? 3 : 2;
    if (total > 0)
        CUDA_TRY(c, cudaMemcpyAsync(indices, dind, sizeof(int64_t) * total, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(c, cudaFreeAsync(dptr, st));
    CUDA_TRY(c, cudaFreeAsync(dind, st));
    if (inv) CUDA_TRY(c, cudaFreeAsync(inv, st));
    CUDA_TRY(c, cudaStreamSynchronize(st));
    return CG_OK;
}

static int neighbor_check(cg_context *c, double radius)
{
    if (!c->grid_current || c->n != c->n_owned)
        return fail(c, CG_ERR_STATE, "no grid over the stored positions: call cg_build_grid first");
    if (!(radius > 0)) return fail(c, CG_ERR_VALUE, "radius must be positive, got %g", radius);
    if (radius > c->geo.L)
        return fail(c, CG_ERR_STENCIL, "radius %g exceeds box_length %g", radius, c->geo.L);
    return CG_OK;
}

extern "C" {

int64_t cg_slab_list_epoch(const cg_context *c)
{
    if (!c) return -1;
    return c->slab.planned && c->slab.list_mode ? c->list_builds : -1;
}

int cg_behavior(cg_context *c, int64_t step_index, double volume_growth_rate, double division_diameter,
                int division_enabled, uint64_t next_uid, int64_t *divisions)
{
    if (!c || !divisions) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (c->n_owned != c->n) return fail(c, CG_ERR_STATE, "cg_behavior on a slab context with ghosts");
    return c->prec == CG_FP64 ? behavior_t<double>(c, step_index, volume_growth_rate, division_diameter,
                                                   division_enabled != 0, next_uid, divisions)
                              : behavior_t<float>(c, step_index, volume_growth_rate, division_diameter,
                                                  division_enabled != 0, next_uid, divisions);
}

int cg_unit_vectors(cg_context *c, int64_t n, const uint64_t *uid, int64_t step, double *out)
{
    if (!c || n < 0) return CG_ERR_VALUE;
    if (n == 0) return CG_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    uint64_t *du = nullptr;
    double *dv = nullptr;
    CUDA_TRY(c, cudaMalloc(&du, 8 * (size_t)n));
    CUDA_TRY(c, cudaMalloc(&dv, 24 * (size_t)n));
    cudaStream_t st = c->stream;
    CUDA_TRY(c, cudaMemcpyAsync(du, uid, 8 * (size_t)n, cudaMemcpyHostToDevice, st));
    unit_vector_kernel<<<cdiv(n, kThreads), kThreads, 0, st>>>((int)n, du, (uint64_t)step, dv);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(out, dv, 24 * (size_t)n, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(du);
    cudaFree(dv);
    c->launches += 1;
    if (e != cudaSuccess) return fail(c, CG_ERR_CUDA, "cg_unit_vectors: %s", cudaGetErrorString(e));
    return CG_OK;
}

int cg_list_stats(cg_context *c, int64_t out[6])
{
    if (!c || !out) return CG_ERR_VALUE;
    out[0] = c->list_builds;
    out[1] = c->list_steps;
    out[2] = c->list_valid ? 1 : 0;
    out[3] = (int64_t)llround(c->list_skin_used * 1e6);
    out[4] = c->overlapped_steps;
    out[5] = c->inner_steps;
    return CG_OK;
}

int cg_neighbor_counts(cg_context *c, double radius, int64_t *counts)
{
    if (!c || !counts) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    int rc = neighbor_check(c, radius);
    if (rc || c->n == 0) return rc;
    return c->prec == CG_FP64 ? neighbor_query_t<double>(c, radius, counts, nullptr, nullptr)
                              : neighbor_query_t<float>(c, radius, counts, nullptr, nullptr);
}

int cg_neighbor_fill(cg_context *c, double radius, const int64_t *indptr, int64_t *indices)
{
    if (!c || !indptr) return CG_ERR_VALUE;
    CUDA_TRY(c, cudaSetDevice(c->device));
    int rc = neighbor_check(c, radius);
    if (rc || c->n == 0) return rc;
    return c->prec == CG_FP64 ? neighbor_query_t<double>(c, radius, nullptr, indptr, indices)
                              : neighbor_query_t<float>(c, radius, nullptr, indptr, indices);
}

}  // extern "C"


