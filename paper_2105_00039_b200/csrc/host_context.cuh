// host_context.cuh -- part of the cellgrid_b200.cu translation unit (host side):
// context state, device buffers, host geometry (spatial.py:99-116), launch helpers.
// Included once, in order, by cellgrid_b200.cu; not a standalone header.
#pragma once

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
    bool sub_built = false;   // the last list build also wrote both sub-lists (run_sweep)
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
