// cellgrid_b200.cu -- the library's single translation unit: the C ABI
// (include/cellgrid_b200.h) over the host driver parts host_context.cuh,
// host_step.cuh, host_slab.cuh and host_behavior.cuh.
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

#include "host_context.cuh"
#include "host_step.cuh"
#include "host_slab.cuh"
#include "host_behavior.cuh"

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


