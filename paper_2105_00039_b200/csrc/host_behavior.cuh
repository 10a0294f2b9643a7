// host_behavior.cuh -- part of the cellgrid_b200.cu translation unit (host side):
// behaviour phase driver (engine.py:191-232), see behavior.cuh.
// Included once, in order, by cellgrid_b200.cu; not a standalone header.
#pragma once

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
