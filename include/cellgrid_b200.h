/*
 * cellgrid_b200.h -- C ABI of the B200 mechanical-interaction step.
 *
 * Plain pointers and sizes only (no torch / CUDA types).  A context owns all
 * device buffers of one agent population on one GPU; they persist across
 * steps.  Host buffers are borrowed for the duration of a call.  Calls on one
 * context must be serialised by the caller (reference SPEC.md:462: the engine
 * is not shared across concurrent step calls).  Every entry point returns a
 * CG_* status; cg_last_error() holds the message of the last failure.
 *
 * Reference interfaces replaced (paths relative to
 * /root/reference/pkg/src/cellgrid/):
 *   cg_step          engine.py:279-341  step(pool, config, step_index)
 *                    (sort -> grid -> force -> apply, counters of StepStats)
 *   cg_box_ids       kernels.py:107-129 box_ids_parallel(...)
 *   cg_force_phase   kernels.py:302-333 force_phase_parallel(...) -> (evals, cands, ndeg)
 *   cg_build_grid +  spatial.py:89-127  build_grid(...) -> UniformGrid (box_index, box_count)
 *   cg_grid_export
 *   cg_upload/download  the AgentPool SoA columns (pool.py:58-66) crossing the boundary
 * Status codes map 1:1 onto the reference exception classes (see
 * paper_2105_00039_b200/_native.py).
 */
#ifndef CELLGRID_B200_H
#define CELLGRID_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CG_ABI_VERSION 6

/* status codes */
#define CG_OK 0
#define CG_ERR_VALUE 1          /* ValueError (bad argument, empty pool, dtype) */
#define CG_ERR_GRID_OVERFLOW 2  /* spatial.GridOverflowError (spatial.py:111-116) */
#define CG_ERR_STENCIL 3        /* spatial.StencilTooSmallError (spatial.py:143-145) */
#define CG_ERR_POOL_CAPACITY 4  /* pool.PoolCapacityError (pool.py:151-152) */
#define CG_ERR_CUDA 5           /* CUDA runtime failure */
#define CG_ERR_NO_DEVICE 6      /* no sm_100 device / bad ordinal */
#define CG_ERR_STATE 7          /* call out of order (e.g. step before upload) */

/* precision (PrecisionMode, pool.py:34-46) */
#define CG_FP64 0
#define CG_FP32 1

/* cg_step flags */
#define CG_STEP_SORT 1          /* Z-order re-sort due this step (engine.py:305-309) */
#define CG_STEP_FREEZE 2        /* SimulationConfig.freeze_displacement (engine.py:324) */
#define CG_STEP_RECORD 4        /* keep per-agent m / nk for cg_record_export */

/* cg_set_option keys */
#define CG_OPT_SUMMATION 1      /* 0 = uid order (bit-exact vs reference), 1 = stencil order */
#define CG_OPT_SWEEP 3          /* 0 = reference-order thread-per-agent sweep, 1 = production sweep (default) */
#define CG_OPT_RELAYOUT_EVERY 4 /* move the records into slot order on every k-th sort step (k >= 1, default 1) */
#define CG_OPT_PATH 5           /* 0 = auto (by agents per box), 1 = sparse (uid-sorted survivor lists),
                                   2 = dense (boxes ordered by (z, uid), CG_OPT_SUMMATION applies) */
#define CG_OPT_LIST_SKIN 6      /* neighbour-list reuse: -1 = auto (skin 0.26 x box length on sparse pools,
                                   0.07 on dense ones; default), 0 = off, k > 0 = skin of k/1000 length units.
                                   Results are identical with or without it (csrc/list.cuh). */
#define CG_OPT_INNER_LIST 7     /* second-level list on the sparse path: k = 0 off, k > 0 = a sub-list of the
                                   partners within r_i + r_j + (k/1000) x skin, rebuilt from the neighbour
                                   list while the motion allows (default 173) -- identical results */
#define CG_OPT_MID_LIST 8       /* optional middle level: k > 0 = a sub-list within r_i + r_j + (k/1000) x skin
                                   written from the neighbour list, from which the short sub-list is refreshed
                                   (default 385; 0 = off) -- identical results */

typedef struct cg_context cg_context;

/* Per-step statistics: the StepStats fields (engine.py:134-151) the path owns. */
typedef struct {
    int64_t step_id;
    int64_t agent_count;
    int64_t force_evals;        /* ordered pairs with positive overlap */
    int64_t candidates;         /* ordered stencil pairs examined */
    int64_t degenerate_pairs;   /* coincident-centre pairs */
    int64_t grid_dims[3];
    int64_t grid_occupied_boxes;
    int64_t grid_max_occupancy;
    double box_length;
    double origin[3];
    float t_sort_ms, t_grid_ms, t_force_ms, t_total_ms;   /* CUDA-event times */
    int32_t sweep_kind;         /* 0 grid sweep, 1 grid sweep + neighbour-list build, 2 list sweep */
    int32_t reserved;
} cg_step_stats;

int cg_abi_version(void);
int cg_device_count(int *count);

int cg_create(int device, int precision, cg_context **out);
void cg_destroy(cg_context *ctx);
const char *cg_last_error(const cg_context *ctx);
int cg_set_option(cg_context *ctx, int key, int value);
/* Opaque cudaStream_t of the context (for event timing by the caller). */
void *cg_stream(cg_context *ctx);

/* Columns in the context precision; uid is uint64.  n may be 0. */
int cg_upload(cg_context *ctx, int64_t n, const void *px, const void *py, const void *pz,
              const void *diameter, const void *adherence, const uint64_t *uid);
/* Any pointer may be NULL to skip that column.  Columns come back in the
 * reference's storage order: upload order until the first sort step, then the
 * (Morton code, uid) order of the last sort step (morton.py:67-74). */
int cg_download(cg_context *ctx, void *px, void *py, void *pz, void *diameter,
                void *adherence, uint64_t *uid, void *dx, void *dy, void *dz);
int64_t cg_count(const cg_context *ctx);
/* cg_step followed by cg_download, with the transfers overlapped: the columns
 * the step does not change (diameter, adherence, uid, in the reference's new
 * order) are copied to the host while the sweep runs.  Same results. */
int cg_step_download(cg_context *ctx, const double params[5], double interaction_radius, int64_t box_cap,
                     int flags, cg_step_stats *stats, void *px, void *py, void *pz, void *diameter,
                     void *adherence, uint64_t *uid, void *dx, void *dy, void *dz);
/* Kernels launched by this context so far (evidence for bench gpu_launches). */
int64_t cg_launch_count(const cg_context *ctx);
/* Page-locked host memory for staging pool columns (NULL on failure). */
void *cg_host_alloc(int64_t bytes);
void cg_host_free(void *p);

/* One mechanical step.  params = ForceParams (kappa, gamma, timestep,
 * max_displacement, adherence_scale), mechanics.py:47-75.
 * interaction_radius: NaN = None.  box_cap: spatial.DEFAULT_BOX_CAP (1<<24).
 * If stats != NULL the call waits for the step and fills it; otherwise the
 * step is only enqueued and cg_fetch_stats(step_id) collects it later. */
int cg_step(cg_context *ctx, const double params[5], double interaction_radius,
            int64_t box_cap, int flags, cg_step_stats *stats);
int cg_fetch_stats(cg_context *ctx, int64_t step_id, cg_step_stats *stats);
/* Grid only (spatial.py:89-127 build_grid): no sweep, pool unchanged.  Fills
 * the grid fields of stats (dims, origin, box_length, occupancy). */
int cg_build_grid(cg_context *ctx, double interaction_radius, int64_t box_cap,
                  cg_step_stats *stats);
int cg_synchronize(cg_context *ctx);

/* Grid of the last step: box_index per storage index (n), box_count in flat
 * box order (prod(dims)).  Either pointer may be NULL. */
int cg_grid_export(cg_context *ctx, int64_t *box_index, int64_t *box_count);
/* Per-agent stencil candidates m and colliding pairs nk of the last step that
 * ran with CG_STEP_RECORD (storage order). */
int cg_record_export(cg_context *ctx, int32_t *m, int32_t *nk);

/* Kernel-level drop-ins (host buffers in, host buffers out). */
int cg_box_ids(cg_context *ctx, int64_t n, const void *px, const void *py, const void *pz,
               double ox, double oy, double oz, double box_length,
               int64_t dimx, int64_t dimy, int64_t dimz, int64_t *out);
int cg_force_phase(cg_context *ctx, int64_t n, const void *px, const void *py, const void *pz,
                   const void *radii, const void *adherence, const uint64_t *uid,
                   const int64_t *box_index, int64_t dimx, int64_t dimy, int64_t dimz,
                   const void *params7, void *out_dx, void *out_dy, void *out_dz,
                   int64_t counters[3]);

/* ---- behaviour phase: engine.grow_and_divide
 * (engine.py:191-232) on the resident pool, before the step.  Every agent's
 * volume pi/6 d^3 grows by volume_growth_rate (pool dtype), d = cbrt(volume /
 * (pi/6)); with division_enabled, agents with d >= division_diameter split in
 * ascending uid: both halves get d = cbrt(half volume / (pi/6)), the daughter
 * is placed at mother radius / 4 along rng.unit_vector(uid, step_index)
 * (rng.py:41-54) and appended (pool.py:199-217 append_many) with uid next_uid +
 * rank, zero displacement, the mother's adherence.  cbrt is numpy's SVML
 * routine and the direction numpy's Philox + ziggurat, restated bit for bit
 * (csrc/behavior_math.h).  *divisions receives the number of divisions; the
 * caller advances its next_uid by it.  The pool grows in place (capacity is
 * extended as needed); the storage order of existing agents is unchanged. */
int cg_behavior(cg_context *ctx, int64_t step_index, double volume_growth_rate, double division_diameter,
                int division_enabled, uint64_t next_uid, int64_t *divisions);
/* rng.unit_vector(uid[i], step) for n uids (rng.py:41-54): out is n x 3 f64. */
int cg_unit_vectors(cg_context *ctx, int64_t n, const uint64_t *uid, int64_t step, double *out);

/* Neighbour-list reuse counters (CG_OPT_LIST_SKIN): out[0] list builds,
 * out[1] steps served from lists, out[2] lists currently valid, out[3] skin of
 * the last build in 1e-6 length units, out[4] slab list steps whose interior
 * sweep overlapped the ghost refresh, out[5] list steps that swept the
 * sub-list (CG_OPT_INNER_LIST). */
int cg_list_stats(cg_context *ctx, int64_t out[6]);

/* ---- radius queries: kernels.grid_neighbor_counts /
 * grid_neighbor_fill (kernels.py:427-520) behind spatial.neighbor_counts /
 * neighbor_csr (spatial.py:158-169).  Closed-ball f64 predicate
 * d2 <= radius^2 over the 27-box stencil of the grid built by cg_build_grid
 * (CG_ERR_STATE otherwise); radius <= box_length (CG_ERR_STENCIL).  Agents
 * and neighbour indices are in the reference's storage order; every row of the
 * CSR table ascends by neighbour uid.  counts: n int64; indptr: n + 1 int64
 * (exclusive prefix of the counts); indices: indptr[n] int64. */
int cg_neighbor_counts(cg_context *ctx, double radius, int64_t *counts);
int cg_neighbor_fill(cg_context *ctx, double radius, const int64_t *indptr, int64_t *indices);

/* ---- x-slab decomposition (multi-GPU).  The reference has no
 * distributed layer: these entry points carry the same step across ranks,
 * one context per GPU.  Rank r owns the agents whose global box plane lies in
 * [X_r, X_r+1), X_k = floor(k dimx / world), and sees planes X_r - 1 and
 * X_r+1 as ghosts.  Device buffers (send/recv) are raw device pointers owned
 * by the caller (e.g. torch CUDA tensors handed to NCCL); records are
 * cg_record_bytes() each.  Per step, on every rank, ONE exchange round:
 *   cg_local_bbox -> all-reduce (MAX of the 11 values, minima negated) ->
 *   cg_slab_plan -> all-to-all of the 3-per-rank counts -> cg_slab_pack(send)
 *   -> exchange of the records -> cg_slab_unpack(recv) -> cg_slab_step.
 * pack, unpack and step are enqueued on the context's stream (cg_stream) and
 * do not wait for the host: the caller orders its exchange of send / recv on
 * that stream (or waits on it), as NCCL does when issued on cg_stream.
 * Owned agents' results are those of a single-GPU step over the global pool. */
int64_t cg_record_bytes(const cg_context *ctx);
/* Pre-size the agent buffers (before cg_upload) for arrivals and ghosts. */
int cg_reserve(cg_context *ctx, int64_t capacity);
/* Exact bbox of the owned agents (min xyz, max xyz), max diameter, the last
 * step's largest squared displacement, a neighbour-list veto (the build's
 * overflow count, or 1 when this rank neither built lists nor ran a list step
 * last), the negated min diameter and the largest uid: all eleven are
 * all-reduced with MAX (after negating the three minima), so every rank takes
 * the same list decision in cg_slab_plan and knows whether the global pool is
 * uniform and whether every uid is below 2^32. */
int cg_local_bbox(cg_context *ctx, double out[11]);
/* Geometry from the global bbox (spatial.py:99-116; GridOverflowError as
 * cg_step) and slab planes: planes = {X_rank, X_rank+1}.  counts (3 * world):
 * for destination rank q, counts[3q] = owned agents that migrate to q (0 for
 * q == rank), counts[3q+1] = owned agents in q's ghost band below its slab,
 * counts[3q+2] = owned agents in q's ghost band above it (band: 1 plane, 3
 * with neighbour lists).  With neighbour lists, a step whose lists are still
 * valid (decided identically on every rank from the all-reduced bbox[7..8])
 * keeps the partition: no migrants, and the ghost runs are the refresh of the
 * ghosts every rank holds since the last rebuild. */
int cg_slab_plan(cg_context *ctx, const double bbox[11], double interaction_radius, int64_t box_cap,
                 int world, int rank, int64_t *counts, int64_t planes[2]);
/* Outgoing records -> send, grouped by destination rank (ascending), each
 * destination's run = [migrants][lo ghosts][hi ghosts] with the cg_slab_plan
 * counts; then the migrants leave the owned set (compacted). */
int cg_slab_pack(cg_context *ctx, void *send);
/* recv = the runs received from every source rank (ascending), run sizes
 * recv_counts[3s .. 3s+2] as in cg_slab_plan: migrants join the owned set,
 * ghosts are this step's candidates (dropped after cg_slab_step). */
int cg_slab_unpack(cg_context *ctx, const void *recv, const int64_t *recv_counts);
/* The mechanical step on the owned agents over the slab's sub-grid. */
int cg_slab_step(cg_context *ctx, const double params[5], int flags, cg_step_stats *stats);
/* Optional, between cg_slab_pack and cg_slab_unpack of a neighbour-list step:
 * enqueue the list sweep of the owned agents whose lists hold no ghost (build
 * planes at least 3 from either slab face) so it runs while the ghost refresh
 * is in flight; the following cg_slab_step sweeps only the boundary agents.
 * A no-op on rebuild steps (same flags as the cg_slab_step that follows). */
int cg_slab_step_interior(cg_context *ctx, const double params[5], int flags);
/* After cg_slab_plan: -1 for a rebuild step, else the id of the list epoch
 * (constant between rebuilds): a refresh step whose run sizes -- sent and
 * received -- are those of the previous refresh step of the same epoch, so a
 * caller may skip the counts all-to-all. */
int64_t cg_slab_list_epoch(const cg_context *ctx);

#ifdef __cplusplus
}
#endif
#endif /* CELLGRID_B200_H */
