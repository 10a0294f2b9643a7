"""Generate golden fixtures from the reference implementation itself.

Runs ONLY in the build container, where the reference is mounted read-only at
/root/reference (cellgrid 0.1.0, numba kernels).  The outputs (tests/golden/
*.npz) are committed; nothing on the GPU box reads /root/reference.

For every fixture the script records the pre-step pool, then replays
reference engine.step (engine.py:279-341) with the reference's own functions:
  spatial.build_grid -> morton.compute_sort_permutation -> pool.apply_permutation
  -> spatial.build_grid -> per-agent kernels._gather_stencil/_sum_forces_sorted
  (to expose per-agent m / nk, which the public API only reports as totals)
and cross-checks the replay against the public engine.step on a copy
(counters, displacements, positions and storage order must be identical).

Usage (from the repo root):
  NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \
    python tests/golden/make_golden.py
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import cellgrid  # noqa: E402
from cellgrid import engine, kernels, morton, spatial  # noqa: E402
from cellgrid.geometry import Aabb  # noqa: E402
from cellgrid.mechanics import ForceParams  # noqa: E402
from cellgrid.pool import AgentPool, PrecisionMode  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def per_agent_counts(pool, grid, params_arr):
    """m (stencil candidates) and nk (colliding pairs) per storage index."""
    n = pool.count
    radii = pool.radii()
    dims = [int(d) for d in grid.dims]
    cap = max(1, grid.stencil_candidate_cap())
    cand = np.empty(cap, np.int64)
    keep = np.empty(cap, np.int64)
    tmp = np.empty(1, pool.dtype)
    m_out = np.empty(n, np.int32)
    nk_out = np.empty(n, np.int32)
    for i in range(n):
        m = kernels._gather_stencil(i, grid.box_index[i], dims[0], dims[1], dims[2],
                                    grid.box_head, grid.successors, cand)
        _, _, _, nk, _ = kernels._sum_forces_sorted(
            i, cand, m, keep, pool.position_x, pool.position_y, pool.position_z, radii,
            pool.uid, params_arr, tmp)
        m_out[i] = m
        nk_out[i] = nk
    return m_out, nk_out


def snapshot(pool):
    return dict(px=pool.position_x.copy(), py=pool.position_y.copy(),
                pz=pool.position_z.copy(), diam=pool.diameter.copy(),
                adh=pool.adherence.copy(), uid=pool.uid.copy())


def replay(pool, cfg, k):
    """One reference step with grid/per-agent outputs exposed; mutates pool."""
    par = cfg.strategy
    parallel = not isinstance(par, engine.Serial)
    sort_due = cfg.morton_sort_every > 0 and k % cfg.morton_sort_every == 0
    if sort_due and pool.count > 1:
        pre = spatial.build_grid(pool, cfg.interaction_radius, parallel=parallel)
        morton.reorder_pool(pool, morton.compute_sort_permutation(pool, pre))
    grid = spatial.build_grid(pool, cfg.interaction_radius, parallel=parallel)
    params_arr = cfg.force_params.as_array(pool.dtype)
    m, nk = per_agent_counts(pool, grid, params_arr)
    evals, cands, ndeg = engine._dispatch_force_phase(pool, grid, params_arr, cfg.strategy)
    out = dict(evals=int(evals), cands=int(cands), ndeg=int(ndeg), m=m, nk=nk,
               box_length=float(grid.box_length), origin=np.asarray(grid.origin, np.float64),
               dims=np.asarray(grid.dims, np.int64), box_index=grid.box_index.astype(np.int64),
               box_count=grid.box_count.astype(np.int32),
               occupied=grid.occupied_box_count, max_occ=grid.max_occupancy,
               sorted_uid=pool.uid.copy())
    if not cfg.freeze_displacement:
        pool.position_x += pool.displacement_x
        pool.position_y += pool.displacement_y
        pool.position_z += pool.displacement_z
    out.update(dx=pool.displacement_x.copy(), dy=pool.displacement_y.copy(),
               dz=pool.displacement_z.copy(), out_px=pool.position_x.copy(),
               out_py=pool.position_y.copy(), out_pz=pool.position_z.copy(),
               out_uid=pool.uid.copy())
    return out


def make(name, pool, cfg, steps=1, note=""):
    inp = snapshot(pool)
    check = pool.copy()
    rec = {}
    for k in range(steps):
        r = replay(pool, cfg, k)
        s = engine.step(check, cfg, k)
        assert (s.force_evals, s.candidates, s.degenerate_pairs) == (r["evals"], r["cands"], r["ndeg"]), name
        assert np.array_equal(check.uid, pool.uid), name
        for c in ("position_x", "position_y", "position_z", "displacement_x"):
            assert np.array_equal(getattr(check, c), getattr(pool, c)), (name, c)
        for key, val in r.items():
            rec["s%d_%s" % (k, key)] = np.asarray(val)
    fp = cfg.force_params
    np.savez_compressed(
        os.path.join(OUT, name + ".npz"), steps=steps, dtype=str(pool.dtype),
        sort_every=cfg.morton_sort_every, freeze=cfg.freeze_displacement,
        interaction_radius=(np.nan if cfg.interaction_radius is None
                            else float(cfg.interaction_radius)),
        params=np.asarray([fp.kappa, fp.gamma, fp.timestep, fp.max_displacement,
                           fp.adherence_scale], np.float64),
        state_hash=pool.state_hash(), note=note,
        **{"in_" + k: v for k, v in inp.items()}, **rec)
    print("%-28s n=%-6d steps=%d evals(s0)=%d cands(s0)=%d ndeg(s0)=%d" % (
        name, inp["uid"].shape[0], steps, rec["s0_evals"], rec["s0_cands"], rec["s0_ndeg"]))


def cfg(prec, sort=1, freeze=False, ir=None, fp=None):
    return engine.SimulationConfig(force_params=fp or ForceParams(), strategy=engine.Serial(),
                                   precision=prec, morton_sort_every=sort, steps=1,
                                   freeze_displacement=freeze, interaction_radius=ir)


def main():
    F64, F32 = PrecisionMode.FP64, PrecisionMode.FP32
    for prec, tag in ((F64, "f64"), (F32, "f32")):
        make("c1_" + tag, AgentPool.spawn_grid(32, 8.0, 10.0, 0.4, precision=prec), cfg(prec),
             note="C1: spawn_grid(32, 8.0, 10.0, 0.4), one step, Morton sort")
        for seed in range(3):
            make("rand600_s%d_%s" % (seed, tag),
                 AgentPool.spawn_random(600, Aabb.cube(60.0), 10.0, 0.4, seed, precision=prec),
                 cfg(prec), note="spawn_random(600, cube(60), 10, 0.4, seed)")
        make("dense3000_" + tag,
             AgentPool.spawn_random(3000, Aabb.cube(40.0), 10.0, 0.4, 4, precision=prec),
             cfg(prec), note="very dense: nk > 32 exercises the argsort branch")
        make("multistep_" + tag,
             AgentPool.spawn_random(2000, Aabb.cube(100.0), 10.0, 0.4, 3, precision=prec),
             cfg(prec, sort=2), steps=5, note="5 steps, Morton sort every 2nd step")
    # degenerate / touching fixture
    pos = np.array([[0, 0, 0], [0, 0, 0], [6, 0, 0], [20, 0, 0], [30, 0, 0]], np.float64)
    for prec, tag in ((F64, "f64"), (F32, "f32")):
        make("degenerate_" + tag, AgentPool.from_arrays(pos, 10.0, 0.4, prec), cfg(prec),
             note="coincident pair + touching pair (distance exactly 10)")
    # faces: spacing == box_length puts every agent exactly on a box face
    make("faces_f64", AgentPool.spawn_grid(4, 10.0, 10.0, 0.4), cfg(F64),
         note="spawn_grid(4, 10, 10): half-open face rule")
    # heterogeneous diameters / adherence, custom params, interaction radius
    rng = np.random.default_rng(11)
    n = 1500
    het = AgentPool.from_arrays(rng.uniform(0, 70, (n, 3)), rng.uniform(6.0, 12.0, n),
                                rng.uniform(0.0, 3.0, n))
    make("hetero_f64", het, cfg(F64, ir=14.0,
                                fp=ForceParams(kappa=3.0, gamma=0.5, timestep=0.05,
                                               max_displacement=1.5, adherence_scale=0.7)),
         steps=3, note="random diameters 6-12, adherence 0-3, interaction_radius 14")
    # frozen, unsorted (benchmark B conventions, bench.py:167-172, 250-255)
    side = cellgrid.box_side_for_density(20000, 5.0, 27.0)
    for sort in (1, 0):
        make("benchB20k_d27_sort%d" % sort,
             AgentPool.spawn_random(20000, Aabb.cube(side), 10.0, 0.4, 0),
             cfg(F64, sort=sort, freeze=True), steps=2,
             note="benchmark-B pool, 20k agents, ref-density 27, frozen")


if __name__ == "__main__":
    main()
