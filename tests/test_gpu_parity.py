"""GPU parity: the CUDA path (through the C ABI) against the reference's golden
vectors and the C oracle.

Bars (north star): box assignment, box counts/offsets, per-agent candidate and
colliding-pair counts and the step counters bit-exact; displacements
bit-exact in uid summation mode (the reference's order) and within 1e-12
relative in stencil mode (tolerance written below, well inside the 1e-9 the
north star allows).  The only non-correctly-rounded operation on the path is
cos/sin of the degenerate-pair direction (kernels.py:99-100), so fixtures with
coincident centres compare displacements to 1e-12 relative instead.
"""

import numpy as np
import pytest

import oracle
from conftest import golden_names, ir_from_golden, load_golden, params_from_golden, pool_from_golden

pytestmark = pytest.mark.gpu

STENCIL_RTOL = 1e-12   # fp64, per-agent vector relative error
FP32_RTOL = 1e-4       # fp32 stencil order vs the reference's fp32 uid order


def _native():
    from paper_2105_00039_b200 import _native
    return _native


def _ctx(dtype, summation="uid", sweep="v7", relayout_every=1, path="auto"):
    N = _native()
    ctx = N.Context(0, dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, {"uid": 0, "stencil": 1}[summation])
    ctx.set_option(N.CG_OPT_SWEEP, {"agent": 0, "v7": 1}[sweep])
    ctx.set_option(N.CG_OPT_RELAYOUT_EVERY, relayout_every)
    ctx.set_option(N.CG_OPT_PATH, {"auto": 0, "sparse": 1, "dense": 2}[path])
    return ctx


def _params5(g):
    return np.asarray(g["params"], np.float64)


def _by_uid(uid, *cols):
    o = np.argsort(uid)
    return [c[o] for c in cols]


def _vec_close(mine, ref, rtol):
    """Per-agent relative error of a 3-vector: |a_i - b_i| <= rtol * |b_i| (norms).
    Components of a displacement can cancel to ~0, so the error is measured
    against the agent's vector magnitude, not per component."""
    a = np.stack([np.asarray(c, np.float64) for c in mine], 1)
    b = np.stack([np.asarray(c, np.float64) for c in ref], 1)
    err = np.linalg.norm(a - b, axis=1)
    scale = np.linalg.norm(b, axis=1)
    return bool(np.all(err <= rtol * scale)), float(np.max(err / np.maximum(scale, 1e-300)))


def _reference_state(g, k):
    """Pool columns before step k in the reference's storage order."""
    if k == 0:
        return [g[c] for c in ("in_px", "in_py", "in_pz", "in_diam", "in_adh", "in_uid")]
    s = "s%d_" % (k - 1)
    uid = g[s + "out_uid"]
    pos = np.searchsorted(g["in_uid"][np.argsort(g["in_uid"])], uid)
    order = np.argsort(g["in_uid"])[pos]
    return [g[s + "out_px"], g[s + "out_py"], g[s + "out_pz"], g["in_diam"][order],
            g["in_adh"][order], uid]


@pytest.mark.parametrize("sweep,relayout,path", [
    ("v7", 1, "auto"), ("v7", 1, "sparse"), ("v7", 1, "dense"), ("v7", 2, "sparse"),
    ("v7", 3, "dense"), ("v7", 1000, "sparse"), ("agent", 1, "auto")])
@pytest.mark.parametrize("summation", ["uid", "stencil"])
@pytest.mark.parametrize("name", golden_names())
def test_golden(cuda_required, name, summation, sweep, relayout, path):
    """uid mode chains all steps on the device (bit-exact end to end); stencil
    mode restarts every step from the reference's state, because its last-ulp
    differences legitimately move later bounding boxes.  relayout = the device
    moves records into slot order on every k-th sort step; downloads must show
    the reference's storage order regardless."""
    g = load_golden(name)
    dt = g["in_px"].dtype
    N = _native()
    ctx = _ctx(dt, summation, sweep=sweep, relayout_every=relayout, path=path)
    # the sparse path always sums in uid order (bit-exact)
    exact = summation == "uid" or (sweep == "v7" and path == "sparse")
    every = int(g["sort_every"])
    for k in range(int(g["steps"])):
        s = "s%d_" % k
        if k == 0 or not exact:
            ctx.upload(*_reference_state(g, k))
        degenerate = int(g[s + "ndeg"]) > 0
        flags = N.CG_STEP_RECORD
        if every > 0 and k % every == 0:
            flags |= N.CG_STEP_SORT
        if bool(g["freeze"]):
            flags |= N.CG_STEP_FREEZE
        st = ctx.step(_params5(g), ir_from_golden(g), 1 << 24, flags)
        assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
            int(g[s + "evals"]), int(g[s + "cands"]), int(g[s + "ndeg"]))
        assert st.box_length == float(g[s + "box_length"])
        assert list(st.origin) == list(g[s + "origin"])
        assert list(st.grid_dims) == list(g[s + "dims"])
        assert st.grid_max_occupancy == int(g[s + "max_occ"])
        assert st.grid_occupied_boxes == int(g[s + "occupied"])
        cols = ctx.download()
        # storage order: the reference's (Morton code, uid) order
        assert np.array_equal(cols["uid"], g[s + "out_uid"])
        nb = int(np.prod(g[s + "dims"]))
        box_index, box_count = ctx.grid_export(nb)
        assert np.array_equal(box_index, g[s + "box_index"])
        assert np.array_equal(box_count, g[s + "box_count"])
        m, nk = ctx.record_export()
        assert np.array_equal(m, g[s + "m"])
        assert np.array_equal(nk, g[s + "nk"])
        pairs = (("dx", "dx"), ("dy", "dy"), ("dz", "dz"),
                 ("px", "out_px"), ("py", "out_py"), ("pz", "out_pz"))
        if exact and not degenerate:
            for mine, ref in pairs:
                assert np.array_equal(cols[mine], g[s + ref]), (k, mine)
        else:
            rtol = STENCIL_RTOL if dt == np.float64 else FP32_RTOL
            for grp in (pairs[:3], pairs[3:]):
                ok, worst = _vec_close([cols[a] for a, _ in grp], [g[s + b] for _, b in grp], rtol)
                assert ok, (k, grp[0][0], worst)
    ctx.close()


def test_public_step_and_run_match_golden(cuda_required):
    """engine.step / engine.run (the drop-in API) on the multistep fixture."""
    import paper_2105_00039_b200 as P
    g = load_golden("multistep_f64")
    cfg = P.SimulationConfig(force_params=params_from_golden(g), strategy=P.Gpu(),
                             morton_sort_every=int(g["sort_every"]), steps=int(g["steps"]))
    pool = pool_from_golden(g)
    for k in range(int(g["steps"])):
        st = P.step(pool, cfg, k)
        assert st.force_evals == int(g["s%d_evals" % k])
    assert pool.state_hash() == str(g["state_hash"])
    pool2 = pool_from_golden(g)
    rep = P.run(pool2, cfg)
    assert rep.final_state_hash == str(g["state_hash"])
    assert [s.force_evals for s in rep.steps] == [int(g["s%d_evals" % k]) for k in range(5)]
    assert np.array_equal(pool2.uid, g["s4_out_uid"])


@pytest.mark.parametrize("which", ["serial", "parallel", "voxel"])
def test_reference_strategies_run_on_the_device(cuda_required, which):
    """A reference configuration with a CPU strategy (Serial / AgentParallel /
    VoxelTiled, which the reference guarantees bit-identical, engine.py:5)
    runs unchanged on the B200 path and reproduces the reference's pool."""
    import paper_2105_00039_b200 as P
    strat = {"serial": P.Serial(), "parallel": P.AgentParallel(8), "voxel": P.VoxelTiled(8)}[which]
    g = load_golden("multistep_f64")
    cfg = P.SimulationConfig(force_params=params_from_golden(g), strategy=strat,
                             morton_sort_every=int(g["sort_every"]), steps=int(g["steps"]))
    pool = pool_from_golden(g)
    rep = P.run(pool, cfg)
    assert rep.final_state_hash == str(g["state_hash"])
    assert rep.strategy == P.strategy_label(strat)
    pool = pool_from_golden(g)
    for k in range(int(g["steps"])):
        assert P.step(pool, cfg, k).force_evals == int(g["s%d_evals" % k])
    assert pool.state_hash() == str(g["state_hash"])


def test_build_grid_matches_oracle(cuda_required):
    import paper_2105_00039_b200 as P
    g = load_golden("rand600_s1_f64")
    pool = pool_from_golden(g)
    grid = P.build_grid(pool)
    L, origin, dims, nb = oracle.geometry(pool)
    bidx = oracle.box_ids(pool, L, origin, dims)
    count, start, _ = oracle.csr(bidx, nb)
    assert grid.box_length == L and np.array_equal(grid.origin, origin)
    assert np.array_equal(grid.dims, dims)
    assert np.array_equal(grid.box_index, bidx)
    assert np.array_equal(grid.box_count, count)
    assert np.array_equal(grid.box_offsets, start)
    # linked-cell view equals reference link_chains (kernels.py:132-145)
    head = np.full(nb, -1, np.int64)
    succ = np.full(pool.count, -1, np.int64)
    for i, b in enumerate(bidx):
        succ[i] = head[b]
        head[b] = i
    assert np.array_equal(grid.box_head, head)
    assert np.array_equal(grid.successors, succ)


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_c2_against_oracle(cuda_required, prec):
    """C2 (1M random, ref-density 27) vs the C oracle: counters, box ids, per-agent
    m/nk exact; displacements bit-exact (uid order)."""
    from paper_2105_00039_b200 import workloads
    from paper_2105_00039_b200.mechanics import ForceParams
    from paper_2105_00039_b200.pool import PrecisionMode
    N = _native()
    pm = PrecisionMode.FP64 if prec == "fp64" else PrecisionMode.FP32
    pool = workloads.c2(pm)
    ctx = _ctx(pool.dtype)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter,
               pool.adherence, pool.uid)
    st = ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24,
                  N.CG_STEP_SORT | N.CG_STEP_RECORD)
    r = oracle.step(pool, ForceParams(), sort=True, threads=16)
    assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
        r.force_evals, r.candidates, r.degenerate_pairs)
    cols = ctx.download()
    assert np.array_equal(cols["uid"], pool.uid)
    m, nk = ctx.record_export()
    assert np.array_equal(m, r.m) and np.array_equal(nk, r.nk)
    for mine, ref in (("dx", "displacement_x"), ("dy", "displacement_y"), ("dz", "displacement_z"),
                      ("px", "position_x"), ("py", "position_y"), ("pz", "position_z")):
        assert np.array_equal(cols[mine], getattr(pool, ref)), mine
    ctx.close()


def test_kernel_level_dropins(cuda_required):
    """cg_box_ids / cg_force_phase == kernels.box_ids_parallel / force_phase_parallel."""
    import ctypes
    N = _native()
    g = load_golden("dense3000_f64")
    pool = pool_from_golden(g)
    L, origin, dims, nb = oracle.geometry(pool)
    ref_ids = oracle.box_ids(pool, L, origin, dims)
    ctx = N.Context(0, np.float64)
    out = np.empty(pool.count, np.int64)
    N.check(N.load().cg_box_ids(ctx.h, pool.count, N.ptr(pool.position_x), N.ptr(pool.position_y),
                                N.ptr(pool.position_z), origin[0], origin[1], origin[2], L,
                                int(dims[0]), int(dims[1]), int(dims[2]), N.ptr(out)), ctx.h)
    assert np.array_equal(out, ref_ids)
    count, start, members = oracle.csr(ref_ids, nb)
    params7 = np.array([2.0, 1.0, 0.01, 3.0, 1.0, 0.0, 1.0])
    (rdx, rdy, rdz), _, _, rc = oracle.force_phase(pool, ref_ids, dims, start, members, params7, 8)
    radii = pool.radii()
    dx, dy, dz = (np.empty(pool.count) for _ in range(3))
    counters = np.zeros(3, np.int64)
    N.check(N.load().cg_force_phase(
        ctx.h, pool.count, N.ptr(pool.position_x), N.ptr(pool.position_y), N.ptr(pool.position_z),
        N.ptr(radii), N.ptr(pool.adherence), N.ptr(pool.uid), N.ptr(ref_ids),
        int(dims[0]), int(dims[1]), int(dims[2]), N.ptr(params7), N.ptr(dx), N.ptr(dy), N.ptr(dz),
        N.ptr(counters)), ctx.h)
    assert list(counters) == list(rc)
    assert np.array_equal(dx, rdx) and np.array_equal(dy, rdy) and np.array_equal(dz, rdz)
    ctx.close()


def test_errors_map_to_reference_exceptions(cuda_required):
    import paper_2105_00039_b200 as P
    N = _native()
    pool = P.AgentPool.spawn_random(100, P.Aabb.cube(1000.0), 10.0, 0.4, 0)
    ctx = _ctx(np.float64)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter,
               pool.adherence, pool.uid)
    with pytest.raises(P.GridOverflowError):
        ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1000, N.CG_STEP_SORT)
    with pytest.raises(ValueError):
        ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), -1.0, 1 << 24, 0)
    # the failed calls left the resident pool untouched
    cols = ctx.download()
    assert np.array_equal(cols["px"], pool.position_x) and np.array_equal(cols["uid"], pool.uid)
    with pytest.raises(ValueError):
        P.step(pool, P.SimulationConfig(precision=P.PrecisionMode.FP32))
    with pytest.raises(P.GridOverflowError):
        P.build_grid(pool, box_cap=10)
    empty = P.AgentPool.empty()
    assert P.step(empty, P.SimulationConfig()).agent_count == 0
    with pytest.raises(ValueError):
        P.build_grid(empty)
    ctx.close()


def test_determinism_and_sort_invariance(cuda_required):
    """Repeat runs hash identically; sorted vs unsorted frozen runs give the same
    uid -> position map bit for bit."""
    import paper_2105_00039_b200 as P
    g = load_golden("benchB20k_d27_sort1")
    hashes = set()
    for sort in (1, 0, 1):
        pool = pool_from_golden(g)
        rep = P.run(pool, P.SimulationConfig(strategy=P.Gpu(), morton_sort_every=sort, steps=3,
                                             freeze_displacement=False))
        hashes.add(rep.final_state_hash)
    assert len(hashes) == 1
