"""Neighbour-list reuse (csrc/list.cuh) changes nothing observable: the same
pool stepped with lists (auto skin, and a small explicit skin that forces
frequent rebuilds) and without (CG_OPT_LIST_SKIN = 0) gives bit-identical
counters, grid statistics, storage order, per-agent m / nk, displacements and
positions at every step -- and list steps really ran.  Anchored to the
reference through the C oracle on the first steps."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

PARAMS5 = np.array([2.0, 1.0, 0.01, 3.0, 1.0])


def _pools():
    from paper_2105_00039_b200.pool import AgentPool, PrecisionMode
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    yield "lattice", AgentPool.from_arrays(jittered_lattice_positions(24, 8.0, 1.0, 0), 10.0, 0.4)
    rng = np.random.default_rng(3)
    # sparse pools (about 1.5 agents per box: the path lists apply to)
    side = 10.0 * (30000 / 1.5) ** (1 / 3)
    yield "random", AgentPool.from_arrays(rng.uniform(0, side, (30000, 3)), 10.0, 0.4)
    yield "hetero", AgentPool.from_arrays(rng.uniform(0, 250.0, (20000, 3)), rng.uniform(4.0, 12.0, 20000),
                                          rng.uniform(0.0, 1.0, 20000))
    yield "lattice_f32", AgentPool.from_arrays(jittered_lattice_positions(20, 8.0, 1.0, 1), 10.0, 0.4,
                                               PrecisionMode.FP32)


POOLS = list(_pools())


def _run(pool, skin, steps, summation, sort_every=1, freeze_at=(), record=True):
    from paper_2105_00039_b200 import _native as N
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, summation)
    ctx.set_option(N.CG_OPT_LIST_SKIN, skin)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    out = []
    for k in range(steps):
        flags = N.CG_STEP_RECORD if record else 0
        if sort_every and k % sort_every == 0:
            flags |= N.CG_STEP_SORT
        if k in freeze_at:
            flags |= N.CG_STEP_FREEZE
        st = ctx.step(PARAMS5, None, 1 << 24, flags)
        cols = ctx.download()
        if record:
            m, nk = ctx.record_export()
            nb = int(np.prod(list(st.grid_dims)))
            bi, bc = ctx.grid_export(nb)
        else:
            m = nk = bi = bc = np.zeros(0)
        out.append(((st.force_evals, st.candidates, st.degenerate_pairs, st.grid_occupied_boxes,
                     st.grid_max_occupancy, tuple(st.grid_dims)), cols, m, nk, bi, bc))
    stats = ctx.list_stats()
    ctx.close()
    return out, stats


@pytest.mark.parametrize("summation", [0, 1])
@pytest.mark.parametrize("name,pool", POOLS, ids=[p[0] for p in POOLS])
def test_lists_change_nothing(cuda_required, name, pool, summation):
    steps = 10
    ref, s0 = _run(pool, 0, steps, summation)
    assert s0["list_steps"] == 0
    for skin in (-1, 300):
        got, s1 = _run(pool, skin, steps, summation, freeze_at=(4,))
        ref2, _ = _run(pool, 0, steps, summation, freeze_at=(4,))
        if name.startswith("lattice"):     # small motions: the lists serve steps
            assert s1["list_steps"] > 0, (name, skin, s1)
        else:                              # deep random overlaps: lists are built and expire
            assert s1["builds"] > 0, (name, skin, s1)
        for k, (a, b) in enumerate(zip(got, ref2)):
            assert a[0] == b[0], (name, skin, k)
            for col in a[1]:
                assert np.array_equal(a[1][col], b[1][col]), (name, skin, k, col)
            for q in range(2, 6):
                assert np.array_equal(a[q], b[q]), (name, skin, k, q)
    # unsorted steps (storage order kept) and the lists-off run agree too
    got, s2 = _run(pool, -1, 6, summation, sort_every=0)
    ref3, _ = _run(pool, 0, 6, summation, sort_every=0)
    for a, b in zip(got, ref3):
        assert a[0] == b[0]
        for col in a[1]:
            assert np.array_equal(a[1][col], b[1][col])


def test_lists_match_oracle(cuda_required):
    """lattice pool, 6 chained steps in uid order: lists-on device == C oracle."""
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    pool = POOLS[0][1]
    ref = pool.copy()
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 0)
    ctx.set_option(N.CG_OPT_LIST_SKIN, -1)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    for k in range(6):
        st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT)
        r = oracle.step(ref, ForceParams(), sort=True, threads=8)
        assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
            r.force_evals, r.candidates, r.degenerate_pairs)
        cols = ctx.download()
        assert np.array_equal(cols["uid"], ref.uid)
        for a, b in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"),
                     ("dx", "displacement_x"), ("dy", "displacement_y"), ("dz", "displacement_z")):
            assert np.array_equal(cols[a], getattr(ref, b)), (k, a)
    assert ctx.list_stats()["list_steps"] >= 3
    ctx.close()


def test_list_overflow_falls_back(cuda_required):
    """A sparse pool with one crowded spot (more than 48 partners within the
    skin for some agents): the build reports the overflow, the lists are not
    used, and every step still matches the list-free run bit for bit."""
    from paper_2105_00039_b200.pool import AgentPool
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    pos = jittered_lattice_positions(20, 8.0, 1.0, 4)
    rng = np.random.default_rng(9)
    pos[:80] = 80.0 + rng.uniform(-4.0, 4.0, (80, 3))     # 80 agents inside one box
    pool = AgentPool.from_arrays(pos, 10.0, 0.4)
    got, st = _run(pool, -1, 12, 0)
    ref, _ = _run(pool, 0, 12, 0)
    assert st["builds"] >= 1 and st["list_steps"] == 0, st
    for a, b in zip(got, ref):
        assert a[0] == b[0]
        for col in a[1]:
            assert np.array_equal(a[1][col], b[1][col])


@pytest.mark.parametrize("sort_every", [1, 0])
@pytest.mark.parametrize("name,pool", POOLS, ids=[p[0] for p in POOLS])
def test_step_download_equals_step_then_download(cuda_required, name, pool, sort_every):
    """cg_step_download (transfers overlapped with the sweep) returns exactly
    what cg_step followed by cg_download returns, step after step (uploads
    between steps, as engine.step does)."""
    from paper_2105_00039_b200 import _native as N
    a, b = N.Context(0, pool.dtype), N.Context(0, pool.dtype)
    try:
        cur_a = cur_b = {"px": pool.position_x, "py": pool.position_y, "pz": pool.position_z,
                         "diameter": pool.diameter, "adherence": pool.adherence, "uid": pool.uid}
        for k in range(3):
            flags = N.CG_STEP_SORT if sort_every and k % sort_every == 0 else 0
            a.upload(cur_a["px"], cur_a["py"], cur_a["pz"], cur_a["diameter"], cur_a["adherence"], cur_a["uid"])
            b.upload(cur_b["px"], cur_b["py"], cur_b["pz"], cur_b["diameter"], cur_b["adherence"], cur_b["uid"])
            sa, cur_a = a.step_download(PARAMS5, None, 1 << 24, flags)
            sb = b.step(PARAMS5, None, 1 << 24, flags)
            cur_b = b.download()
            assert (sa.force_evals, sa.candidates) == (sb.force_evals, sb.candidates)
            for col in cur_b:
                assert np.array_equal(cur_a[col], cur_b[col]), (name, k, col)
    finally:
        a.close()
        b.close()


def test_lists_long_run_matches_oracle(cuda_required):
    """60 chained uid-order steps of a 32,768-agent jittered lattice (several
    list epochs and rebuilds): lists on (three levels, two levels, the
    neighbour list alone), lists off and the C oracle agree bit for bit at the end
    (positions, displacements, storage order)."""
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    from paper_2105_00039_b200.pool import AgentPool
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    pool = AgentPool.from_arrays(jittered_lattice_positions(32, 8.0, 1.0, 11), 10.0, 0.4)
    params = ForceParams(timestep=0.02)
    p5 = np.array([params.kappa, params.gamma, params.timestep, params.max_displacement, params.adherence_scale])
    outs = []
    # defaults (three levels), the short sub-list only, no sub-lists, no lists
    for skin, inner, mid in ((-1, None, None), (-1, None, 0), (-1, 0, 0), (0, None, None)):
        ctx = N.Context(0, pool.dtype)
        ctx.set_option(N.CG_OPT_SUMMATION, 0)
        ctx.set_option(N.CG_OPT_LIST_SKIN, skin)
        if inner is not None:
            ctx.set_option(N.CG_OPT_INNER_LIST, inner)
        if mid is not None:
            ctx.set_option(N.CG_OPT_MID_LIST, mid)
        ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
        sts = [ctx.step(p5, None, 1 << 24, N.CG_STEP_SORT) for _ in range(60)]
        evals = [(s.force_evals, s.candidates, s.degenerate_pairs, s.grid_occupied_boxes, s.grid_max_occupancy)
                 for s in sts]
        outs.append((evals, ctx.download(), ctx.list_stats()))
        ctx.close()
    assert outs[0][2]["builds"] >= 3 and outs[0][2]["list_steps"] >= 30, outs[0][2]
    assert outs[0][2]["inner_steps"] > 0 and outs[1][2]["inner_steps"] > 0 and outs[2][2]["inner_steps"] == 0, \
        [o[2] for o in outs]
    ref = pool.copy()
    ref_evals = []
    for _ in range(60):
        r = oracle.step(ref, params, sort=True, threads=8)
        ref_evals.append((r.force_evals, r.candidates, r.degenerate_pairs, int(np.count_nonzero(r.box_count)),
                          int(r.box_count.max())))
    assert outs[0][0] == outs[1][0] == outs[2][0] == outs[3][0] == ref_evals
    for _, cols, _ in outs:
        assert np.array_equal(cols["uid"], ref.uid)
        for a, b in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"), ("dx", "displacement_x")):
            assert np.array_equal(cols[a], getattr(ref, b)), a


@pytest.mark.parametrize("name,pool", POOLS, ids=[p[0] for p in POOLS])
def test_fused_list_steps_change_nothing(cuda_required, name, pool):
    """Steps without CG_STEP_RECORD take the fused list path (box counting in
    the list sweep, candidates and statistics from the box-stencil pass):
    counters, grid statistics and every column equal the list-free run."""
    got, st = _run(pool, -1, 12, 0, freeze_at=(5,), record=False)
    ref, _ = _run(pool, 0, 12, 0, freeze_at=(5,), record=False)
    if name.startswith("lattice"):
        assert st["list_steps"] > 0, st
    for k, (a, b) in enumerate(zip(got, ref)):
        assert a[0] == b[0], (name, k)
        for col in a[1]:
            assert np.array_equal(a[1][col], b[1][col]), (name, k, col)


@pytest.mark.parametrize("spacing,ir", [(8.0, 11.0), (10.0, 12.5)])
def test_lists_with_interaction_radius(cuda_required, spacing, ir):
    """interaction_radius above the diameter: larger boxes (L = ir) and a skin
    of 0.07 L (still on the sparse path, where lists apply); list steps equal
    list-free steps and the oracle."""
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    from paper_2105_00039_b200.pool import AgentPool
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    pool = AgentPool.from_arrays(jittered_lattice_positions(24, spacing, 1.0, 21), 10.0, 0.4)
    outs = []
    for skin in (-1, 0):
        ctx = N.Context(0, pool.dtype)
        ctx.set_option(N.CG_OPT_SUMMATION, 0)
        ctx.set_option(N.CG_OPT_LIST_SKIN, skin)
        ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
        sts = [ctx.step(PARAMS5, ir, 1 << 24, N.CG_STEP_SORT) for _ in range(12)]
        outs.append(([(s.force_evals, s.candidates, s.grid_occupied_boxes) for s in sts], ctx.download(),
                     ctx.list_stats()))
        ctx.close()
    assert outs[0][2]["list_steps"] > 0
    ref = pool.copy()
    ref_c = []
    for _ in range(12):
        r = oracle.step(ref, ForceParams(), sort=True, interaction_radius=ir, threads=8)
        ref_c.append((r.force_evals, r.candidates, int(np.count_nonzero(r.box_count))))
    assert outs[0][0] == outs[1][0] == ref_c
    for cols in (outs[0][1], outs[1][1]):
        assert np.array_equal(cols["uid"], ref.uid)
        assert np.array_equal(cols["px"], ref.position_x) and np.array_equal(cols["dz"], ref.displacement_z)


def _dense_pool(n, density, seed):
    from paper_2105_00039_b200.geometry import Aabb
    from paper_2105_00039_b200.pool import AgentPool
    from paper_2105_00039_b200.workloads import box_side_for_density
    return AgentPool.spawn_random(n, Aabb.cube(box_side_for_density(n, 10.0, density)), 10.0, 0.4, seed)


@pytest.mark.parametrize("density", [27.0, 100.0])
def test_dense_lists_match_oracle(cuda_required, density):
    """Dense pools (the z-sorted-box path): lists sized from the density are
    built by the grid sweep and serve frozen steps (benchmark B) and then
    moving steps; every step equals the C oracle bit for bit in uid order."""
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    pool = _dense_pool(12000, density, 5)
    ref = pool.copy()
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 0)
    ctx.set_option(N.CG_OPT_LIST_SKIN, -1)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    kinds = []
    for k in range(10):
        freeze = k < 6
        st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT | (N.CG_STEP_FREEZE if freeze else 0))
        kinds.append(int(st.sweep_kind))
        r = oracle.step(ref, ForceParams(), sort=True, freeze=freeze, threads=8)
        assert (st.force_evals, st.candidates, st.degenerate_pairs, st.grid_max_occupancy) == (
            r.force_evals, r.candidates, r.degenerate_pairs, int(r.box_count.max())), k
        cols = ctx.download()
        assert np.array_equal(cols["uid"], ref.uid)
        for a, b in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"),
                     ("dx", "displacement_x"), ("dy", "displacement_y"), ("dz", "displacement_z")):
            assert np.array_equal(cols[a], getattr(ref, b)), (k, a)
    assert kinds[:6] == [0, 1, 2, 2, 2, 2], kinds
    ctx.close()


@pytest.mark.parametrize("summation", [0, 1])
def test_dense_lists_change_nothing_uid(cuda_required, summation):
    """Dense moving pool, 12 steps: in uid summation the lists change nothing;
    in stencil summation list steps sum in uid order (the reference's), so the
    comparison is against uid-order results within 1e-9 relative."""
    pool = _dense_pool(15000, 40.0, 8)
    got, s1 = _run(pool, -1, 12, summation, freeze_at=(0, 1, 2, 3))
    ref, _ = _run(pool, 0, 12, 0, freeze_at=(0, 1, 2, 3))
    assert s1["builds"] > 0
    for k, (a, b) in enumerate(zip(got, ref)):
        assert a[0] == b[0], k
        for col in a[1]:
            if summation == 0 or col in ("uid", "diameter", "adherence"):
                assert np.array_equal(a[1][col], b[1][col]), (k, col)
            else:
                np.testing.assert_allclose(a[1][col], b[1][col], rtol=1e-9, atol=1e-12)
        for q in range(2, 6):
            assert np.array_equal(a[q], b[q]), (k, q)


@pytest.mark.parametrize("n,density,skin", [(8000, 350.0, 0), (8000, 350.0, -1), (3000, 1100.0, 0)])
def test_very_dense_pools_match_oracle(cuda_required, n, density, skin):
    """More survivors than the warp's shared-memory queue (256): the second
    warp pass with global queues (<= 1024) and, beyond that, the thread rounds;
    with lists on, wide lists.  Bit-identical to the oracle in uid order."""
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    pool = _dense_pool(n, density, 11)
    ref = pool.copy()
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 0)
    ctx.set_option(N.CG_OPT_LIST_SKIN, skin)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    kinds = []
    for k in range(4):
        freeze = k < 3
        st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT | (N.CG_STEP_FREEZE if freeze else 0))
        kinds.append(int(st.sweep_kind))
        r = oracle.step(ref, ForceParams(), sort=True, freeze=freeze, threads=8)
        assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
            r.force_evals, r.candidates, r.degenerate_pairs), k
        cols = ctx.download()
        assert np.array_equal(cols["uid"], ref.uid)
        for a, b in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"),
                     ("dx", "displacement_x"), ("dy", "displacement_y"), ("dz", "displacement_z")):
            assert np.array_equal(cols[a], getattr(ref, b)), (k, a)
    if skin:
        assert kinds[:3] == [0, 1, 2], kinds
    ctx.close()


@pytest.mark.parametrize("fp32", [False, True], ids=["fp64", "fp32"])
def test_coincident_centres_on_list_steps(cuda_required, fp32):
    """Frozen pool with 200 exactly coincident pairs: every list step meets
    dist == 0, which leaves the call-free arithmetic (fp64: the agent is
    deferred to list_slow_kernel; fp32: the inline slow path) -- counters,
    degenerate pairs and every column equal the list-free run."""
    from paper_2105_00039_b200.pool import AgentPool, PrecisionMode
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    pos = jittered_lattice_positions(20, 8.0, 1.0, 4)
    pool = AgentPool.from_arrays(np.vstack([pos, pos[::40]]), 10.0, 0.4,
                                 PrecisionMode.FP32 if fp32 else PrecisionMode.FP64)
    frozen = tuple(range(8))
    got, st = _run(pool, -1, 8, 0, freeze_at=frozen, record=False)
    ref, _ = _run(pool, 0, 8, 0, freeze_at=frozen, record=False)
    assert st["list_steps"] > 0, st
    assert got[-1][0][2] > 0   # degenerate pairs on the list steps
    for k, (a, b) in enumerate(zip(got, ref)):
        assert a[0] == b[0], k
        for col in a[1]:
            assert np.array_equal(a[1][col], b[1][col]), (k, col)


def test_build_writes_the_sub_lists(cuda_required):
    """A sparse list build also writes the middle and short sub-lists
    (host_step.cuh run_sweep, sweep7.cuh LIST): every list step after the
    build sweeps a sub-list -- none refreshes from the whole list while the
    motion stays inside the short list's delta -- and the steps equal the C
    oracle bit for bit."""
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    pool = POOLS[0][1]
    ref = pool.copy()
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 0)
    ctx.set_option(N.CG_OPT_LIST_SKIN, -1)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    kinds = []
    for k in range(4):
        st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT)
        kinds.append(int(st.sweep_kind))
        r = oracle.step(ref, ForceParams(), sort=True, threads=8)
        assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
            r.force_evals, r.candidates, r.degenerate_pairs), k
        cols = ctx.download()
        for a, b in (("px", "position_x"), ("dx", "displacement_x"), ("dz", "displacement_z")):
            assert np.array_equal(cols[a], getattr(ref, b)), (k, a)
    stats = ctx.list_stats()
    ctx.close()
    assert kinds[:2] == [0, 1] and kinds[2] == 2, kinds
    # the first list step right after the build already swept a sub-list
    n_list = kinds.count(2)
    assert stats["list_steps"] == n_list and stats["inner_steps"] == n_list, (kinds, stats)
