"""The BASELINE configurations at full size against the C oracle (which is
pinned bit-exactly to the reference, tests/test_oracle.py), on the production
path -- fused list sweeps, no CG_STEP_RECORD, the bench's options -- plus
size-independent properties:

* C4 (16,777,216 agents, fp64): 10 chained steps (a grid sweep, a list build,
  list sweeps) equal the oracle's counters at every step and its storage
  order, positions and displacements after steps 1, 5 and 10; step 0
  reproduces the reference's own counters recorded in SURVEY.md 8d
  (109,695,208 evaluations, 890,262,272 candidates, 207^3 boxes);
* C4 fp32: 5 chained steps (grid sweep, list build, whole-list and sub-list
  sweeps) equal the oracle's fp32 step;
* C3 (2M, density 4, 27 and 100, frozen as in benchmark B), with and without the
  Z-order sort, 2 steps: counters, storage order, displacements;
* C2 (1M random, fp64 and fp32), 3 chained steps: the reference's step-0
  counters and the oracle's pool after every step;
* the candidates counter equals sum_b count_b * (S_b - 1) over the exported
  grid; two runs are identical; lists on / off and 300-step runs agree.
The oracle runs on every host core (OpenMP), a few seconds per C4 step."""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PARAMS5 = np.array([2.0, 1.0, 0.01, 3.0, 1.0])


@pytest.fixture(scope="module")
def c4():
    from paper_2105_00039_b200 import workloads
    return workloads.c4()


@pytest.fixture(scope="module")
def c4f():
    from paper_2105_00039_b200 import workloads
    from paper_2105_00039_b200.pool import PrecisionMode
    return workloads.c4(PrecisionMode.FP32)


def _ctx(pool, skin=-1):
    from paper_2105_00039_b200 import _native as N
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 0)
    ctx.set_option(N.CG_OPT_LIST_SKIN, skin)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    return ctx


def _stencil_sum(counts):
    s = counts.astype(np.int64)
    for ax in range(3):
        p = np.pad(s, [(1, 1) if a == ax else (0, 0) for a in range(3)])
        sl = [slice(None)] * 3
        out = 0
        for d in range(3):
            sl[ax] = slice(d, d + s.shape[ax])
            out = out + p[tuple(sl)]
        s = out
    return s


def test_c4_counters_are_consistent(cuda_required, c4):
    from paper_2105_00039_b200 import _native as N
    ctx = _ctx(c4)
    try:
        st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT)
        dims = [int(d) for d in st.grid_dims]
        _, bc = ctx.grid_export(int(np.prod(dims)))
    finally:
        ctx.close()
    counts = bc.reshape(dims)
    assert counts.sum() == c4.count
    assert st.candidates == int((counts * (_stencil_sum(counts) - 1)).sum())
    assert st.force_evals % 2 == 0 and st.force_evals > 0
    assert st.grid_max_occupancy == counts.max() and st.grid_occupied_boxes == np.count_nonzero(counts)


def test_c4_lists_deterministic_and_sort_invariant(cuda_required, c4):
    from paper_2105_00039_b200 import _native as N
    runs = []
    for skin in (-1, -1, 0):
        ctx = _ctx(c4, skin)
        try:
            evals = [ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT).force_evals for _ in range(9)]
            stats = ctx.list_stats()
            runs.append((evals, ctx.download(), stats))
        finally:
            ctx.close()
    assert runs[0][2]["list_steps"] > 0 and runs[2][2]["list_steps"] == 0
    for other in runs[1:]:
        assert other[0] == runs[0][0]
        for col in runs[0][1]:
            assert np.array_equal(other[1][col], runs[0][1][col]), col
    # frozen: sorted vs unsorted step, same uid -> position map
    out = []
    for flags in (N.CG_STEP_SORT | N.CG_STEP_FREEZE, N.CG_STEP_FREEZE):
        ctx = _ctx(c4)
        try:
            ctx.step(PARAMS5, None, 1 << 24, flags)
            cols = ctx.download()
        finally:
            ctx.close()
        o = np.argsort(cols["uid"])
        out.append({k: v[o] for k, v in cols.items()})
    for col in out[0]:
        assert np.array_equal(out[0][col], out[1][col]), col


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_c4_long_run_lists_change_nothing(cuda_required, c4, c4f, prec):
    """300 resident C4 steps (dozens of list epochs): every step's counters and
    the final pool are identical with and without neighbour lists."""
    from paper_2105_00039_b200 import _native as N
    pool = c4 if prec == "fp64" else c4f
    runs = []
    for skin in (-1, 0):
        ctx = _ctx(pool, skin)
        try:
            ids = [ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT, wait=False) for _ in range(300)]
            ctx.synchronize()
            counters = [(s.force_evals, s.candidates, s.degenerate_pairs, s.grid_occupied_boxes,
                         s.grid_max_occupancy) for s in (ctx.fetch_stats(i) for i in ids[-60:])]
            runs.append((counters, ctx.download(), ctx.list_stats()))
        finally:
            ctx.close()
    assert runs[0][2]["builds"] >= 5 and runs[0][2]["list_steps"] >= 200, runs[0][2]
    assert runs[0][0] == runs[1][0]
    for col in runs[0][1]:
        assert np.array_equal(runs[0][1][col], runs[1][1][col]), col


ORACLE_THREADS = os.cpu_count() or 8
COLS = (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"),
        ("dx", "displacement_x"), ("dy", "displacement_y"), ("dz", "displacement_z"))


def _bench_ctx(pool):
    """A context with bench.py's default options (uid summation, relayout
    every sort step, auto skin)."""
    from paper_2105_00039_b200 import _native as N
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 0)
    ctx.set_option(N.CG_OPT_RELAYOUT_EVERY, 1)
    ctx.set_option(N.CG_OPT_LIST_SKIN, -1)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    return ctx


def _same_pool(cols, ref, tag):
    assert np.array_equal(cols["uid"], ref.uid), (tag, "storage order")
    for a, b in COLS:
        assert np.array_equal(cols[a], getattr(ref, b)), (tag, a)


def test_c4_chained_steps_match_oracle(cuda_required, c4):
    import oracle
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    ref = c4.copy()
    ctx = _bench_ctx(c4)
    kinds = []
    try:
        for k in range(10):
            st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT)
            kinds.append(int(st.sweep_kind))
            r = oracle.step(ref, ForceParams(), sort=True, threads=ORACLE_THREADS)
            got = (st.force_evals, st.candidates, st.degenerate_pairs, st.grid_occupied_boxes,
                   st.grid_max_occupancy, tuple(int(d) for d in st.grid_dims))
            want = (r.force_evals, r.candidates, r.degenerate_pairs, int(np.count_nonzero(r.box_count)),
                    int(r.box_count.max()), tuple(int(d) for d in r.dims))
            assert got == want, (k, got, want)
            if k == 0:   # the reference's own counters (measured with cellgrid)
                assert (st.force_evals, st.candidates) == (109_695_208, 890_262_272)
                assert tuple(int(d) for d in st.grid_dims) == (207, 207, 207)
            if k == 1:
                assert st.force_evals == 109_257_834
            if k in (0, 4, 9):
                _same_pool(ctx.download(), ref, ("c4", k))
    finally:
        ctx.close()
    assert kinds[:3] == [0, 1, 2] and kinds.count(2) >= 5, kinds


def test_c4_fp32_chained_steps_match_oracle(cuda_required, c4f):
    """The fp32 variant at full size: a grid sweep, a list build and list steps
    (sub-list written, then swept) equal the oracle's fp32 step bit for bit."""
    import oracle
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.mechanics import ForceParams
    ref = c4f.copy()
    ctx = _bench_ctx(c4f)
    kinds = []
    try:
        for k in range(5):
            st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT)
            kinds.append(int(st.sweep_kind))
            r = oracle.step(ref, ForceParams(), sort=True, threads=ORACLE_THREADS)
            assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
                r.force_evals, r.candidates, r.degenerate_pairs), k
            if k in (1, 4):
                _same_pool(ctx.download(), ref, ("c4f", k))
    finally:
        ctx.close()
    assert kinds == [0, 1, 2, 2, 2], kinds


@pytest.mark.parametrize("sort", [True, False], ids=["sorted", "unsorted"])
@pytest.mark.parametrize("density", [4.0, 27.0, 100.0])
def test_c3_full_size_matches_oracle(cuda_required, density, sort):
    import oracle
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200 import workloads
    from paper_2105_00039_b200.mechanics import ForceParams
    pool = workloads.c3(density)
    ref = pool.copy()
    ctx = _bench_ctx(pool)
    try:
        for k in range(2):
            flags = N.CG_STEP_FREEZE | (N.CG_STEP_SORT if sort else 0)
            st = ctx.step(PARAMS5, None, 1 << 24, flags)
            r = oracle.step(ref, ForceParams(), sort=sort, freeze=True, threads=ORACLE_THREADS)
            assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
                r.force_evals, r.candidates, r.degenerate_pairs), (density, sort, k)
            _same_pool(ctx.download(), ref, ("c3", density, sort, k))
    finally:
        ctx.close()


C2_STEP0 = {"fp64": (26_429_658, 166_986_922), "fp32": (26_429_648, 166_986_902)}


@pytest.mark.parametrize("prec", ["fp64", "fp32"])
def test_c2_chained_steps_match_oracle(cuda_required, prec):
    import oracle
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200 import workloads
    from paper_2105_00039_b200.mechanics import ForceParams
    from paper_2105_00039_b200.pool import PrecisionMode
    pool = workloads.c2(PrecisionMode.FP64 if prec == "fp64" else PrecisionMode.FP32)
    ref = pool.copy()
    ctx = _bench_ctx(pool)
    try:
        for k in range(3):
            st = ctx.step(PARAMS5, None, 1 << 24, N.CG_STEP_SORT)
            r = oracle.step(ref, ForceParams(), sort=True, threads=ORACLE_THREADS)
            assert (st.force_evals, st.candidates, st.degenerate_pairs) == (
                r.force_evals, r.candidates, r.degenerate_pairs), (prec, k)
            if k == 0:
                assert (st.force_evals, st.candidates) == C2_STEP0[prec]
                assert tuple(int(d) for d in st.grid_dims) == (56, 56, 56)
            _same_pool(ctx.download(), ref, ("c2", prec, k))
    finally:
        ctx.close()
