"""C4 at full size (16,777,216 agents, fp64) -- the bench workload -- through
size-independent properties (the oracle is too slow at this size; C2 at 1 M is
checked against it directly in test_gpu_parity.py):

* the candidates counter equals sum_b count_b * (S_b - 1), S_b the population
  of box b's clamped 27-box stencil, from the exported grid (numpy);
* ordered colliding pairs come in pairs (the force predicate is symmetric);
* two runs give the same state hash (determinism);
* neighbour-list steps change nothing: a run with lists equals a run without,
  column for column, after several steps (list steps included);
* the Z-order sort changes only the storage order: uid -> position maps of a
  sorted and an unsorted frozen step are identical."""

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
    assert runs[0][2]["builds"] >= 10 and runs[0][2]["list_steps"] >= 200, runs[0][2]
    assert runs[0][0] == runs[1][0]
    for col in runs[0][1]:
        assert np.array_equal(runs[0][1][col], runs[1][1][col]), col
