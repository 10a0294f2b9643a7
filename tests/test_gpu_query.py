"""Radius queries on the device grid against the
reference's own tables (tests/golden/nbr_*.npz) and the brute-force oracle.
Bar: bit-exact -- counts, CSR offsets and every row's uid-ascending neighbour
list, in the reference's storage order."""

import glob
import os

import numpy as np
import pytest

from oracle import oracle

pytestmark = pytest.mark.gpu

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "nbr_*.npz")))


def _pool(g):
    from paper_2105_00039_b200.pool import AgentPool
    return AgentPool(position_x=g["px"].copy(), position_y=g["py"].copy(), position_z=g["pz"].copy(),
                     diameter=g["diam"].copy(), adherence=g["adh"].copy(), uid=g["uid"].copy())


def _ir(g):
    ir = float(g["interaction_radius"])
    return None if np.isnan(ir) else ir


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p)[4:-4] for p in GOLDEN])
def test_neighbor_tables_match_reference(cuda_required, path):
    from paper_2105_00039_b200 import spatial
    g = np.load(path)
    pool = _pool(g)
    grid = spatial.build_grid(pool, interaction_radius=_ir(g))
    assert grid.box_length == float(g["box_length"])
    r = float(g["radius"])
    assert np.array_equal(spatial.neighbor_counts(grid, pool, r), g["counts"])
    indptr, indices = spatial.neighbor_csr(grid, pool, r)
    assert np.array_equal(indptr, g["indptr"])
    assert np.array_equal(indices, g["indices"])
    assert spatial.neighbor_table_hash(pool, indptr, indices) == str(g["table_hash"])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("summation", [0, 1])
def test_neighbor_table_after_steps(cuda_required, dtype, summation):
    """Queries on a context whose storage was re-sorted by steps (the lazy
    reference order, pres != identity, and relaid slot storage)."""
    from paper_2105_00039_b200 import _native as N
    from paper_2105_00039_b200.pool import AgentPool, PrecisionMode
    from paper_2105_00039_b200.workloads import jittered_lattice_positions
    pos = jittered_lattice_positions(18, spacing=7.5, jitter=1.5, seed=3)
    prec = PrecisionMode.FP64 if dtype == np.float64 else PrecisionMode.FP32
    pool = AgentPool.from_arrays(pos, 10.0, 0.4, prec)
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, summation)
    try:
        ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
        with pytest.raises(RuntimeError):
            ctx.neighbor_counts(5.0)                  # no grid over the stored positions yet
        for k in range(3):
            ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24, N.CG_STEP_SORT if k != 1 else 0)
        with pytest.raises(RuntimeError):
            ctx.neighbor_counts(5.0)                  # the step moved the agents off its grid
        ctx.build_grid(12.0, 1 << 24)
        indptr, indices = ctx.neighbor_csr(9.0)
        cols = ctx.download()
    finally:
        ctx.close()
    want_p, want_i = oracle.neighbor_csr(cols["px"], cols["py"], cols["pz"], cols["uid"], 9.0)
    assert np.array_equal(indptr, want_p)
    assert np.array_equal(indices, want_i)


def test_neighbor_rows_large_pool(cuda_required):
    """300k agents: symmetric table, rows uid-ascending, and a sample of rows
    against the brute-force predicate."""
    from paper_2105_00039_b200 import spatial
    from paper_2105_00039_b200.pool import AgentPool
    rng = np.random.default_rng(7)
    n = 300_000
    pool = AgentPool.from_arrays(rng.uniform(0, 400, (n, 3)), 10.0, 0.4)
    grid = spatial.build_grid(pool)
    r = 10.0
    indptr, indices = spatial.neighbor_csr(grid, pool, r)
    counts = np.diff(indptr)
    assert counts.sum() % 2 == 0
    owner = np.repeat(np.arange(n), counts)
    fwd = np.sort(owner * n + indices)
    rev = np.sort(indices * n + owner)
    assert np.array_equal(fwd, rev)
    same_row = owner[1:] == owner[:-1]
    assert np.all(np.diff(pool.uid[indices].astype(np.int64))[same_row] > 0)
    x, y, z = pool.position_x, pool.position_y, pool.position_z
    for i in rng.integers(0, n, 64):
        d2 = (x - x[i]) ** 2 + (y - y[i]) ** 2 + (z - z[i]) ** 2
        hit = np.flatnonzero(d2 <= r * r)
        hit = hit[hit != i]
        hit = hit[np.argsort(pool.uid[hit])]
        assert np.array_equal(indices[indptr[i]:indptr[i + 1]], hit)


def test_neighbor_radius_errors(cuda_required):
    from paper_2105_00039_b200 import spatial
    from paper_2105_00039_b200.pool import AgentPool
    pool = AgentPool.from_arrays(np.random.default_rng(0).uniform(0, 50, (500, 3)), 10.0, 0.4)
    grid = spatial.build_grid(pool)
    with pytest.raises(spatial.StencilTooSmallError):
        spatial.neighbor_counts(grid, pool, 10.5)
    with pytest.raises(ValueError):
        spatial.neighbor_csr(grid, pool, 0.0)
    pool.position_x[0] += 100.0                     # grid no longer indexes this pool
    with pytest.raises(ValueError):
        spatial.neighbor_counts(grid, pool, 5.0)
