"""Gpu rows of the reference's benchmark harness, on the device.

tests/golden/report_ref.csv was written by the reference's own harness
(tests/golden/make_golden_report.py: cellgrid.bench.run_benchmark_b/a and
lookup_comparison_rows with the Serial strategy).  The harness itself exists
only in the build container, where tests/test_refstub.py drives it with the
Gpu strategy installed; here the same engine calls it would make for a
``Gpu()`` row run on the B200 -- benchmark B: a frozen warm-up step then the
timed steps (bench.py:241-262); benchmark A: engine.run with growth
(bench.py:210-238); the grid lookup row (bench.py:264-310) -- and every
deterministic column must equal the reference-written row."""

import csv
import os

import pytest

REF = os.path.join(os.path.dirname(__file__), "golden", "report_ref.csv")

pytestmark = pytest.mark.gpu


def _ref_rows():
    with open(REF, newline="") as f:
        return list(csv.DictReader(f))


def _cols(stats, agents, state_hash):
    last = stats[-1]
    return {"agents": agents, "force_evals": sum(s.force_evals for s in stats),
            "candidates": sum(s.candidates for s in stats), "bytes_modeled": sum(s.bytes_modeled for s in stats),
            "state_hash": state_hash, "grid_dims": "%dx%dx%d" % tuple(last.grid_dims),
            "grid_occupied_boxes": last.grid_occupied_boxes, "grid_max_occupancy": last.grid_max_occupancy,
            "divisions": sum(s.divisions for s in stats)}


def _check(mine, ref):
    for k, v in mine.items():
        assert str(v) == ref[k], (ref["bench"], k, v, ref[k])


def test_benchmark_b_rows(cuda_required):
    import paper_2105_00039_b200 as P
    from paper_2105_00039_b200.workloads import box_side_for_density
    for ref in [r for r in _ref_rows() if r["bench"] == "B"]:
        side = box_side_for_density(3000, 5.0, float(ref["density_target"]))
        pool = P.AgentPool.spawn_random(3000, P.Aabb.cube(side), 10.0, 0.4, 0)
        sim = P.SimulationConfig(strategy=P.Gpu(), steps=2, freeze_displacement=True)
        P.step(pool, sim, 0)                        # warm-up, untimed
        stats = [P.step(pool, sim, k + 1) for k in range(2)]
        _check(_cols(stats, pool.count, pool.state_hash()), ref)


def test_benchmark_a_row(cuda_required):
    import paper_2105_00039_b200 as P
    ref = [r for r in _ref_rows() if r["bench"] == "A" and r["strategy"] == "serial"][0]
    sim = P.SimulationConfig(strategy=P.Gpu(), steps=3, growth=P.GrowthParams(100.0, 12.0))
    report = P.run(P.AgentPool.spawn_grid(6, 10.0, 10.0, 0.4), sim)
    _check(_cols(report.steps, report.final_count, report.final_state_hash), ref)


def test_lookup_row(cuda_required):
    import paper_2105_00039_b200 as P
    from paper_2105_00039_b200 import spatial
    ref = [r for r in _ref_rows() if r["strategy"] == "lookup"][0]
    pool = P.AgentPool.spawn_grid(6, 10.0, 10.0, 0.4)
    radius = pool.max_diameter()
    grid = spatial.build_grid(pool, interaction_radius=radius)
    indptr, indices = spatial.neighbor_csr(grid, pool, radius)
    assert spatial.neighbor_table_hash(pool, indptr, indices) == ref["neighbor_hash"]
    assert str(int(indptr[-1])) == ref["candidates"]
    assert "%dx%dx%d" % tuple(grid.dims) == ref["grid_dims"]
