"""The Gpu strategy installed into the UNMODIFIED reference package
(paper_2105_00039_b200.refstub = the INTEGRATION.md section 2 stub) and driven
by the reference's own benchmark harness (cellgrid.bench.run_benchmark_a/b,
bench.py:210-262): ``gpu(0)`` rows appear beside the reference's ``serial``
rows and agree with them column for column on everything deterministic.

CPU test: the reference is importable only in the build container, and the
native context is replaced by the oracle-backed mock (tests/native_mock.py), so
what is checked is the plumbing above the C ABI -- config and pool
translation, StepStats, growth, labels, the CSV layer.  The device path under
the same engine.step is checked against the oracle by the GPU suite."""

import os

import pytest

REF_SRC = "/root/reference/pkg/src"
DETERMINISTIC = ("bench", "backend", "precision", "density_target", "density_measured", "agents", "steps",
                 "force_evals", "candidates", "bytes_modeled", "ai_flops_per_byte", "state_hash",
                 "neighbor_hash", "grid_dims", "grid_occupied_boxes", "grid_max_occupancy", "divisions")


@pytest.fixture
def cellgrid(monkeypatch):
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference package not present (GPU box)")
    pytest.importorskip("numba")
    monkeypatch.syspath_prepend(REF_SRC)
    import cellgrid as cg
    import cellgrid.bench  # noqa: F401
    from paper_2105_00039_b200 import engine, refstub
    from native_mock import MockContext
    monkeypatch.setattr(engine, "_context", lambda strategy, dtype: MockContext(strategy.device, dtype))
    refstub.install(cg)
    yield cg
    refstub.uninstall(cg)


def _pairs(rows):
    serial = [r for r in rows if r.strategy == "serial"]
    gpu = [r for r in rows if r.strategy.startswith("gpu(")]
    assert len(serial) == len(gpu) > 0
    return zip(serial, gpu)


def test_benchmark_b_rows(cellgrid, tmp_path):
    from paper_2105_00039_b200 import Gpu, report
    cfg = cellgrid.bench.BenchmarkBConfig(agent_count=2000, target_densities=(3.0, 17.0), steps=2,
                                          sample_count=200)
    rows = report.run_benchmark_b(cfg, [cellgrid.engine.Serial(), Gpu()], cellgrid=cellgrid)
    for s, g in _pairs(rows):
        assert g.strategy == "gpu(0)"
        for col in DETERMINISTIC:
            assert getattr(s, col) == getattr(g, col), col
    out = tmp_path / "b.csv"
    cellgrid.bench.write_report(rows, out)
    back = cellgrid.bench.read_report(out)
    assert [r.strategy for r in back] == [r.strategy for r in rows]


def test_benchmark_a_rows_with_growth(cellgrid):
    from paper_2105_00039_b200 import Gpu, report
    cfg = cellgrid.bench.BenchmarkAConfig(side_count=5, steps=6, repeats=1)
    rows = report.run_benchmark_a(cfg, [cellgrid.engine.Serial(), Gpu()], cellgrid=cellgrid, warmup=False)
    for s, g in _pairs([r for r in rows if r.strategy != "lookup"]):
        for col in DETERMINISTIC:
            assert getattr(s, col) == getattr(g, col), col
        assert g.divisions > 0


def test_engine_run_and_labels(cellgrid):
    """engine.run of the reference with Gpu: the stub's step runs every step."""
    from paper_2105_00039_b200 import Gpu
    eng = cellgrid.engine
    assert eng.strategy_label(Gpu(1)) == "gpu(1)" and eng.strategy_label(eng.Serial()) == "serial"
    pool_a = cellgrid.pool.AgentPool.spawn_grid(4, 8.0, 10.0, 0.4)
    pool_b = cellgrid.pool.AgentPool.spawn_grid(4, 8.0, 10.0, 0.4)
    ra = eng.run(pool_a, eng.SimulationConfig(strategy=eng.Serial(), steps=3))
    rb = eng.run(pool_b, eng.SimulationConfig(strategy=Gpu(), steps=3))
    assert rb.strategy == "gpu(0)" and ra.final_state_hash == rb.final_state_hash
    assert [s.force_evals for s in ra.steps] == [s.force_evals for s in rb.steps]
    with pytest.raises(TypeError):
        eng.SimulationConfig(strategy=object())
