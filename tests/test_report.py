"""Report layer against a CSV written by the reference's
own harness (tests/golden/make_golden_report.py): the file reads and writes
back byte for byte, and the same benchmark rows run through the Gpu strategy
reproduce every deterministic column (counters, densities, grid statistics,
state and neighbour-table hashes)."""

import os

import pytest

REF = os.path.join(os.path.dirname(__file__), "golden", "report_ref.csv")
DETERMINISTIC = ("bench", "backend", "precision", "density_target", "density_measured", "agents", "steps",
                 "force_evals", "candidates", "bytes_modeled", "ai_flops_per_byte", "state_hash",
                 "neighbor_hash", "grid_dims", "grid_occupied_boxes", "grid_max_occupancy", "divisions")


def test_report_csv_round_trip(tmp_path):
    from paper_2105_00039_b200 import report
    rows = report.read_report(REF)
    assert len(rows) == 4 and rows[0].bench == "B" and rows[-1].strategy == "lookup"
    out = tmp_path / "r.csv"
    report.write_report(rows, out)
    assert out.read_bytes() == open(REF, "rb").read()
    assert report.CSV_HEADER.split(",")[-1] == "ai_flops_per_byte"


@pytest.mark.gpu
def test_gpu_rows_match_reference_rows(cuda_required):
    import paper_2105_00039_b200 as P
    from paper_2105_00039_b200 import report
    ref = report.read_report(REF)
    b = report.BenchmarkBConfig(agent_count=3000, target_densities=(3.0, 17.0), steps=2,
                                strategy=P.Gpu(), sample_count=300)
    rows = report.run_benchmark_b(b)
    a = report.BenchmarkAConfig(side_count=6, steps=3, strategy=P.Gpu(), repeats=1)
    rows += report.run_benchmark_a(a, warmup=False)
    pool = report.spawn_benchmark_a_pool(a)
    rows += report.lookup_comparison_rows(pool, pool.max_diameter(), bench="A", backends=("grid",))
    assert len(rows) == len(ref)
    for mine, theirs in zip(rows, ref):
        for col in DETERMINISTIC:
            assert getattr(mine, col) == getattr(theirs, col), (mine.bench, col)
        assert mine.strategy == ("lookup" if theirs.strategy == "lookup" else P.strategy_label(P.Gpu()))
