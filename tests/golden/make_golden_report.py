"""Reference report CSVs (reference bench.py:210-330) for the report layer
(SURVEY.md 8f row 4): benchmark B over two densities and a small benchmark A
with the Serial strategy, plus a grid lookup row, written by the reference's
write_report.  Build container only (reference at /root/reference); outputs
tests/golden/report_*.csv are committed.

Usage (repo root):
  NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONDONTWRITEBYTECODE=1 \\
    python tests/golden/make_golden_report.py
"""

from __future__ import annotations

import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from cellgrid import bench, engine  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def main():
    b = bench.BenchmarkBConfig(agent_count=3000, target_densities=(3.0, 17.0), steps=2,
                               strategy=engine.Serial(), sample_count=300)
    rows = bench.run_benchmark_b(b)
    a = bench.BenchmarkAConfig(side_count=6, steps=3, strategy=engine.Serial(), repeats=1)
    rows += bench.run_benchmark_a(a, warmup=False)
    pool = bench.spawn_benchmark_a_pool(a)
    rows += bench.lookup_comparison_rows(pool, pool.max_diameter(), bench="A", backends=("grid",))
    bench.write_report(rows, os.path.join(OUT, "report_ref.csv"))
    for r in rows:
        print(r.bench, r.strategy, r.agents, r.force_evals, r.candidates, r.state_hash[:12], r.neighbor_hash[:12])


if __name__ == "__main__":
    main()
