"""Benchmark B (density sweep, reference bench.py:241-261) through the report
layer: one CSV row per density, GPU strategy, the reference's CSV columns.

usage: python tools/bench_b_csv.py OUT.csv [agent_count] [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2105_00039_b200 import report  # noqa: E402

out = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 100_000
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
rows = report.run_benchmark_b(report.BenchmarkBConfig(agent_count=n, steps=steps))
report.write_report(rows, out)
for r in rows:
    print(r.density_target, round(r.density_measured, 2), r.agents, r.steps, round(r.t_total_ms, 3), r.force_evals)
