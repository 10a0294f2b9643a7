"""Per-config device timings for BASELINE.json's configurations (C1-C4), fp64
and fp32, C3 with and without the Z-order sort; one JSON line per run (mean
over 12 steps after 3 warm-up steps; step kinds 0 grid sweep, 1 list build,
2 list sweep).

usage: python tools/configs.py [names...]   names: c1 c2 c2f c4 c4f c3_<d> c3_<d>_nosort
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native as N, workloads  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402


def run(name, steps=12, warm=3):
    prec = PrecisionMode.FP32 if name.endswith("f") else PrecisionMode.FP64
    base = name.rstrip("f")
    nosort = base.endswith("_nosort")
    base = base.replace("_nosort", "")
    if base == "c1":
        pool = workloads.c1(prec)
    elif base == "c2":
        pool = workloads.c2(prec)
    elif base == "c4":
        pool = workloads.c4(prec)
    else:
        pool = workloads.c3(float(base[3:]), prec)
    ctx = N.Context(0, pool.dtype)
    ctx.set_option(N.CG_OPT_SUMMATION, 1)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    params = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
    flags = 0 if nosort else N.CG_STEP_SORT
    if base.startswith("c3"):
        flags |= N.CG_STEP_FREEZE     # benchmark B is frozen (bench.py:250-255)
    for _ in range(warm):
        ctx.step(params, None, 1 << 24, flags)
    sts = [ctx.step(params, None, 1 << 24, flags) for _ in range(steps)]
    tot = float(np.mean([s.t_total_ms for s in sts]))
    st = sts[-1]
    kinds = [int(s.sweep_kind) for s in sts]
    out = {"config": name, "agents": pool.count, "dtype": str(np.dtype(pool.dtype)), "sort": not nosort,
           "ms_total": tot, "ms_total_median": float(np.median([s.t_total_ms for s in sts])),
           "step_kinds": {k: kinds.count(k) for k in sorted(set(kinds))},
           "ms_grid": st.t_grid_ms, "ms_sort": st.t_sort_ms, "ms_force": st.t_force_ms,
           "agent_updates_per_s": pool.count / (tot * 1e-3),
           "pair_interactions_per_s": st.force_evals / (tot * 1e-3),
           "evals_per_agent": st.force_evals / pool.count, "cands_per_agent": st.candidates / pool.count,
           "dims": list(st.grid_dims), "max_occupancy": st.grid_max_occupancy}
    ctx.close()
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["c1", "c2", "c2f", "c4", "c4f"]:
        run(nm)
