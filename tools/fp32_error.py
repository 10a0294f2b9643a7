"""Measured error of the fp32 variant against the fp64 path (north star: "an
fp32 variant is reported separately with its measured error bound").

The fp32 pool is the fp64 pool downcast (pool.py:178-190 semantics: the same
layout), both stepped on the device; displacements and positions are matched by
uid.  Reports the max / 99.9th-percentile relative displacement error (per
agent, vector norm, agents with a non-zero fp64 displacement), the max absolute
position error, and the colliding-pair count difference.

usage: python tools/fp32_error.py [c1|c2|c4|c3_<d>] [steps]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native as N, workloads  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402


def make(name, prec):
    if name == "c1":
        return workloads.c1(prec)
    if name == "c2":
        return workloads.c2(prec)
    if name == "c4":
        return workloads.c4(prec)
    return workloads.c3(float(name[3:]), prec)


def run(pool, steps):
    ctx = N.Context(0, pool.dtype)
    ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
    evals = []
    for _ in range(steps):
        st = ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24, N.CG_STEP_SORT)
        evals.append(st.force_evals)
    cols = ctx.download()
    ctx.close()
    o = np.argsort(cols["uid"])
    return {k: v[o] for k, v in cols.items()}, evals


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c2"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    r64, e64 = run(make(name, PrecisionMode.FP64), steps)
    r32, e32 = run(make(name, PrecisionMode.FP32), steps)
    d64 = np.stack([r64[k] for k in ("dx", "dy", "dz")], 1)
    d32 = np.stack([r32[k].astype(np.float64) for k in ("dx", "dy", "dz")], 1)
    nrm = np.linalg.norm(d64, axis=1)
    moving = nrm > 0
    rel = np.linalg.norm(d32 - d64, axis=1)[moving] / nrm[moving]
    gate_flips = int(np.count_nonzero((np.linalg.norm(d32, axis=1) > 0) != moving))
    p64 = np.stack([r64[k] for k in ("px", "py", "pz")], 1)
    p32 = np.stack([r32[k].astype(np.float64) for k in ("px", "py", "pz")], 1)
    out = {"config": name, "steps": steps, "agents": int(d64.shape[0]),
           "moving_agents": int(moving.sum()),
           "disp_rel_err_max": float(rel.max()) if rel.size else 0.0,
           "disp_rel_err_p999": float(np.quantile(rel, 0.999)) if rel.size else 0.0,
           "disp_rel_err_median": float(np.median(rel)) if rel.size else 0.0,
           "adherence_gate_flips": gate_flips,
           "pos_abs_err_max": float(np.abs(p32 - p64).max()),
           "force_evals_fp64": e64, "force_evals_fp32": e32}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
