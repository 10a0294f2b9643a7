"""A/B timing of library builds: per step kind, the mean device time of the
step (CUDA events inside the library) over a resident run.

usage: CG_LIB=path/to/lib.so python tools/ab_steps.py <config> <steps> [tag]
config: c4, c2, c1, c3_<density>, suffix 'f' = fp32; env SKIN = CG_OPT_LIST_SKIN,
FREEZE=1 freezes displacements.  Prints one JSON line.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native, workloads  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
tag = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(os.environ.get("CG_LIB", "default"))
pm = PrecisionMode.FP32 if name.endswith("f") else PrecisionMode.FP64
base = name.rstrip("f")
makers = {"c1": lambda: workloads.c1(pm), "c2": lambda: workloads.c2(pm), "c4": lambda: workloads.c4(pm)}
pool = makers.get(base, lambda: workloads.c3(float(base[3:]), pm))()
ctx = _native.Context(0, pool.dtype)
ctx.set_option(_native.CG_OPT_LIST_SKIN, int(os.environ.get("SKIN", "-1")))
if os.environ.get("INNER"):
    ctx.set_option(_native.CG_OPT_INNER_LIST, int(os.environ["INNER"]))
if os.environ.get("MID"):
    ctx.set_option(_native.CG_OPT_MID_LIST, int(os.environ["MID"]))
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
flags = _native.CG_STEP_SORT | (_native.CG_STEP_FREEZE if os.environ.get("FREEZE") else 0)
kinds, tot, force, evals = [], [], [], []
for k in range(steps):
    st = ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24, flags)
    kinds.append(int(st.sweep_kind))
    tot.append(st.t_total_ms)
    force.append(st.t_force_ms)
    evals.append(int(st.force_evals))
out = {"tag": tag, "config": name, "steps": steps}
w = slice(3, None)   # skip the upload's plain sweep and the first list epoch's start
out["mean_ms"] = float(np.mean(tot[w]))
for kd, nm in ((0, "grid"), (1, "build"), (2, "list")):
    sel = [i for i in range(3, steps) if kinds[i] == kd]
    if sel:
        out[nm] = {"n": len(sel), "total_ms": float(np.mean([tot[i] for i in sel])),
                   "force_ms": float(np.mean([force[i] for i in sel]))}
out["evals_last"] = evals[-1]
out["evals_hash"] = int(np.sum(np.array(evals, dtype=np.int64) * np.arange(1, steps + 1)))
got = ctx.download()
out["pos_hash"] = float(np.sum(got["px"] * 1.0 + got["py"] * 2.0 + got["pz"] * 3.0))
out["list_stats"] = ctx.list_stats()
print(json.dumps(out), flush=True)
