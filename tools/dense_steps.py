"""Per-step device times of the first steps of the frozen benchmark-B pools
(C3): step 0 grid sweep, step 1 the list-building grid sweep, then list steps.

usage: python tools/dense_steps.py [density ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native as N, workloads  # noqa: E402

for d in [float(a) for a in sys.argv[1:]] or [27.0, 100.0]:
    pool = workloads.c3(d)
    for skin in (-1, 0):
        ctx = N.Context(0, pool.dtype)
        ctx.set_option(N.CG_OPT_SUMMATION, 1)
        ctx.set_option(N.CG_OPT_LIST_SKIN, skin)
        ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
        sts = [ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24, N.CG_STEP_SORT | N.CG_STEP_FREEZE)
               for _ in range(8)]
        print(json.dumps({"density": d, "lists": skin != 0, "kinds": [int(s.sweep_kind) for s in sts],
                          "ms": [round(s.t_total_ms, 3) for s in sts]}), flush=True)
        ctx.close()
