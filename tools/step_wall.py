"""Host wall time vs device time per step (C2 by default), for a summation mode.
usage: python tools/step_wall.py [c2|c4] [0|1]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native as N, workloads  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
summ = int(sys.argv[2]) if len(sys.argv) > 2 else 0
pool = workloads.c2() if name == "c2" else workloads.c4()
ctx = N.Context(0, pool.dtype)
ctx.set_option(N.CG_OPT_SUMMATION, summ)
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
P = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
for k in range(10):
    t0 = time.perf_counter()
    st = ctx.step(P, None, 1 << 24, N.CG_STEP_SORT)
    t1 = time.perf_counter()
    print(k, st.sweep_kind, "wall %.3f ms  device %.3f ms" % ((t1 - t0) * 1e3, st.t_total_ms), flush=True)
