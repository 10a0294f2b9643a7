"""Small dense pool, a few frozen then moving steps (lists on): a
compute-sanitizer target for the dense list build, the warp sweep's second
pass and the list sweep.  usage: python tools/dense_probe.py [n] [density] [summation]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native as N  # noqa: E402
from paper_2105_00039_b200.geometry import Aabb  # noqa: E402
from paper_2105_00039_b200.pool import AgentPool  # noqa: E402
from paper_2105_00039_b200.workloads import box_side_for_density  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 12000
dens = float(sys.argv[2]) if len(sys.argv) > 2 else 216.0
summation = int(sys.argv[3]) if len(sys.argv) > 3 else 0
pool = AgentPool.spawn_random(n, Aabb.cube(box_side_for_density(n, 10.0, dens)), 10.0, 0.4, 5)
ctx = N.Context(0, pool.dtype)
ctx.set_option(N.CG_OPT_SUMMATION, summation)
ctx.set_option(N.CG_OPT_LIST_SKIN, -1)
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
P = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
for k in range(8):
    st = ctx.step(P, None, 1 << 24, N.CG_STEP_SORT | (N.CG_STEP_FREEZE if k < 5 else 0))
    print(k, st.sweep_kind, st.force_evals, st.candidates, flush=True)
ctx.download()
ctx.close()
