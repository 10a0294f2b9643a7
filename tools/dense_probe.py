import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_2105_00039_b200 import _native as N
from paper_2105_00039_b200.geometry import Aabb
from paper_2105_00039_b200.pool import AgentPool
from paper_2105_00039_b200.workloads import box_side_for_density
pool = AgentPool.spawn_random(12000, Aabb.cube(box_side_for_density(12000, 5.0, 27.0)), 10.0, 0.4, 5)
ctx = N.Context(0, pool.dtype)
ctx.set_option(N.CG_OPT_SUMMATION, 0)
ctx.set_option(N.CG_OPT_LIST_SKIN, -1)
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
P = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
for k in range(8):
    st = ctx.step(P, None, 1 << 24, N.CG_STEP_SORT | N.CG_STEP_FREEZE)
    print(k, st.sweep_kind, st.force_evals, st.candidates, flush=True)
