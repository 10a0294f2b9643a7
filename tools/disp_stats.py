"""Per-step displacement statistics (max / p99.9 / mean |d|) of a workload on
the device -- sizing data for neighbour-list reuse.
usage: python tools/disp_stats.py [c4|c2|c1|c3_<d>] [steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native, workloads  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
pm = PrecisionMode.FP64
pool = {"c4": workloads.c4, "c2": workloads.c2, "c1": workloads.c1}.get(
    name, lambda p: workloads.c3(float(name[3:]), p))(pm)
ctx = _native.Context(0, pool.dtype)
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
acc = 0.0
for k in range(steps):
    st = ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24, 1)
    c = ctx.download(columns=("dx", "dy", "dz"))
    nrm = np.sqrt(c["dx"] ** 2 + c["dy"] ** 2 + c["dz"] ** 2)
    acc += nrm.max()
    print("step %2d evals/agent %.2f  max|d| %.4f  p99.9 %.4f  mean %.5f  moving %.3f  sum(max) %.3f" % (
        k, st.force_evals / pool.count, nrm.max(), np.quantile(nrm, 0.999), nrm.mean(),
        np.count_nonzero(nrm) / pool.count, acc), flush=True)
