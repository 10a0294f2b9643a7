"""C4 list-life probe: after a 'build' at step 0, per step k the largest
net displacement max|p - p0| and the relative spread D_rel: over each
4x4x4 block of build boxes plus its 26 neighbour blocks, the diameter of
the union of the (p - p0) bounding boxes.  A list with skin s could serve
while D_rel <= s and max|p - p0| < L/2 (Next)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2105_00039_b200 import _native, workloads  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402

pool = workloads.c4(PrecisionMode.FP64)
ctx = _native.Context(0, pool.dtype)
ctx.set_option(_native.CG_OPT_LIST_SKIN, 0)
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
L = 10.0


def grab():
    c = ctx.download(columns=("px", "py", "pz", "uid"))
    o = np.argsort(c["uid"])
    return torch.tensor(np.stack([c[k][o] for k in ("px", "py", "pz")], 1), device="cuda")


P0 = grab()
lo = P0.min(0).values
sb = torch.floor((P0 - lo) / (4 * L)).long()
dims = sb.max(0).values + 1
sid = (sb[:, 0] * dims[1] + sb[:, 1]) * dims[2] + sb[:, 2]
nsb = int(dims.prod())
for k in range(40):
    ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24, 1)
    if k % 4 != 3:
        continue
    D = grab() - P0
    mx = torch.full((nsb, 3), -1e30, device="cuda", dtype=torch.float64)
    mn = torch.full((nsb, 3), 1e30, device="cuda", dtype=torch.float64)
    for c in range(3):
        mx[:, c].scatter_reduce_(0, sid, D[:, c], "amax")
        mn[:, c].scatter_reduce_(0, sid, D[:, c], "amin")
    mx = mx.view(int(dims[0]), int(dims[1]), int(dims[2]), 3).permute(3, 0, 1, 2)[None]
    mn = mn.view(int(dims[0]), int(dims[1]), int(dims[2]), 3).permute(3, 0, 1, 2)[None]
    umx = torch.nn.functional.max_pool3d(mx, 3, 1, 1)
    umn = -torch.nn.functional.max_pool3d(-mn, 3, 1, 1)
    ext = (umx - umn).clamp(min=0)
    drel = float(ext.pow(2).sum(1).sqrt().max())
    print("step %2d max|p-p0| %.3f  D_rel %.3f" % (k, float(D.norm(dim=1).max()), drel), flush=True)
