import os, sys, time
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2105_00039_b200 import _native, workloads
from paper_2105_00039_b200.pool import PrecisionMode
pool = workloads.c4(PrecisionMode.FP64)
ctx = _native.Context(0, pool.dtype)
ctx.set_option(_native.CG_OPT_SUMMATION, 1)
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
P = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
for _ in range(5): ctx.step(P, None, 1 << 24, 1)
stream = torch.cuda.ExternalStream(ctx.stream)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); ctx.synchronize()
e0.record(stream)
ids = [ctx.step(P, None, 1 << 24, 1, wait=False) for _ in range(40)]
e1.record(stream); ctx.synchronize(); torch.cuda.synchronize()
wall = e0.elapsed_time(e1) / 40
sts = [ctx.fetch_stats(i) for i in ids[-40:]]
dev = np.mean([s.t_total_ms for s in sts])
kinds = [int(s.sweep_kind) for s in sts]
print("events per step %.3f ms; device (ev0->ev3) per step %.3f ms; gap %.3f ms; kinds %s" % (wall, dev, wall - dev, {k: kinds.count(k) for k in set(kinds)}))
