import os, sys
sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2105_00039_b200 import _native, workloads
from paper_2105_00039_b200.pool import PrecisionMode
pool = workloads.c4(PrecisionMode.FP64)
ctx = _native.Context(0, pool.dtype)
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence, pool.uid)
c0 = ctx.download(columns=("px","py","pz","uid")); o=np.argsort(c0["uid"]); P0=np.stack([c0[k][o] for k in ("px","py","pz")],1)
acc=0.0
for k in range(24):
    ctx.step(np.array([2.0,1.0,0.01,3.0,1.0]), None, 1<<24, 1)
    c = ctx.download(columns=("px","py","pz","dx","dy","dz","uid")); o=np.argsort(c["uid"])
    P=np.stack([c[q][o] for q in ("px","py","pz")],1)
    d=np.sqrt(c["dx"]**2+c["dy"]**2+c["dz"]**2).max()
    acc+=d
    net=np.sqrt(((P-P0)**2).sum(1))
    print("step %2d sum(max|d|) %.3f  max net %.3f  p99.99 net %.3f"%(k,acc,net.max(),np.quantile(net,0.9999)),flush=True)
