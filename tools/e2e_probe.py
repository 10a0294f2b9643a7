"""Where the end-to-end (host pool -> device step -> host pool) time goes:
upload, step and download timed separately with pinned host columns, plus the
raw pinned H2D / D2H copy rates for the same byte counts.
usage: python tools/e2e_probe.py [c4|c2|c1] [reps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2105_00039_b200 import _native, workloads  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
pool = {"c4": workloads.c4, "c2": workloads.c2, "c1": workloads.c1}[name](PrecisionMode.FP64)
pin = _native.PinnedArray.copy_of
cols = {k: pin(getattr(pool, a)) for k, a in (("px", "position_x"), ("py", "position_y"), ("pz", "position_z"),
                                                ("diameter", "diameter"), ("adherence", "adherence"), ("uid", "uid"))}
outs = {k: _native.PinnedArray.empty(pool.count, np.uint64 if k == "uid" else np.float64)
        for k in ("px", "py", "pz", "diameter", "adherence", "uid", "dx", "dy", "dz")}
ctx = _native.Context(0, pool.dtype)
P = np.array([2.0, 1.0, 0.01, 3.0, 1.0])
t = {"upload": [], "step": [], "download": []}
for r in range(reps + 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.upload(cols["px"], cols["py"], cols["pz"], cols["diameter"], cols["adherence"], cols["uid"])
    t1 = time.perf_counter()
    ctx.step(P, None, 1 << 24, _native.CG_STEP_SORT)
    t2 = time.perf_counter()
    ctx.download(into=outs)
    t3 = time.perf_counter()
    if r:
        t["upload"].append(t1 - t0)
        t["step"].append(t2 - t1)
        t["download"].append(t3 - t2)
for k, v in t.items():
    print("%-9s %8.2f ms" % (k, 1e3 * np.median(v)))
print("total     %8.2f ms" % (1e3 * sum(np.median(v) for v in t.values())))
# the fused call: step + download with the unchanged columns copied during the sweep
tf = []
for r in range(reps + 1):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx.upload(cols["px"], cols["py"], cols["pz"], cols["diameter"], cols["adherence"], cols["uid"])
    t1 = time.perf_counter()
    ctx.step_download(P, None, 1 << 24, _native.CG_STEP_SORT, into=outs)
    t2 = time.perf_counter()
    if r:
        tf.append(t2 - t1)
print("step_download %8.2f ms (step + download %.2f ms)" % (1e3 * np.median(tf),
                                                          1e3 * (np.median(t["step"]) + np.median(t["download"]))))
# raw pinned copy rates
n = pool.count
h = torch.empty(n * 6, dtype=torch.float64, pin_memory=True)
d = torch.empty(n * 6, dtype=torch.float64, device="cuda")
for label, src, dst in (("H2D", h, d), ("D2H", d, h)):
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    print("%s pinned %.1f GB/s (%.0f MB)" % (label, src.numel() * 8 / dt / 1e9, src.numel() * 8 / 1e6))
