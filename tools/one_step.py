"""Minimal driver for ncu captures: upload a config and run a few steps.

usage: python tools/one_step.py <c1|c2|c4|c3_<d>>[f] [summation 0|1] [relayout_every k] [steps]
(env SWEEP=0|1 selects the sweep kernel: 0 reference-order, 1 production; PATH_OPT = CG_OPT_PATH; SKIN = CG_OPT_LIST_SKIN)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2105_00039_b200 import _native, workloads  # noqa: E402
from paper_2105_00039_b200.pool import PrecisionMode  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
summ = int(sys.argv[2]) if len(sys.argv) > 2 else 1
order = int(sys.argv[3]) if len(sys.argv) > 3 else 1
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 2
pm = PrecisionMode.FP32 if name.endswith("f") else PrecisionMode.FP64
base = name.rstrip("f")
makers = {"c1": lambda: workloads.c1(pm), "c2": lambda: workloads.c2(pm),
          "c4": lambda: workloads.c4(pm)}
pool = makers.get(base, lambda: workloads.c3(float(base[3:]), pm))()
ctx = _native.Context(0, pool.dtype)
ctx.set_option(_native.CG_OPT_SUMMATION, summ)
ctx.set_option(_native.CG_OPT_RELAYOUT_EVERY, order)
ctx.set_option(_native.CG_OPT_SWEEP, int(os.environ.get("SWEEP", "1")))
ctx.set_option(_native.CG_OPT_PATH, int(os.environ.get("PATH_OPT", "0")))
ctx.set_option(_native.CG_OPT_LIST_SKIN, int(os.environ.get("SKIN", "-1")))
ctx.upload(pool.position_x, pool.position_y, pool.position_z, pool.diameter, pool.adherence,
           pool.uid)
tf, tt = [], []
for k in range(steps):
    st = ctx.step(np.array([2.0, 1.0, 0.01, 3.0, 1.0]), None, 1 << 24, 1)
    tf.append(st.t_force_ms)
    tt.append(st.t_total_ms)
print("force %.3f ms total %.3f ms (median of %d; mean total %.3f) lists %s" % (
    np.median(tf[1:] or tf), np.median(tt[1:] or tt), steps, np.mean(tt[1:] or tt), ctx.list_stats()))
if os.environ.get("VERBOSE"):
    print(" ".join("%.2f" % t for t in tt))
