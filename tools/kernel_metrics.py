"""profiles/kernel_metrics.json from ncu --set full reports: per kernel, DRAM
bytes read + written per launch (the bench line's roofline.traffic) and the
FP64 pipe's busy fraction (roofline.fp64_pipe_frac).

usage: python tools/kernel_metrics.py <config_precision> <kernel name>=<report.ncu-rep>[@<template>] ...
e.g.   python tools/kernel_metrics.py c4_fp64 list_sweep_kernel=gpurun_out/prof_list.ncu-rep
A report holding several launches: @<substring of the kernel name> picks the
first launch whose name contains it (e.g. "@<double, 1, 1, 0>").
Entries of other configs / kernels already in the file are kept.
"""
import csv
import io
import json
import os
import subprocess
import sys

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "kernel_metrics.json")


def metrics(rep, pick=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units = rows[0], rows[1]
    col = head.index("Kernel Name")
    vals = next(r for r in rows[2:] if pick is None or pick in r[col])
    d = dict(zip(head, vals))
    u = dict(zip(head, units))

    def num(k):
        v = float(d[k].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(u.get(k, "byte"), 1)
        return v * scale
    return {"traffic": int(num("dram__bytes_read.sum") + num("dram__bytes_write.sum")),
            "fp64_pipe_frac": float(d["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"]) / 100.0,
            "issue_active_frac": float(d["smsp__issue_active.avg.pct_of_peak_sustained_active"]) / 100.0,
            "ncu_ms": num("gpu__time_duration.sum") * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3,
                                                       "ms": 1.0, "msecond": 1.0}[u.get("gpu__time_duration.sum", "ms")],
            "kernel_name": d.get("Kernel Name", "")}


def main():
    cfg = sys.argv[1]
    try:
        data = json.load(open(OUT))
    except (OSError, ValueError):
        data = {}
    for arg in sys.argv[2:]:
        name, rep = arg.split("=", 1)
        rep, _, pick = rep.partition("@")
        m = metrics(rep, pick or None)
        m["source"] = "ncu --set full --clock-control none, one launch: %s" % os.path.basename(rep)
        data.setdefault(cfg, {})[name] = m
    json.dump(data, open(OUT, "w"), indent=1)
    print(json.dumps(data, indent=1))


if __name__ == "__main__":
    main()
