"""Per-source-line totals from an ncu report: instructions executed and warp
stall samples, for the lines carrying most of either.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname = [], None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] in ("Function Name", "Line No"):
        hdr = rec if rec[0] == "Line No" else None
        continue
    if rec[0].isdigit() and len(rec) > 8 and rec[2] == "-":   # a source line (its SASS rows follow)
        try:
            rows.append((fname, int(rec[0]), rec[1].strip()[:70], int(rec[4]), int(rec[7])))
        except ValueError:
            pass
tot_s = sum(r[3] for r in rows) or 1
tot_i = sum(r[4] for r in rows) or 1
print("total stall samples %d, warp instructions %d" % (tot_s, tot_i))
for r in sorted(rows, key=lambda r: -(r[3] / tot_s + r[4] / tot_i))[:top]:
    print("%-14s %4d  samp %5.1f%%  inst %5.1f%%  %s" % (r[0], r[1], 100.0 * r[3] / tot_s, 100.0 * r[4] / tot_i, r[2]))
