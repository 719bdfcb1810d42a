#!/usr/bin/env python
"""Top CUDA source lines by warp-stall samples for one kernel of an ncu report.

    python scripts/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [--top 30] [--skip N]
"""
import argparse
import csv
import io
import subprocess

ap = argparse.ArgumentParser()
ap.add_argument("rep")
ap.add_argument("kernel")
ap.add_argument("--top", type=int, default=30)
ap.add_argument("--skip", type=int, default=0)
a = ap.parse_args()
out = subprocess.run(["ncu", "-i", a.rep, "--page", "source", "--csv", "-k", "regex:" + a.kernel,
                      "--launch-skip", str(a.skip), "--launch-count", "1", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
for rec in csv.reader(io.StringIO(out)):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] == "Function Name":
        continue
    if len(rec) < 8 or rec[2] != "-":  # SASS rows interleaved: keep CUDA-line rows only
        continue
    try:
        samp, nis, inst = int(rec[4]), int(rec[5]), int(rec[7])
    except ValueError:
        continue
    rows.append((samp, nis, inst, f"{fname}:{rec[0]}", rec[1].strip()[:90]))
tot = sum(r[0] for r in rows) or 1
rows.sort(reverse=True)
print(f"total samples {tot}")
for s, n, i, loc, src in rows[:a.top]:
    print(f"{100 * s / tot:5.1f}% {n:7d} {i:9d}  {loc:22s} {src}")
