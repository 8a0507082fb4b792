#!/usr/bin/env python
"""Per-source-line executed warp instructions from an ncu `--print-source cuda,sass` csv page.
usage: src_lines.py page.csv UNITS [TOP]"""
import csv
import sys

units = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
fname, out, tot = "?", [], 0
h = None
for r in csv.reader(open(sys.argv[1])):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if r[0] == "Line No":
        h = r
        iE = 7
        iS = 4
        continue
    if h is None or len(r) < 8 or not r[0]:
        continue
    try:
        n = int(r[iE])
    except ValueError:
        continue
    tot += n
    out.append((n, int(r[iS]) if r[iS].isdigit() else 0, f"{fname}:{r[0]}", r[1].strip()[:90]))
out.sort(reverse=True)
print(f"total {tot / units:.1f} warp instructions per unit")
for n, s, loc, src in out[:top]:
    print(f"{n / units:8.1f} {100 * n / tot:5.1f}%  samp {s:6d}  {loc:28s} {src}")
