#!/usr/bin/env python
"""Opcode histogram of an ncu SASS source page (csv): executed warp instructions per opcode
and per unit of work, plus stall samples.  usage: sass_hist.py page.csv UNITS [TOP]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
units = float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
h = rows[1]
iS, iE, iSamp = h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
iW = h.index("L1 Wavefronts Shared") if "L1 Wavefronts Shared" in h else None
ops, samp, wf = collections.Counter(), collections.Counter(), collections.Counter()
tot = tots = 0
for r in rows[2:]:
    if len(r) <= iE or not r[iE].isdigit():
        continue
    s = r[iS].strip()
    if s.startswith("@"):
        s = s.split(None, 1)[1]
    op = s.split()[0].split(".")[0] if s else "?"
    n = int(r[iE])
    ops[op] += n
    samp[op] += int(r[iSamp] or 0)
    if iW is not None and r[iW].isdigit():
        wf[op] += int(r[iW])
    tot += n
    tots += int(r[iSamp] or 0)
print(f"total warp instructions per unit: {tot / units:.1f}; shared wavefronts per unit: {sum(wf.values()) / units:.1f}")
for op, n in ops.most_common(top):
    print(f"{op:10s} {n / units:8.1f}/unit  {100 * n / tot:5.1f}%  samples {100 * samp[op] / max(tots, 1):5.1f}%  wf {wf[op] / units:6.1f}")
