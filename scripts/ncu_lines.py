#!/usr/bin/env python
"""Per-source-line instruction and stall attribution of one kernel from an ncu report.

usage: python scripts/ncu_lines.py REPORT.ncu-rep OBJ.o MANGLED_SUBSTR [--top N]

The ncu CLI prints per-SASS-instruction metrics only; this joins them with the line table
nvdisasm -g prints for the same cubin (the .o under paper_2605_00342_b200/build/ the profiled
library was linked from), by offset from the function start.
"""
import collections
import csv
import io
import re
import subprocess
import sys
import tempfile
import os


def sass_lines(obj, fn_sub):
    d = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                   capture_output=True)
    cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True,
                         text=True).stdout
    out, on, cur = {}, False, None
    for ln in txt.splitlines():
        if ln.startswith("//---------------------"):
            on = fn_sub in ln
            continue
        if not on:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", ln)
        if m:
            out[int(m.group(1), 16)] = (cur, m.group(2))
    return out


def main():
    rep, obj, fn_sub = sys.argv[1:4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    table = sass_lines(obj, fn_sub)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    ci = hdr.index("Instructions Executed")
    cs = hdr.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[hdr_i + 1:] if r and r[0].startswith("0x")]
    a0 = int(body[0][0], 16)
    inst = collections.Counter()
    stall = collections.Counter()
    opc = collections.Counter()
    tot_i = tot_s = 0
    for r in body:
        off = int(r[0], 16) - a0
        key, _ = table.get(off, (("?", 0), ""))
        n = int(r[ci] or 0)
        s = int(r[cs] or 0)
        inst[key] += n
        stall[key] += s
        op = r[1].strip().split()[0] if r[1].strip() else "?"
        if op.startswith("@"):
            op = r[1].strip().split()[1]
        opc[op.split(".")[0]] += n
        tot_i += n
        tot_s += s
    print(f"total instructions {tot_i}, stall samples {tot_s}")
    print("\n# top lines by instructions executed")
    for key, n in inst.most_common(top):
        print(f"{key[0]}:{key[1]:<6} inst {n:>12} ({100 * n / tot_i:5.1f}%)  stall {100 * stall[key] / max(tot_s, 1):5.1f}%")
    print("\n# top lines by stall samples")
    for key, n in stall.most_common(top // 2):
        print(f"{key[0]}:{key[1]:<6} stall {100 * n / max(tot_s, 1):5.1f}%  inst {100 * inst[key] / tot_i:5.1f}%")
    print("\n# opcodes")
    for op, n in opc.most_common(30):
        print(f"{op:<10} {n:>12} ({100 * n / tot_i:5.1f}%)")


if __name__ == "__main__":
    main()
