#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into profiles/: key metrics per kernel launch.

usage: python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep profiles/r01_fused.md [--traffic-key KEY]
Writes a markdown table and, with --traffic-key, records DRAM bytes per launch into
profiles/traffic.json (read by bench.py for the roofline "traffic" field).
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = [
    ("GPU Speed Of Light Throughput", "Duration"),
    ("GPU Speed Of Light Throughput", "DRAM Throughput"),
    ("GPU Speed Of Light Throughput", "Memory Throughput"),
    ("GPU Speed Of Light Throughput", "Compute (SM) Throughput"),
    ("GPU Speed Of Light Throughput", "SM Frequency"),
    ("Compute Workload Analysis", "Executed Ipc Active"),
    ("Compute Workload Analysis", "Issue Slots Busy"),
    ("Memory Workload Analysis", "Memory Throughput"),
    ("Memory Workload Analysis", "L1/TEX Hit Rate"),
    ("Memory Workload Analysis", "L2 Hit Rate"),
    ("Scheduler Statistics", "Eligible Warps Per Scheduler"),
    ("Warp State Statistics", "Warp Cycles Per Issued Instruction"),
    ("Warp State Statistics", "Avg. Active Threads Per Warp"),
    ("Instruction Statistics", "Executed Instructions"),
    ("Launch Statistics", "Registers Per Thread"),
    ("Launch Statistics", "Grid Size"),
    ("Launch Statistics", "Block Size"),
    ("Launch Statistics", "Dynamic Shared Memory Per Block"),
    ("Occupancy", "Achieved Active Warps Per SM"),
    ("Occupancy", "Theoretical Occupancy"),
]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__inst_executed.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def run(args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True).stdout


def main():
    rep, out = sys.argv[1], sys.argv[2]
    key = None
    if "--traffic-key" in sys.argv:
        key = sys.argv[sys.argv.index("--traffic-key") + 1]
    det = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "details", "--csv"]))))
    hdr = det[0]
    rows = [dict(zip(hdr, r)) for r in det[1:]]
    raw = list(csv.reader(io.StringIO(run(["-i", rep, "--page", "raw", "--csv"]))))
    rhdr = raw[0]
    runits = dict(zip(rhdr, raw[1])) if len(raw) > 1 else {}
    rraw = [dict(zip(rhdr, r)) for r in raw[2:]] if len(raw) > 2 else []
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}

    def val(rr, k):
        return float(rr[k].replace(",", "")) * scale.get(runits.get(k, "byte"), 1)
    kernels = {}
    for r in rows:
        kid = (r.get("ID"), r.get("Kernel Name"))
        kernels.setdefault(kid, {})[(r.get("Section Name"), r.get("Metric Name"))] = (
            r.get("Metric Value"), r.get("Metric Unit"))
    lines = [f"# ncu summary: `{os.path.basename(rep)}`", ""]
    traffic = {}
    for i, ((kid, name), m) in enumerate(kernels.items()):
        lines.append(f"## launch {kid}: `{name[:140]}`")
        lines.append("")
        lines.append("| metric | value | unit |")
        lines.append("|---|---|---|")
        for sec, met in WANT:
            if (sec, met) in m:
                v, u = m[(sec, met)]
                lines.append(f"| {met} | {v} | {u} |")
        if i < len(rraw):
            rr = rraw[i]
            for k in RAW:
                if k in rr:
                    lines.append(f"| {k} | {rr[k]} | {runits.get(k, '')} |")
            try:
                rd = val(rr, "dram__bytes_read.sum")
                wr = val(rr, "dram__bytes_write.sum")
                traffic[kid] = rd + wr
                lines.append(f"| dram read+write | {rd + wr:.4g} | byte |")
            except ValueError:
                pass
        lines.append("")
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    open(out, "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
    if key and traffic:
        tf = os.path.join(os.path.dirname(out), "traffic.json")
        d = json.load(open(tf)) if os.path.exists(tf) else {}
        d[key] = list(traffic.values())[0]
        json.dump(d, open(tf, "w"), indent=1)


if __name__ == "__main__":
    main()
