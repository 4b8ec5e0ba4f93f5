#!/usr/bin/env python3
"""Summarise an `ncu --set full` report (.ncu-rep) as text for profiles/:
per captured launch, the speed-of-light / occupancy / scheduler metrics, the
top warp-stall reasons and the FP64 / DMMA pipe utilisation.

usage: tools/ncu_full_summary.py report.ncu-rep "command description" > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

WANT = ["Duration", "Grid Size", "Block Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy", "Compute (SM) Throughput", "Memory Throughput",
        "DRAM Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "Issue Slots Busy", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Executed Instructions"]
PIPES = ["sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
         "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
         "dram__bytes_read.sum", "dram__bytes_write.sum"]


def csv_rows(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, title):
    print(f"ncu --set full --clock-control none: {title}")
    det = csv_rows(rep, "details")
    h = det[0]
    ii, ki, mi, vi, ui = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    launches = {}
    for r in det[1:]:
        if len(r) <= vi:
            continue
        d = launches.setdefault(r[ii], {"name": r[ki].split("(")[0], "m": {}})
        if r[mi] in WANT and r[mi] not in d["m"]:
            d["m"][r[mi]] = f"{r[vi]} {r[ui]}".strip()
    raw = csv_rows(rep, "raw")
    rh = raw[0]
    stall = [i for i, n in enumerate(rh) if n.startswith("smsp__pcsamp_warps_issue_stalled_")
             and not n.endswith("not_issued")]
    pipes = {n: rh.index(n) for n in PIPES if n in rh}
    units = raw[1] if len(raw) > 1 else []
    for k, r in zip(sorted(launches, key=int), raw[2:]):
        d = launches[k]
        print(f"\n== launch {k}: {d['name']}")
        for w in WANT:
            if w in d["m"]:
                print(f"  {w:36s} {d['m'][w]}")
        for n, i in pipes.items():
            print(f"  {n:36s} {r[i]} {units[i] if i < len(units) else ''}")
        top = sorted(((float(r[i].replace(',', '') or 0), rh[i].replace("smsp__pcsamp_warps_issue_stalled_", ""))
                      for i in stall), reverse=True)[:6]
        tot = sum(float(r[i].replace(',', '') or 0) for i in stall) or 1.0
        print("  top stall reasons (share of samples): " +
              ", ".join(f"{n} {100 * v / tot:.0f}%" for v, n in top))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
