#!/usr/bin/env python3
"""One profiles/ text summary of an .ncu-rep (--set full): the one-line launch summary of
tools/ncu_summary.py, the speed-of-light / occupancy lines of the details page, and the share of
each warp-stall reason among the PC samples.
Usage: python tools/ncu_report.py rep.ncu-rep > profiles/<name>.txt"""
import csv
import io
import os
import subprocess
import sys

KEEP = ("Memory Throughput", "DRAM Throughput", "Duration", "Executed Ipc", "Issue Slots Busy",
        "Mem Busy", "Max Bandwidth", "L1/TEX Hit Rate", "L2 Hit Rate", "Block Size", "Grid Size",
        "Registers Per Thread", "Driver Shared Memory", "Dynamic Shared Memory", "Static Shared Memory", "Block Limit", "Theoretical Occupancy",
        "Achieved Occupancy")
STALL = "smsp__pcsamp_warps_issue_stalled_"


def main(rep):
    here = os.path.dirname(os.path.abspath(__file__))
    print(subprocess.run([sys.executable, os.path.join(here, "ncu_summary.py"), rep], capture_output=True,
                         text=True).stdout.rstrip())
    print()
    det = subprocess.run(["ncu", "-i", rep, "--page", "details"], capture_output=True, text=True).stdout
    for line in det.splitlines():
        if any(line.strip().startswith(k) for k in KEEP):
            print(line.rstrip())
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    hdr, vals = r[0], r[2]
    st = {}
    for h, v in zip(hdr, vals):
        if h.startswith(STALL) and not h.endswith("_not_issued"):
            try:
                st[h[len(STALL):]] = float(v.replace(",", ""))
            except ValueError:
                pass
    tot = sum(st.values())
    if tot > 0:
        print()
        print("warp stall samples (share):")
        for k, v in sorted(st.items(), key=lambda kv: -kv[1]):
            if v / tot >= 0.005:
                print(f"{k:<30s} {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
