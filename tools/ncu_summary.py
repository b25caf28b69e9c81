#!/usr/bin/env python3
"""Summarise an .ncu-rep (details page) into the key lines we track."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Avg. Active Threads Per Warp", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Executed Instructions", "Issue Slots Busy", "Compute (SM) Throughput",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Limit Registers",
        "Block Limit Shared Mem", "Branch Efficiency"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    r = csv.DictReader(io.StringIO(out))
    seen = {}
    for row in r:
        k = row.get("Metric Name", "")
        if k in KEYS and k not in seen:
            seen[k] = f"{row.get('Metric Value')} {row.get('Metric Unit')}"
    for k in KEYS:
        if k in seen:
            print(f"{k:40s} {seen[k]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout.splitlines()
    if len(raw) >= 3:
        hdr = next(csv.reader([raw[0]]))
        units = next(csv.reader([raw[1]]))
        vals = next(csv.reader([raw[2]]))
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                     "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"):
            if name in hdr:
                i = hdr.index(name)
                print(f"{name:40s} {vals[i]} {units[i]}")


if __name__ == "__main__":
    main(sys.argv[1])
