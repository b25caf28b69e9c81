#!/usr/bin/env python3
"""Per-source-line instructions executed and warp-stall samples of one kernel
in an ncu report:  python tools/ncu_lines.py REPORT.ncu-rep KERNEL_REGEX [N]"""
import csv
import io
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kre}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
cur, hdr, out = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0] or len(r) < len(hdr) - 2:
        continue
    ie = hdr.index("Instructions Executed")
    ws = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        n = float(r[ie].replace(",", "") or 0)
        w = float(r[ws].replace(",", "") or 0)
    except ValueError:
        continue
    out.append((n, w, cur, r[0], r[1].strip()[:70]))
tn = sum(o[0] for o in out) or 1
tw = sum(o[1] for o in out) or 1
print(f"instructions {tn:.4g}  stall samples {tw:.4g}")
for n, w, f, l, s in sorted(out, key=lambda o: -(o[0] / tn + o[1] / tw))[:top]:
    print(f"inst {n / tn * 100:5.1f}%  stall {w / tw * 100:5.1f}%  {f}:{l}  {s}")
