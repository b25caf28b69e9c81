#!/usr/bin/env python3
"""GPU debug: c1 (2M points) projected repeatedly; determinism across runs
and mismatches against the oracle, with per-point diagnostics."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np, torch
import oracle
from paper_2005_03156_b200 import fastmap, synth
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 2_000_000
cfg = synth.config(name)
soup = cfg.make_soup()
pts = cfg.make_points(n, soup=soup)
want = oracle.assign(soup, pts)
idx = fastmap.build_index(soup, device=0)
d = torch.from_numpy(pts).cuda()
outs = [idx.project(d).cpu().numpy() for _ in range(3)]
host = idx.project(pts)
for k, o in enumerate(outs + [host]):
    bad = np.flatnonzero(o != want)
    print("run", k, "mismatches", bad.size, "first", bad[:8].tolist(), "got", o[bad[:8]].tolist(),
          "want", want[bad[:8]].tolist(), flush=True)
print("run0 vs run1 differ", int((outs[0] != outs[1]).sum()))
grid, arena, g = idx.export()
bad = np.flatnonzero(outs[0] != want)[:20]
for i in bad.tolist():
    px, py = pts[i]
    fx, fy = (px - g["gx0"]) * g["inv_w"], (py - g["gy0"]) * g["inv_h"]
    e = int(grid[int(fy) * g["nx"] + int(fx)])
    print(i, px, py, "cell", int(fx), int(fy), "entry", hex(e), "got", outs[0][i], "want", want[i], "nbr", outs[0][max(0,i-2):i+3].tolist(), want[max(0,i-2):i+3].tolist())
