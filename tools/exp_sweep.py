#!/usr/bin/env python3
"""Tuning sweep (GPU): time fm_query on c2 for a library variant and index
resolutions, plus an all-hit index (streaming ceiling).  One JSON line per
case.  Usage: FASTMAP_B200_LIB=... python tools/exp_sweep.py [m ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

from paper_2005_03156_b200 import fastmap, synth

N = int(os.environ.get("SWEEP_POINTS", 100_000_000))
cfg = synth.config(os.environ.get("SWEEP_CONFIG", "c2"))
soup = cfg.make_soup()
pts = cfg.make_points(N, soup=soup)
d = torch.from_numpy(pts).cuda()
out = torch.empty(N, dtype=torch.int32, device="cuda")


def timeit(idx, reps=10):
    for _ in range(3):
        idx.project(d, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        idx.project(d, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


lib = os.environ.get("SWEEP_LIB_TAG") or os.path.basename(os.environ.get("FASTMAP_B200_LIB", "default"))
ms_list = [float(x) for x in sys.argv[1:]] or [0.0]
for m in ms_list:
    idx = fastmap.build_index(soup, fastmap.CoverParams(cells_per_polygon=m), device=0)
    st = idx.stats()
    ms = timeit(idx)
    c = torch.zeros(4, dtype=torch.int64, device="cuda")
    idx.project(d, out=out, counters=c)
    torch.cuda.synchronize()
    c = c.cpu().tolist()
    print(json.dumps({"lib": lib, "m": m, "nx": st["nx"], "ny": st["ny"], "ms": ms,
                      "pts_per_s": N / ms * 1e3, "grid_MB": st["grid_bytes"] / 1e6,
                      "arena_MB": st["arena_bytes"] / 1e6,
                      "query_grid_MB": st["query_grid_bytes"] / 1e6, "ls": st["query_block_log2"],
                      "boundary_frac": c[1] / N, "cands_per_bpt": c[2] / max(1, c[1]),
                      "edges_per_bpt": c[3] / max(1, c[1])}), flush=True)
    idx.close()
# streaming ceiling: one rectangle covering the whole point box -> all hits
box = synth.expanded_box()
rect = fastmap.Soup.from_rings([[[(box[0] - 1, box[2] - 1), (box[1] + 1, box[2] - 1),
                                  (box[1] + 1, box[3] + 1), (box[0] - 1, box[3] + 1)]]])
idx = fastmap.build_index(rect, device=0)
ms = timeit(idx)
print(json.dumps({"lib": lib, "case": "all_hit", "ms": ms, "pts_per_s": N / ms * 1e3,
                  "GBps_20B": 20 * N / ms / 1e6}), flush=True)
