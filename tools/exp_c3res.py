#!/usr/bin/env python3
"""Grid-resolution sweep on one config: for each cells_per_polygon value,
build the index (timed), print its statistics, time the stream and binned
query paths over n device-generated points (CUDA events, 3 calls after 2
warm-ups) and check every answer against the first resolution's (the ids
must not depend on the index resolution).

  python tools/exp_c3res.py c3 1e9 0 6.5 9.3      (0 = the default plan)"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch

from paper_2005_03156_b200 import fastmap, synth

name = sys.argv[1]
n = int(float(sys.argv[2]))
ms_list = [float(x) for x in sys.argv[3:]] or [0.0]
tiles = [float(x) for x in __import__("os").environ.get("EXP_TILES", "32e6 128e6").split()]
reps = 3
cfg = synth.config(name)
soup = cfg.make_soup()
pts = torch.empty((n, 2), dtype=torch.float64, device="cuda")
cfg.make_points_device(pts, soup=soup)
out = torch.empty(n, dtype=torch.int32, device="cuda")
ref = None


def timed(idx):
    for _ in range(2):
        idx.project(pts, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        idx.project(pts, out=out)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for m in ms_list:
    t0 = time.time()
    idx = fastmap.build_index(soup, fastmap.CoverParams(cells_per_polygon=m), device=0)
    build_s = time.time() - t0
    st = idx.stats()
    c = torch.zeros(4, dtype=torch.int64, device="cuda")
    k = min(n, 100_000_000)
    idx.project(pts[:k], out=out[:k], counters=c)
    c = c.cpu().tolist()
    print(json.dumps({"m": m, "build_s": round(build_s, 1), "nx": st["nx"], "ny": st["ny"],
                      "cells_M": st["nx"] * st["ny"] / 1e6,
                      "boundary_cell_frac": st["cells_boundary"] / (st["nx"] * st["ny"]),
                      "split": st["cells_split"], "slots_phase1": st["slots_phase1"],
                      "slots_total": st["slots_total"], "arena_GB": st["arena_bytes"] / 1e9,
                      "grid_GB": st["grid_bytes"] / 1e9,
                      "boundary_pt_frac": c[1] / c[0], "cands_per_bpt": c[2] / max(1, c[1]),
                      "edges_per_bpt": c[3] / max(1, c[1])}), flush=True)
    idx.set_query_path("stream")
    ms = timed(idx)
    if ref is None:
        ref = out.clone()
    print(json.dumps({"m": m, "path": "stream", "ms": ms, "pts_per_s": n / ms * 1e3,
                      "equal_to_first": bool(torch.equal(out, ref))}), flush=True)
    for tb in tiles:
        idx.set_query_path("binned", tb)
        plan = idx.query_plan(n)
        ms = timed(idx)
        print(json.dumps({"m": m, "path": "binned", "tile_bytes": tb, **plan, "ms": ms,
                          "pts_per_s": n / ms * 1e3, "equal_to_first": bool(torch.equal(out, ref))}),
              flush=True)
    idx.close()
    del idx
    torch.cuda.empty_cache()
