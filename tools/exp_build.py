#!/usr/bin/env python3
"""GPU vs host index build times; full-scale config 3 build + query on the GPU."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

import oracle
from paper_2005_03156_b200 import fastmap, synth

names = sys.argv[1:] or ["c2", "c4"]
for name in names:
    cfg = synth.config(name)
    t0 = time.time()
    soup = cfg.make_soup()
    gen_s = time.time() - t0
    row = {"config": name, "polys": soup.n_polys, "verts": soup.n_vertices, "gen_s": gen_s}
    t0 = time.time()
    idx = fastmap.build_index(soup, device=0)
    torch.cuda.synchronize()
    row["gpu_build_s"] = time.time() - t0
    st = idx.stats()
    row.update({k: st[k] for k in ("nx", "ny", "cells_boundary", "slots_phase1", "slots_total",
                                   "cells_split", "arena_bytes")})
    if name in ("c2", "c4", "c3mini") and os.environ.get("HOST_BUILD", "1") == "1":
        t0 = time.time()
        h = fastmap.build_index(soup, device=-1)
        row["host_build_s"] = time.time() - t0
        h.close()
    n = int(os.environ.get("QPOINTS", 100_000_000))
    pts = cfg.make_points(n, soup=soup) if name != "c4" else cfg.make_points(n, soup=soup)
    d = torch.from_numpy(pts).cuda()
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3):
        idx.project(d, out=out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        idx.project(d, out=out)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    row.update({"query_points": n, "query_ms": ms, "pts_per_s": n / ms * 1e3})
    chk = np.random.default_rng(1).choice(n, 20000, replace=False)
    got = out.cpu().numpy()[chk]
    want = oracle.assign(soup, pts[chk])
    row["mismatches_vs_oracle_20k"] = int((got != want).sum())
    print(json.dumps(row), flush=True)
    del d, out
    idx.close()
