#!/usr/bin/env python3
"""A/B of the exact query paths on one config: stream vs binned at several
tile sizes.  Points are generated on the GPU (synth_gpu.cu); each leg is
timed with CUDA events over `reps` calls after 2 warm-ups; answers of every
leg must equal the stream path's.

  python tools/exp_binned.py c3 1000000000 [tile_bytes ...]"""
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch

from paper_2005_03156_b200 import fastmap, synth

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 200_000_000
tiles = [float(x) for x in sys.argv[3:]] or [8e6, 32e6, 128e6]
reps = 3
cfg = synth.config(name)
soup = cfg.make_soup()
t0 = time.time()
idx = fastmap.build_index(soup, device=0)
print(json.dumps({"config": name, "n": n, "build_s": time.time() - t0}), flush=True)
pts = torch.empty((n, 2), dtype=torch.float64, device="cuda")
cfg.make_points_device(pts, soup=soup)
out = torch.empty(n, dtype=torch.int32, device="cuda")


def timed():
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


idx.set_query_path("stream")
ms = timed()
ref = out.clone()
print(json.dumps({"path": "stream", "ms": ms, "pts_per_s": n / ms * 1e3}), flush=True)
for tb in tiles:
    idx.set_query_path("binned", tb)
    plan = idx.query_plan(n)
    ms = timed()
    same = bool(torch.equal(out, ref))
    print(json.dumps({"path": "binned", "tile_bytes": tb, **plan, "ms": ms,
                      "pts_per_s": n / ms * 1e3, "equal_to_stream": same}), flush=True)
