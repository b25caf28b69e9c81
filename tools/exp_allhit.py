#!/usr/bin/env python3
"""All-hit ceiling (GPU): 100M c2 points against a one-rectangle index --
every point's cell is a true hit, so fm_query is the pure point stream."""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2005_03156_b200 import fastmap, synth
N = int(os.environ.get("SWEEP_POINTS", 100_000_000))
pts = synth.config("c2").make_points(N)
d = torch.from_numpy(pts).cuda()
out = torch.empty(N, dtype=torch.int32, device="cuda")
box = synth.expanded_box()
rect = fastmap.Soup.from_rings([[[(box[0] - 1, box[2] - 1), (box[1] + 1, box[2] - 1),
                                  (box[1] + 1, box[3] + 1), (box[0] - 1, box[3] + 1)]]])
idx = fastmap.build_index(rect, device=0)
for _ in range(3):
    idx.project(d, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    idx.project(d, out=out)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"all_hit_ms": e0.elapsed_time(e1) / 5}))
