import sys
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2005_03156_b200 import fastmap, synth
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "c2")
soup = cfg.make_soup()
n = int(float(sys.argv[2])) if len(sys.argv) > 2 else 3_000_000
pts = cfg.make_points(n, soup=soup)
idx = fastmap.build_index(soup, device=0)
print(idx.stats()["nx"], idx.stats()["query_block_log2"], idx.query_plan(n))
idx.set_query_path("binned")
d = torch.from_numpy(pts).cuda()
out = idx.project(d)
torch.cuda.synchronize()
print("ok", out[:5])
