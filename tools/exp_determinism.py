#!/usr/bin/env python3
"""Repeat the c2 projection (100M points, with and without the histogram,
exact and approx) and check every run is bit-identical to the first."""
import json, os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2005_03156_b200 import fastmap, synth
reps = int(os.environ.get("REPS", 20))
cfg = synth.config("c2")
soup = cfg.make_soup()
d = torch.from_numpy(cfg.make_points(100_000_000, soup=soup)).cuda()
res = {}
for name, params, mode in (("exact", fastmap.CoverParams(), fastmap.CoverMode.exact),
                           ("approx", fastmap.CoverParams(mode=fastmap.CoverMode.approx, epsilon=5e-3),
                            fastmap.CoverMode.approx)):
    idx = fastmap.build_index(soup, params, device=0)
    h0 = torch.zeros(soup.n_polys, dtype=torch.int64, device="cuda")
    ref = idx.project(d, hist=h0, mode=mode).clone()
    bad = 0
    for r in range(reps):
        h = torch.zeros_like(h0)
        out = idx.project(d, hist=h if r % 2 else None, mode=mode)
        bad += int(not torch.equal(out, ref)) + int(r % 2 == 1 and not torch.equal(h, h0))
    res[name] = {"reps": reps, "differing_runs": bad,
                 "hist_equals_bincount": bool(torch.equal(h0, torch.bincount(ref[ref >= 0].long(), minlength=soup.n_polys)))}
    idx.close()
print(json.dumps(res))
