#!/usr/bin/env python3
"""Simple engine on c3s (20M device-resident points): time per call with
and without the reference's AssignCounters (counting runs scan candidates)."""
import json, os, sys, tempfile, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2005_03156_b200 import fastmap, synth
cfg = synth.config("c3s")
p = tempfile.mktemp(suffix=".fmcb")
cfg.write_fmcb(p)
eng = fastmap.SimpleEngine(fastmap.load_hierarchy(p))
os.unlink(p)
d = torch.from_numpy(cfg.make_points(20_000_000)).cuda()
res = {}
for mode in (fastmap.AssignMode.relaxed, fastmap.AssignMode.strict):
    for counters in (False, True):
        eng.assign(d, mode, counters=counters)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(3):
            eng.assign(d, mode, counters=counters)
        torch.cuda.synchronize()
        res[f"{mode.name}_counters_{counters}_ms_per_20M"] = (time.perf_counter() - t) / 3 * 1e3
print(json.dumps(res))
