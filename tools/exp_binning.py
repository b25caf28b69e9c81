#!/usr/bin/env python3
"""Point binning (north star item 2), measured: what sorting the c2 point
stream by cell would cost and what a cell-coherent query saves.

Legs (100M c2 points resident on the GPU, CUDA events, warm):
  query_random   fm_query on the stream as generated (the product path)
  key            cell key per point (block of 4x4 cells, row-major)
  sort           torch.sort of the 32-bit keys (CUB radix sort) -> permutation
  gather         points in key order (16 B random reads by permutation)
  query_sorted   fm_query on the key-ordered points
  scatter        answers back to input order (4 B random writes)
binned total = key + sort + gather + query_sorted + scatter."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np
import torch

from paper_2005_03156_b200 import _native as N
from paper_2005_03156_b200 import fastmap, synth

n = int(os.environ.get("SWEEP_POINTS", 100_000_000))
cfg = synth.config("c2")
soup = cfg.make_soup()
pts = torch.from_numpy(cfg.make_points(n, soup=soup)).cuda()
idx = fastmap.build_index(soup, device=0)
geo = np.zeros(16, dtype=np.float64)
gl, al = C.c_uint64(0), C.c_uint64(0)
N.check(N.lib().fm_index_export(idx.handle, None, C.byref(gl), None, C.byref(al), N.ptr(geo, C.c_double)))
gx0, gy0, inv_w, inv_h, nx, ny = geo[0], geo[2], geo[6], geo[7], int(geo[8]), int(geo[9])
bnx = (nx + 3) // 4
out = torch.empty(n, dtype=torch.int32, device="cuda")


def timed(fn, reps=5):
    for _ in range(2):
        r = fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        r = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, r


res = {}
res["query_random_ms"], _ = timed(lambda: idx.project(pts, out=out))


def keyf():
    ix = ((pts[:, 0] - gx0) * inv_w).clamp(0, nx - 1).to(torch.int32) >> 2
    iy = ((pts[:, 1] - gy0) * inv_h).clamp(0, ny - 1).to(torch.int32) >> 2
    return iy * bnx + ix


res["key_ms"], key = timed(keyf)
res["sort_ms"], (sk, perm) = timed(lambda: torch.sort(key))
res["gather_ms"], sp = timed(lambda: pts.index_select(0, perm))
sp = sp.contiguous()
out_s = torch.empty(n, dtype=torch.int32, device="cuda")
res["query_sorted_ms"], _ = timed(lambda: idx.project(sp, out=out_s))
back = torch.empty(n, dtype=torch.int32, device="cuda")
res["scatter_ms"], _ = timed(lambda: back.index_copy_(0, perm, out_s))
idx.project(pts, out=out)
torch.cuda.synchronize()
res["answers_equal"] = bool(torch.equal(back, out))
res["binned_total_ms"] = (res["key_ms"] + res["sort_ms"] + res["gather_ms"] + res["query_sorted_ms"]
                          + res["scatter_ms"])
print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in res.items()}))
