#!/usr/bin/env python3
"""A/B of product-library build variants on ONE index: the index is built
once by the default library, then every variant library (ctypes-loaded
side by side; same source, so the same fm_index layout) runs fm_query on
the same handle and points.  Timed with CUDA events (3 calls after 2
warm-ups); every variant's answers must equal the default's.

  python tools/exp_variants.py CONFIG N PATH TILE_BYTES LIB [LIB ...]
  (PATH: stream | binned; LIB: paths of _lib/var/*.so)"""
import ctypes as C
import json
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import torch

from paper_2005_03156_b200 import _native as N
from paper_2005_03156_b200 import fastmap, synth

import os
name, n, path, tb = sys.argv[1], int(float(sys.argv[2])), sys.argv[3], float(sys.argv[4])
libs = sys.argv[5:]
with_hist = os.environ.get("EXPV_HIST", "0") == "1"  # also build the per-block histogram
cfg = synth.config(name)
soup = cfg.make_soup()
t0 = time.time()
idx = fastmap.build_index(soup, fastmap.CoverParams(cells_per_polygon=float(os.environ.get("EXPV_M", "0"))), device=0)
print(json.dumps({"config": name, "n": n, "build_s": time.time() - t0}), flush=True)
pts = torch.empty((n, 2), dtype=torch.float64, device="cuda")
cfg.make_points_device(pts, soup=soup)
out = torch.empty(n, dtype=torch.int32, device="cuda")
hist = torch.zeros(soup.n_polys, dtype=torch.int64, device="cuda") if with_hist else None
code = {"stream": N.PATH_STREAM, "binned": N.PATH_BINNED}[path]


def run(L, reps=3):
    L.fm_index_set_query_path.argtypes = [C.c_void_p, C.c_int, C.c_double]
    L.fm_query_mode.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p,
                                C.c_void_p, C.c_void_p, C.c_void_p]
    assert L.fm_index_set_query_path(idx.handle, code, tb) == 0
    s = torch.cuda.current_stream().cuda_stream

    def q():
        assert L.fm_query_mode(idx.handle, 0, pts.data_ptr(), n, out.data_ptr(),
                               hist.data_ptr() if hist is not None else None, None, s) == 0
    for _ in range(2):
        q()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        q()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


base = N.lib()
ms = run(base)
ref = out.clone()
print(json.dumps({"lib": "default", "path": path, "hist": with_hist, "ms": ms}), flush=True)
for lp in libs:
    L = C.CDLL(lp, mode=C.RTLD_LOCAL)
    ms = run(L)
    print(json.dumps({"lib": lp.split("/")[-1], "path": path, "ms": ms,
                      "equal": bool(torch.equal(out, ref))}), flush=True)
for _ in range(1):  # default again (box drift)
    print(json.dumps({"lib": "default(again)", "path": path, "ms": run(base)}), flush=True)
