#!/usr/bin/env python3
"""The reference CPU path's max_level sweep (the CLI's
--max-level, tools/fastmap.cpp:50, :349-353): for each cover level, the
reference's single-threaded build_cover + build_trie(F=4) time and size,
and query_leaves(exact) via run_chunked on all host threads and on one
thread, over a prefix of the config's stream (oracle/_ref, the unmodified
reference compiled here).  One JSON line per level; a level whose build
exceeds the time budget is reported and the sweep stops.

  python tools/ref_sweep.py CONFIG N_POINTS LEVEL [LEVEL ...]"""
import json
import os
import sys
import time

sys.path.insert(0, __file__.rsplit("/", 2)[0])
import numpy as np

import oracle
from paper_2005_03156_b200 import synth

name, n = sys.argv[1], int(float(sys.argv[2]))
levels = [int(x) for x in sys.argv[3:]]
cfg = synth.config(name)
soup = cfg.make_soup()
pts = cfg.make_points(n, soup=soup)
cores = os.cpu_count() or 1
m = oracle.RefModel(soup)
want = oracle.assign(soup, pts[:200_000])
for lv in levels:
    t0 = time.time()
    bi = m.build_index(lv, 4)
    ids, t = m.query_leaves(pts, threads=cores)
    n1 = min(n, 2_000_000)
    _, t1 = m.query_leaves(pts[:n1], threads=1, want_ids=False)
    line = {"config": name, "max_level": lv, "build_s": round(bi["seconds"], 2), "cover_entries": bi["entries"],
            "index_bytes": bi["bytes"], "points": n, "threads": cores,
            "points_per_s": n / t["seconds"], "one_thread_points_per_s": n1 / t1["seconds"],
            "pip_evals_per_point": t["pip_point_evaluations"] / n,
            "equals_exhaustive_on_first_200k": bool(np.array_equal(ids[:200_000], want))}
    print(json.dumps(line), flush=True)
    if time.time() - t0 > 400:
        print(json.dumps({"config": name, "stopped_after_level": lv, "why": "build + query over 400 s"}), flush=True)
        break
