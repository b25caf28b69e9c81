#!/usr/bin/env python3
"""CPU analysis of the query-side access pattern of an exact index (no GPU):
builds the host-only index for a config, locates a point sample the way the
kernel does, and reports per-point lookup levels, slot kinds and the distinct
bytes touched (working sets).  Usage: python tools/exp_access.py [c2] [n]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import numpy as np

from paper_2005_03156_b200 import fastmap, synth

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4_000_000
cfg = synth.config(name)
soup = cfg.make_soup()
M = float(sys.argv[3]) if len(sys.argv) > 3 else 0.0
idx = fastmap.build_index(soup, fastmap.CoverParams(cells_per_polygon=M), device=-1)
grid, arena, g = idx.export()
pts = cfg.make_points(n, soup=soup)
nx, ny = g["nx"], g["ny"]
ix = np.clip(((pts[:, 0] - g["gx0"]) * g["inv_w"]).astype(np.int64), 0, nx - 1)
iy = np.clip(((pts[:, 1] - g["gy0"]) * g["inv_h"]).astype(np.int64), 0, ny - 1)
inside = (pts[:, 0] >= g["gx0"]) & (pts[:, 0] <= g["gx1"]) & (pts[:, 1] >= g["gy0"]) & (pts[:, 1] <= g["gy1"])
cell = iy * nx + ix
e = np.where(inside, grid[cell], 0xFFFFFFFF).astype(np.uint64)
rec = (e >= 0x80000000) & (e != 0xFFFFFFFF)
half = rec & ((e & 0x40000000) != 0)
k = (e & 0x3FFFFFFF).astype(np.int64)
kind = np.zeros(n, dtype=np.uint8)
kind[rec] = arena[k[rec] * 128]
res = {"config": name, "n": n, "nx": nx, "ny": ny, "boundary_frac": float(rec.mean()),
       "half_frac_of_boundary": float(half.sum() / max(1, rec.sum())),
       "kind_leaf": float((kind == 1).sum() / max(1, rec.sum())),
       "kind_split": float((kind == 3).sum() / max(1, rec.sum())),
       "kind_overflow": float((kind == 2).sum() / max(1, rec.sum()))}
# leaf-slot header stats for the boundary points
hdr = arena[(k[rec] * 128)[:, None] + np.arange(4)[None, :]]
lf = hdr[:, 0] == 1
res["nv_hist"] = np.bincount(hdr[lf, 1], minlength=6).tolist()
res["nc_hist"] = np.bincount(hdr[lf, 2], minlength=5).tolist()
res["nb_hist"] = np.bincount(hdr[lf, 3], minlength=3).tolist()
# fold ls=2: non-uniform blocks
for ls in (1, 2, 3):
    S = 1 << ls
    bnx, bny = (nx + S - 1) // S, (ny + S - 1) // S
    gp = np.full((bny * S, bnx * S), 0xFFFFFFFF, dtype=np.uint32)
    gp[:ny, :nx] = grid.reshape(ny, nx)
    b = gp.reshape(bny, S, bnx, S).transpose(0, 2, 1, 3).reshape(bny, bnx, S * S)
    uni = (b == b[:, :, :1]).all(axis=2)
    blk = (iy >> ls) * bnx + (ix >> ls)
    nonuni_pt = inside & ~uni.reshape(-1)[blk]
    touched = np.unique(blk[nonuni_pt])
    res[f"ls{ls}"] = {"blocks_MB": bnx * bny * 4 / 1e6, "nonuniform_blocks": float((~uni).mean()),
                      "pts_needing_level2": float(nonuni_pt.mean()),
                      "distinct_level2_touched": int(touched.size),
                      "level2_touched_MB_at_32B": touched.size * 32 / 1e6}
# distinct slots touched (working set), and how it grows with the sample
ks = np.unique(k[rec])
res["distinct_slots_touched"] = int(ks.size)
res["slot_touch_MB_128B"] = ks.size * 128 / 1e6
for frac in (0.25, 0.5):
    m = int(n * frac)
    res[f"distinct_slots_first_{frac}"] = int(np.unique(k[:m][rec[:m]]).size)
cells = np.unique(cell[inside])
res["distinct_cells_touched"] = int(cells.size)
print(json.dumps(res, indent=1))

# quick-record feasibility: leaf slots of boundary points, cell-local vertex range
def f64(off):
    b = arena[(k[rec][lf] * 128)[:, None] + off + np.arange(8)[None, :]]
    return b.copy().view(np.float64).reshape(-1)
nvv = hdr[lf, 1].astype(np.int64)
ncc = hdr[lf, 2].astype(np.int64)
nbb = hdr[lf, 3].astype(np.int64)
cx0 = g["gx0"] + ix[rec][lf] * g["w"]
cy0 = g["gy0"] + iy[rec][lf] * g["h"]
offs = [16, 32, 48, 96, 112]
ext = np.zeros(lf.sum())
for j, o in enumerate(offs):
    vx, vy = f64(o), f64(o + 8)
    u, v = (vx - cx0) / g["w"], (vy - cy0) / g["h"]
    m = (nvv > j) & ~((j == 2) & (nvv < 3))
    ext = np.maximum(ext, np.where(m, np.maximum(np.maximum(-u, u - 1), np.maximum(-v, v - 1)), 0))
res2 = {"vertex_outside_cell_max": float(ext.max()),
        "frac_ext_le_1": float((ext <= 1).mean()), "frac_ext_le_3": float((ext <= 3).mean()),
        "fit_nc2_nv5_nb2": float(((ncc <= 2) & (nvv <= 5) & (nbb <= 2)).mean()),
        "fit_nc2_nv4_nb1": float(((ncc <= 2) & (nvv <= 4) & (nbb <= 1)).mean()),
        "fit_nc4_nv5_nb2": float(((ncc <= 4) & (nvv <= 5) & (nbb <= 2)).mean())}
print(json.dumps(res2, indent=1))
