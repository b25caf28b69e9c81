"""Test helper: evaluate the exported cell index on the CPU.

This re-implements the query kernel's record walk (paper_2005_03156_b200/
csrc/query.cuh) in Python so the index BUILDER can be checked against the
oracle on a machine without a GPU.  It is test code only; the product has
no CPU query path.
"""
from __future__ import annotations

import struct

import numpy as np

K_EMPTY = 0xFFFFFFFF
K_RECORD = 0x80000000


def _cross(px, py, lx, ly, hx, hy) -> bool:
    # geometry.hpp:170-174; Python floats are IEEE doubles, no contraction
    return (hx - lx) * (py - ly) - (hy - ly) * (px - lx) > 0.0


def locate(g: dict, grid: np.ndarray, pts: np.ndarray) -> np.ndarray:
    px, py = pts[:, 0], pts[:, 1]
    ax0, ax1 = max(g["gx0"], -180.0), min(g["gx1"], 180.0)
    ay0, ay1 = max(g["gy0"], -90.0), min(g["gy1"], 90.0)
    with np.errstate(invalid="ignore"):
        inside = (px >= ax0) & (px <= ax1) & (py >= ay0) & (py <= ay1)
        tx = np.where(inside, (px - g["gx0"]) * g["inv_w"], 0.0)
        ty = np.where(inside, (py - g["gy0"]) * g["inv_h"], 0.0)
    ix = np.clip(tx.astype(np.int64), 0, g["nx"] - 1)
    iy = np.clip(ty.astype(np.int64), 0, g["ny"] - 1)
    e = grid[iy * g["nx"] + ix]
    return np.where(inside, e, np.uint32(K_EMPTY)).astype(np.uint32)


def parse_record(arena: np.ndarray, entry: int):
    off = (entry & ~K_RECORD) * 16
    buf = arena.data
    n_edges, n_cands, n_words, n_breaks = struct.unpack_from("<4H", buf, off)
    edges = np.frombuffer(buf, dtype="<f8", count=4 * n_edges, offset=off + 16).reshape(-1, 4)
    co = off + 16 + 32 * n_edges
    cands = np.frombuffer(buf, dtype="<i4", count=2 * n_cands, offset=co).reshape(-1, 2)
    mo = co + 8 * n_cands
    masks = np.frombuffer(buf, dtype="<u4", count=n_cands * n_words, offset=mo).reshape(n_cands, n_words) \
        if n_words else np.zeros((n_cands, 0), dtype=np.uint32)
    bo = (mo + 4 * n_cands * n_words + 7) & ~7
    breaks = np.frombuffer(buf, dtype="<f8", count=n_breaks, offset=bo)
    return edges, cands, masks, breaks


def resolve(arena: np.ndarray, entry: int, px: float, py: float) -> int:
    edges, cands, masks, breaks = parse_record(arena, entry)
    bits = []
    for lx, ly, hx, hy in edges.tolist():
        bits.append(1 if (ly < py <= hy and _cross(px, py, lx, ly, hx, hy)) else 0)
    boff = 0
    for c in range(cands.shape[0]):
        leaf, info = int(cands[c, 0]), int(cands[c, 1]) & 0xFFFFFFFF
        nb = info >> 1
        par = info & 1
        for w in range(masks.shape[1]):
            m = int(masks[c, w])
            while m:
                k = (m & -m).bit_length() - 1
                m &= m - 1
                par ^= bits[w * 32 + k]
        for b in breaks[boff:boff + nb].tolist():
            par ^= 1 if py > b else 0
        boff += nb
        if par & 1:
            return leaf
    return -1


def walk(index_export, pts: np.ndarray) -> np.ndarray:
    grid, arena, g = index_export
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    e = locate(g, grid, pts)
    out = np.where(e < K_RECORD, e.astype(np.int64), -1).astype(np.int32)
    rec = np.nonzero((e >= K_RECORD) & (e != K_EMPTY))[0]
    for i in rec.tolist():
        out[i] = resolve(arena, int(e[i]), float(pts[i, 0]), float(pts[i, 1]))
    return out
