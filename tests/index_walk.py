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
K_HALF = 0x40000000      # slot content fits its first 64 bytes
K_DOUBLE = 0x20000000    # double slot (kind 4)
K_INDEX = 0x1FFFFFFF


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


def _align(v, a):
    return (v + a - 1) & ~(a - 1)


SLOT = 128


def leaf_half(nv, nc, nb) -> bool:
    return nc <= 2 and ((nv <= 2 and nb <= 1) or (nv == 3 and nb == 0))


def _eval_leaf_slot(arena, off, px, py) -> int:
    buf = arena.data
    nv, nc, nb = int(arena[off + 1]), int(arena[off + 2]), int(arena[off + 3])
    chain = 1 if nv <= 3 else struct.unpack_from("<I", buf, off + 64)[0]
    ids = struct.unpack_from("<2i", buf, off + 8) + struct.unpack_from("<2i", buf, off + 72)
    masks = arena[off + 4: off + 6].tolist() + arena[off + 68: off + 70].tolist()
    infos = arena[off + 6: off + 8].tolist() + arena[off + 70: off + 72].tolist()
    if nv >= 3:
        breaks = struct.unpack_from("<2d", buf, off + 80)
    else:
        breaks = struct.unpack_from("<d", buf, off + 48) + struct.unpack_from("<d", buf, off + 80)
    v = (np.frombuffer(buf, dtype="<f8", count=6, offset=off + 16).reshape(3, 2).tolist()
         + np.frombuffer(buf, dtype="<f8", count=4, offset=off + 96).reshape(2, 2).tolist())
    m = 0
    for k in range(4):
        if k + 1 < nv and not (chain >> (k + 1)) & 1:
            (ax, ay), (bx, by) = v[k], v[k + 1]
            lx, ly, hx, hy = (ax, ay, bx, by) if ay < by else (bx, by, ax, ay)
            if ly < py <= hy and _cross(px, py, lx, ly, hx, hy):
                m |= 1 << k
    bm = (1 if (nb > 0 and py > breaks[0]) else 0) | (2 if (nb > 1 and py > breaks[1]) else 0)
    for c in range(nc):
        par = (infos[c] >> 7) ^ bin(m & masks[c]).count("1") ^ bin(bm & infos[c] & 3).count("1")
        if par & 1:
            return ids[c]
    return -1


def _eval_double_slot(arena, off, px, py) -> int:
    """kind 4 (index_format.h): 256 bytes, <= 8 candidates, <= 4 breaks, <= 10 vertices."""
    buf = arena.data
    nv, nc, nb = int(arena[off + 1]), int(arena[off + 2]), int(arena[off + 3])
    chain = struct.unpack_from("<I", buf, off + 4)[0]
    ids = struct.unpack_from("<8i", buf, off + 8)
    masks = struct.unpack_from("<8H", buf, off + 40)
    infos = arena[off + 56: off + 64].tolist()
    breaks = struct.unpack_from("<4d", buf, off + 64)
    v = np.frombuffer(buf, dtype="<f8", count=20, offset=off + 96).reshape(10, 2).tolist()
    m = 0
    for k in range(9):
        if k + 1 < nv and not (chain >> (k + 1)) & 1:
            (ax, ay), (bx, by) = v[k], v[k + 1]
            lx, ly, hx, hy = (ax, ay, bx, by) if ay < by else (bx, by, ax, ay)
            if ly < py <= hy and _cross(px, py, lx, ly, hx, hy):
                m |= 1 << k
    bm = 0
    for j in range(nb):
        if py > breaks[j]:
            bm |= 1 << j
    for c in range(nc):
        par = (infos[c] >> 7) ^ bin(m & masks[c]).count("1") ^ bin(bm & infos[c] & 15).count("1")
        if par & 1:
            return ids[c]
    return -1


def _eval_overflow(arena, off, px, py) -> int:
    buf = arena.data
    kind = arena[off]
    if kind == 1:  # compact
        nv, nc, nb = int(arena[off + 1]), int(arena[off + 2]), int(arena[off + 3])
        chain = struct.unpack_from("<I", buf, off + 4)[0]
        cands = np.frombuffer(buf, dtype="<u4", count=2 * nc, offset=off + 8).reshape(-1, 2)
        info = arena[off + 8 + 8 * nc: off + 8 + 9 * nc]
        bo = _align(8 + 9 * nc, 8)
        breaks = np.frombuffer(buf, dtype="<f8", count=nb, offset=off + bo)
        vo = _align(bo + 8 * nb, 16)
        v = np.frombuffer(buf, dtype="<f8", count=2 * nv, offset=off + vo).reshape(-1, 2).tolist()
        m = 0
        for i in range(nv - 1):
            if (chain >> (i + 1)) & 1:
                continue
            (ax, ay), (bx, by) = v[i], v[i + 1]
            lx, ly, hx, hy = (ax, ay, bx, by) if ay < by else (bx, by, ax, ay)
            if ly < py <= hy and _cross(px, py, lx, ly, hx, hy):
                m |= 1 << i
        bm = 0
        for j, b in enumerate(breaks.tolist()):
            if py > b:
                bm |= 1 << j
        for c in range(nc):
            leaf, mask = int(cands[c, 0]), int(cands[c, 1])
            inf = int(info[c])
            par = (inf >> 7) ^ bin(m & mask).count("1") ^ bin(bm & inf & 0x7F).count("1")
            if par & 1:
                return leaf - (1 << 32) if leaf >= (1 << 31) else leaf
        return -1
    assert kind == 2, f"bad overflow record kind {kind}"
    n_words, n_edges, n_cands, n_breaks = struct.unpack_from("<4H", buf, off + 2)
    edges = np.frombuffer(buf, dtype="<f8", count=4 * n_edges, offset=off + 16).reshape(-1, 4)
    co = off + 16 + 32 * n_edges
    cands = np.frombuffer(buf, dtype="<i4", count=2 * n_cands, offset=co).reshape(-1, 2)
    mo = co + 8 * n_cands
    masks = np.frombuffer(buf, dtype="<u4", count=n_cands * n_words, offset=mo).reshape(n_cands, n_words)
    bo = off + _align(mo - off + 4 * n_cands * n_words, 8)
    breaks = np.frombuffer(buf, dtype="<f8", count=n_breaks, offset=bo)
    bits = []
    for lx, ly, hx, hy in edges.tolist():
        bits.append(1 if (ly < py <= hy and _cross(px, py, lx, ly, hx, hy)) else 0)
    boff = 0
    for c in range(cands.shape[0]):
        leaf, info = int(cands[c, 0]), int(cands[c, 1]) & 0xFFFFFFFF
        nbc = info >> 1
        par = info & 1
        for w in range(masks.shape[1]):
            mm = int(masks[c, w])
            while mm:
                k = (mm & -mm).bit_length() - 1
                mm &= mm - 1
                par ^= bits[w * 32 + k]
        for b in breaks[boff:boff + nbc].tolist():
            par ^= 1 if py > b else 0
        boff += nbc
        if par & 1:
            return leaf
    return -1


def resolve(arena: np.ndarray, entry: int, px: float, py: float, slot_bytes: int) -> int:
    """Walk slot `entry` (index_format.h) for point (px, py)."""
    buf = arena.data
    e = entry
    while True:
        off = (e & K_INDEX) * SLOT
        kind = arena[off]
        half = kind in (2, 3) or (kind == 1 and leaf_half(*arena[off + 1: off + 4].tolist()))
        assert bool(e & K_HALF) == half, "half-slot flag disagrees with the slot"
        assert bool(e & K_DOUBLE) == (kind == 4), "double-slot flag disagrees with the slot"
        if half:  # the flag promises nothing past byte 64 is needed
            assert not arena[off + 64: off + SLOT].any()
        if kind == 1:
            return _eval_leaf_slot(arena, off, px, py)
        if kind == 4:
            return _eval_double_slot(arena, off, px, py)
        if kind == 2:
            ovf = struct.unpack_from("<Q", buf, off + 8)[0]
            return _eval_overflow(arena, slot_bytes + ovf, px, py)
        assert kind == 3, f"bad slot kind {kind}"
        x0, y0, ihw, ihh = struct.unpack_from("<4d", buf, off + 8)
        child = struct.unpack_from("<4I", buf, off + 40)
        i = min(max(int((px - x0) * ihw), 0), 1)
        j = min(max(int((py - y0) * ihh), 0), 1)
        e = child[2 * j + i]
        if e == K_EMPTY:
            return -1
        if e < K_RECORD:
            return e


def record_kinds(index_export) -> dict:
    grid, arena, g = index_export
    n_slots = g["slot_bytes"] // SLOT
    count = {"leaf": 0, "overflow": 0, "split": 0, "double": 0}
    names = {1: "leaf", 2: "overflow", 3: "split", 4: "double"}
    k = 0
    while k < n_slots:  # a double slot's second half is not a slot
        kind = int(arena[k * SLOT])
        count[names[kind]] += 1
        k += 2 if kind == 4 else 1
    return count


def walk(index_export, pts: np.ndarray) -> np.ndarray:
    grid, arena, g = index_export
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    e = locate(g, grid, pts)
    out = np.where(e < K_RECORD, e.astype(np.int64), -1).astype(np.int32)
    rec = np.nonzero((e >= K_RECORD) & (e != K_EMPTY))[0]
    for i in rec.tolist():
        out[i] = resolve(arena, int(e[i]), float(pts[i, 0]), float(pts[i, 1]), g["slot_bytes"])
    return out
