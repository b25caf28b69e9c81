"""Test helper: write FMCB hierarchy files (the format of save_hierarchy,
hierarchy.hpp:102-202) from plain Python structures, so tests can build
adversarial hierarchies (overlapping bboxes, holes, file bboxes that differ
from the polygons) and check the product against the reference's own
load_hierarchy / assign on the very same bytes.

A node is a dict: {"rings": [[(lon, lat), ...], ...], "bbox": (x0, x1, y0,
y1) or None (= polygon bbox), "fp": int, "children": [...], "fips": str}.
"""
import struct

import numpy as np


def _bbox(rings):
    if not rings:
        return (0.0, 0.0, 0.0, 0.0)
    v = np.concatenate([np.asarray(r, dtype=np.float64).reshape(-1, 2) for r in rings])
    return (float(v[:, 0].min()), float(v[:, 0].max()), float(v[:, 1].min()), float(v[:, 1].max()))


def _node(out, node, depth):
    out += struct.pack("<q", int(node.get("fp", 0)))
    if depth == 2:
        f = node.get("fips", "000000000000").encode()
        assert len(f) == 12
        out += f
    bb = node.get("bbox") or _bbox(node["rings"])
    out += struct.pack("<4d", *bb)
    verts, starts = [], []
    for r in node["rings"]:
        starts.append(len(verts))
        verts.extend((float(x), float(y)) for x, y in r)
    out += struct.pack("<I", len(verts))
    for x, y in verts:
        out += struct.pack("<2d", x, y)
    out += struct.pack("<I", len(starts))
    for s in starts:
        out += struct.pack("<I", s)
    if depth < 2:
        ch = node.get("children", [])
        out += struct.pack("<I", len(ch))
        for c in ch:
            _node(out, c, depth + 1)


def write_fmcb(path, states):
    n_c = sum(len(s.get("children", [])) for s in states)
    n_b = sum(len(c.get("children", [])) for s in states for c in s.get("children", []))
    out = bytearray(b"FMCB" + struct.pack("<H", 1) + struct.pack("<3Q", len(states), n_c, n_b))
    for s in states:
        _node(out, s, 0)
    with open(path, "wb") as f:
        f.write(bytes(out))


def star(rng, cx, cy, r0, r1, n):
    a = np.sort(rng.random(n)) * 2 * np.pi
    r = r0 + (r1 - r0) * rng.random(n)
    return list(zip(cx + r * np.cos(a), cy + r * np.sin(a)))


def random_hierarchy(seed, n_states=3, n_counties=3, n_blocks=4, spread=1.0):
    """Overlapping star-shaped regions at every level (bboxes overlap heavily,
    polygons overlap sometimes); every 5th block gets a hole, every 7th a
    file bbox larger than its polygon."""
    rng = np.random.default_rng(seed)
    states, k = [], 0
    for s in range(n_states):
        sx, sy = rng.uniform(0, 4 * spread), rng.uniform(0, 3 * spread)
        counties = []
        for c in range(n_counties):
            cx, cy = sx + rng.normal(0, 0.6 * spread), sy + rng.normal(0, 0.6 * spread)
            blocks = []
            for b in range(n_blocks):
                bx, by = cx + rng.normal(0, 0.3 * spread), cy + rng.normal(0, 0.3 * spread)
                rings = [star(rng, bx, by, 0.1 * spread, 0.5 * spread, int(rng.integers(3, 12)))]
                if k % 5 == 0:
                    rings.append(star(rng, bx, by, 0.02 * spread, 0.06 * spread, 5))
                bb = None
                if k % 7 == 3:
                    x0, x1, y0, y1 = _bbox(rings)
                    bb = (x0 - 0.2, x1 + 0.1, y0 - 0.1, y1 + 0.3)
                blocks.append({"rings": rings, "bbox": bb, "fp": b,
                               "fips": f"{s:02d}{c:03d}{b:06d}1"})
                k += 1
            counties.append({"rings": [star(rng, cx, cy, 0.4 * spread, 1.0 * spread, 16)],
                             "fp": c, "children": blocks})
        states.append({"rings": [star(rng, sx, sy, 0.8 * spread, 1.8 * spread, 24)],
                       "fp": s, "children": counties})
    return states


def two_triangles():
    """test_simple_mapper.cpp:104-142: two triangular states whose bboxes
    overlap around a notch neither covers; one county and block each."""
    def state(fp, ring):
        blk = {"rings": [ring], "fp": fp, "fips": f"{fp:02d}0010000011"}
        return {"rings": [ring], "fp": fp,
                "children": [{"rings": [ring], "fp": fp, "children": [blk]}]}
    return [state(1, [(0, 0), (2, 0), (0, 2)]), state(2, [(1, 3), (3, 1), (3, 3)])]
