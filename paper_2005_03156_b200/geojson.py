"""GeoJSON ingestion of the three boundary levels.

Host-side mirror of the reference's ``geojson.hpp``: ``load_boundaries``
(geojson.hpp:154-271) reads the states / counties / blocks
FeatureCollections, wires children to parents by FIPS component match and
orders siblings by ascending fp code; ``ingest`` is the reference CLI's
``fastmap ingest`` (tools/fastmap.cpp:163-170): load, then write the FMCB
hierarchy file (``save_hierarchy``, hierarchy.hpp:187-198) that
:func:`paper_2005_03156_b200.fastmap.load_hierarchy` and the GPU index build
read.  ``write_boundaries`` is the reference's writer (geojson.hpp:322-353).

Expected feature properties (geojson.hpp:6-9):
  states:   STATEFP
  counties: STATEFP, COUNTYFP
  blocks:   STATE_FIPS, CNTY_FIPS, TRACT, BLKGRP, FIPS

Errors are raised as ``RuntimeError`` (the reference's ``std::runtime_error``)
with the reference's messages.  Parsing is host work (as in the reference);
the product's GPU path starts at the FMCB hierarchy.
"""
from __future__ import annotations

import json
import os
import re
import struct
import tempfile
from dataclasses import dataclass, field
from typing import List, Tuple

FIPS_LENGTH = 12  # kFipsLength, hierarchy.hpp
_INT64_MIN, _INT64_MAX = -(1 << 63), (1 << 63) - 1


@dataclass
class RegionNode:
    """hierarchy.hpp RegionNode: fp code, 12-char FIPS (leaves), file bbox
    (x_min, x_max, y_min, y_max), the polygon's nodes and ring starts
    (PolygonGeometry, geometry.hpp:64-87), children."""
    fp_code: int = 0
    fips12: str = ""
    bbox: Tuple[float, float, float, float] = (0.0, 0.0, 0.0, 0.0)
    nodes: List[Tuple[float, float]] = field(default_factory=list)
    ring_starts: List[int] = field(default_factory=list)
    children: List["RegionNode"] = field(default_factory=list)


@dataclass
class RegionHierarchy:
    states: List[RegionNode] = field(default_factory=list)

    def counts(self) -> Tuple[int, int, int]:  # compute_counts
        c = sum(len(s.children) for s in self.states)
        b = sum(len(k.children) for s in self.states for k in s.children)
        return len(self.states), c, b


# ---------------------------------------------------------------------------
# property and geometry parsing (geojson_detail, geojson.hpp:28-150)
# ---------------------------------------------------------------------------

def _is_int(v) -> bool:     # nlohmann is_number_integer (booleans are not numbers)
    return isinstance(v, int) and not isinstance(v, bool)


def _is_number(v) -> bool:  # nlohmann is_number
    return isinstance(v, (int, float)) and not isinstance(v, bool)


def _as_int64(v: int) -> int:  # get<std::int64_t>() of an unsigned wraps
    return ((v - _INT64_MIN) % (1 << 64)) + _INT64_MIN


_STOLL = re.compile(r"[ \t\n\v\f\r]*([+-]?[0-9]+)")


def _stoll(s: str) -> int:
    """std::stoll: leading whitespace, optional sign, decimal digits up to the
    first non-digit; raises ValueError for no digits or out of range."""
    m = _STOLL.match(s)
    if not m:
        raise ValueError("stoll: no conversion")
    v = int(m.group(1))
    if not (_INT64_MIN <= v <= _INT64_MAX):
        raise ValueError("stoll: out of range")
    return v


def _feature_name(path: str, index: int) -> str:
    return f"{path} feature #{index}"


def _parse_code(props, key: str, feature: str) -> int:
    if not isinstance(props, dict) or key not in props:
        raise RuntimeError(f"{feature}: missing property {key}")
    v = props[key]
    try:
        if isinstance(v, str):
            return _stoll(v)
        if _is_int(v):
            return _as_int64(v)
    except ValueError:
        pass
    raise RuntimeError(f"{feature}: property {key} is not a FIPS code")


def _parse_digits(props, key: str, feature: str) -> str:
    if not isinstance(props, dict) or key not in props:
        raise RuntimeError(f"{feature}: missing property {key}")
    v = props[key]
    if isinstance(v, str):
        return v
    if _is_int(v):
        return str(_as_int64(v))
    raise RuntimeError(f"{feature}: property {key} is not usable")


def _append_ring(node: RegionNode, ring, feature: str) -> None:
    if not isinstance(ring, list) or len(ring) < 3:
        raise RuntimeError(f"{feature}: ring with fewer than 3 positions")
    pts = []
    for pos in ring:
        if not isinstance(pos, list) or len(pos) < 2 or not _is_number(pos[0]) or not _is_number(pos[1]):
            raise RuntimeError(f"{feature}: malformed coordinate position")
        pts.append((float(pos[0]), float(pos[1])))
    if len(pts) >= 2 and pts[0] == pts[-1]:  # drop the repeated closing position
        pts.pop()
    if len(pts) < 3:
        raise RuntimeError(f"{feature}: degenerate ring after closing")
    node.ring_starts.append(len(node.nodes))  # PolygonGeometry::add_ring
    node.nodes.extend(pts)


def _parse_geometry(node: RegionNode, feat: dict, feature: str) -> None:
    g = feat.get("geometry")
    if g is None:
        raise RuntimeError(f"{feature}: missing geometry")
    gtype = g.get("type", "") if isinstance(g, dict) else ""
    coords = g.get("coordinates") if isinstance(g, dict) else None
    if not isinstance(coords, list):
        raise RuntimeError(f"{feature}: geometry has no coordinates")
    if gtype == "Polygon":
        for ring in coords:
            _append_ring(node, ring, feature)
    elif gtype == "MultiPolygon":
        for poly in coords:
            if not isinstance(poly, list):
                raise RuntimeError(f"{feature}: malformed MultiPolygon")
            for ring in poly:
                _append_ring(node, ring, feature)
    else:
        raise RuntimeError(f"{feature}: unsupported geometry type '{gtype}'")
    if not node.ring_starts:
        raise RuntimeError(f"{feature}: geometry has no rings")


def _parse_bbox(node: RegionNode, feat: dict) -> None:
    b = feat.get("bbox")
    if isinstance(b, list) and len(b) == 4:
        if not all(_is_number(x) for x in b):  # get<double>() of a non-number: json type_error
            raise TypeError("type must be number, but is " + next(type(x).__name__ for x in b
                                                                   if not _is_number(x)))
        box = (float(b[0]), float(b[2]), float(b[1]), float(b[3]))  # [x0, y0, x1, y1]
        if box[0] <= box[1] and box[2] <= box[3]:  # BBox::valid
            node.bbox = box
            return
    xs = [p[0] for p in node.nodes]
    ys = [p[1] for p in node.nodes]
    node.bbox = (min(xs), max(xs), min(ys), max(ys))  # polygon_bbox


def _features_of(doc, path: str) -> list:
    if (not isinstance(doc, dict) or doc.get("type", "") != "FeatureCollection"
            or not isinstance(doc.get("features"), list)):
        raise RuntimeError(f"{path}: not a GeoJSON FeatureCollection")
    feats = doc["features"]
    for i, f in enumerate(feats):
        if not isinstance(f, dict):
            raise RuntimeError(f"{_feature_name(path, i)}: not a Feature object")
    return feats


def _parse_file(path: str):
    try:
        with open(path, "r", encoding="utf-8") as fh:
            text = fh.read()
    except OSError:
        raise RuntimeError(f"cannot open boundary file: {path}") from None
    def _no_constant(name):  # NaN / Infinity are not JSON (nlohmann rejects them)
        raise ValueError(f"invalid literal {name}")
    try:
        return json.loads(text, parse_constant=_no_constant)
    except ValueError as e:
        raise RuntimeError(f"{path}: {e}") from None


def _props(feat: dict):
    return feat.get("properties", {})


# ---------------------------------------------------------------------------
# load_boundaries (geojson.hpp:154-271)
# ---------------------------------------------------------------------------

def load_boundaries(state_path: str, county_path: str, block_path: str) -> RegionHierarchy:
    """The three levels, children wired to parents by FIPS component match,
    siblings in ascending fp-code order (so the result does not depend on
    feature order)."""
    h = RegionHierarchy()
    state_by_fp = {}
    for i, feat in enumerate(_features_of(_parse_file(state_path), state_path)):
        name = _feature_name(state_path, i)
        node = RegionNode(fp_code=_parse_code(_props(feat), "STATEFP", name))
        _parse_geometry(node, feat, name)
        _parse_bbox(node, feat)
        if node.fp_code in state_by_fp:
            raise RuntimeError(f"{name}: duplicate STATEFP {node.fp_code}")
        state_by_fp[node.fp_code] = len(h.states)
        h.states.append(node)
    if not h.states:
        raise RuntimeError(f"{state_path}: no state features")

    county_by_fp = {}
    for i, feat in enumerate(_features_of(_parse_file(county_path), county_path)):
        name = _feature_name(county_path, i)
        props = _props(feat)
        state_fp = _parse_code(props, "STATEFP", name)
        node = RegionNode(fp_code=_parse_code(props, "COUNTYFP", name))
        _parse_geometry(node, feat, name)
        _parse_bbox(node, feat)
        si = state_by_fp.get(state_fp)
        if si is None:
            raise RuntimeError(f"{name}: references absent state {state_fp}")
        key = (state_fp, node.fp_code)
        if key in county_by_fp:
            raise RuntimeError(f"{name}: duplicate COUNTYFP {node.fp_code}")
        county_by_fp[key] = (si, len(h.states[si].children))
        h.states[si].children.append(node)

    seen_fips = set()
    n_blocks = 0
    for i, feat in enumerate(_features_of(_parse_file(block_path), block_path)):
        name = _feature_name(block_path, i)
        props = _props(feat)
        state_fp = _parse_code(props, "STATE_FIPS", name)
        county_fp = _parse_code(props, "CNTY_FIPS", name)
        tract = _parse_digits(props, "TRACT", name)
        blkgrp = _parse_digits(props, "BLKGRP", name)
        try:
            fp = _stoll(tract + blkgrp)
        except ValueError:
            raise RuntimeError(f"{name}: TRACT/BLKGRP are not digits") from None
        fips = _parse_digits(props, "FIPS", name)
        if len(fips.encode("utf-8")) != FIPS_LENGTH:
            raise RuntimeError(f"{name}: FIPS is not 12 characters")
        if fips in seen_fips:
            raise RuntimeError(f"{name}: duplicate FIPS {fips}")
        seen_fips.add(fips)
        node = RegionNode(fp_code=fp, fips12=fips)
        _parse_geometry(node, feat, name)
        _parse_bbox(node, feat)
        ci = county_by_fp.get((state_fp, county_fp))
        if ci is None:
            raise RuntimeError(f"{name}: references absent county {state_fp}/{county_fp}")
        h.states[ci[0]].children[ci[1]].children.append(node)
        n_blocks += 1
    if n_blocks == 0:
        raise RuntimeError(f"{block_path}: no block features (leaf level is mandatory)")

    key = lambda n: n.fp_code  # noqa: E731
    h.states.sort(key=key)
    for s in h.states:
        s.children.sort(key=key)
        for c in s.children:
            c.children.sort(key=key)
            for a, b in zip(c.children, c.children[1:]):
                if a.fp_code == b.fp_code:
                    raise RuntimeError(f"duplicate block code {b.fp_code} under county {c.fp_code}")
    return h


# ---------------------------------------------------------------------------
# FMCB writer (save_hierarchy, hierarchy.hpp:108-198) and ingest
# ---------------------------------------------------------------------------

def _write_node(out: bytearray, node: RegionNode, depth: int) -> None:
    out += struct.pack("<q", node.fp_code)
    if depth == 2:
        f = node.fips12.encode("utf-8")
        if len(f) != FIPS_LENGTH:
            raise RuntimeError("leaf node without a 12-character FIPS code")
        out += f
    out += struct.pack("<4d", *node.bbox)
    out += struct.pack("<I", len(node.nodes))
    for x, y in node.nodes:
        out += struct.pack("<2d", x, y)
    out += struct.pack("<I", len(node.ring_starts))
    for r in node.ring_starts:
        out += struct.pack("<I", r)
    if depth < 2:
        out += struct.pack("<I", len(node.children))
        for c in node.children:
            _write_node(out, c, depth + 1)


def fmcb_bytes(h: RegionHierarchy) -> bytes:
    out = bytearray(b"FMCB" + struct.pack("<H", 1) + struct.pack("<3Q", *h.counts()))
    for s in h.states:
        _write_node(out, s, 0)
    return bytes(out)


def save_hierarchy(h: RegionHierarchy, path: str) -> None:
    try:
        with open(path, "wb") as fh:
            fh.write(fmcb_bytes(h))
    except OSError:
        raise RuntimeError(f"cannot open for writing: {path}") from None


def ingest(state_path: str, county_path: str, block_path: str, out_fmcb: str) -> Tuple[int, int, int]:
    """``fastmap ingest`` (tools/fastmap.cpp:163-170): GeoJSON -> FMCB.
    Returns (states, counties, blocks)."""
    h = load_boundaries(state_path, county_path, block_path)
    save_hierarchy(h, out_fmcb)
    return h.counts()


def load_boundaries_hierarchy(state_path: str, county_path: str, block_path: str):
    """GeoJSON -> the product's :class:`~paper_2005_03156_b200.fastmap.Hierarchy`
    (through an FMCB image, the format the native loader reads)."""
    from .fastmap import load_hierarchy
    h = load_boundaries(state_path, county_path, block_path)
    fd, tmp = tempfile.mkstemp(suffix=".fmcb")
    os.close(fd)
    try:
        save_hierarchy(h, tmp)
        return load_hierarchy(tmp)
    finally:
        os.unlink(tmp)


# ---------------------------------------------------------------------------
# write_boundaries (geojson.hpp:276-353)
# ---------------------------------------------------------------------------

def _ring_coordinates(node: RegionNode) -> list:
    rings = []
    for r, b in enumerate(node.ring_starts):
        e = node.ring_starts[r + 1] if r + 1 < len(node.ring_starts) else len(node.nodes)
        ring = [[x, y] for x, y in node.nodes[b:e]]
        ring.append(list(node.nodes[b]))
        rings.append(ring)
    return rings


def _feature(node: RegionNode, props: dict) -> dict:
    x0, x1, y0, y1 = node.bbox
    return {"type": "Feature", "bbox": [x0, y0, x1, y1], "properties": props,
            "geometry": {"type": "Polygon", "coordinates": _ring_coordinates(node)}}


def write_boundaries(h: RegionHierarchy, out_dir: str) -> None:
    """states.geojson / counties.geojson / blocks.geojson under ``out_dir``."""
    os.makedirs(out_dir, exist_ok=True)
    states, counties, blocks = [], [], []
    for s in h.states:
        states.append(_feature(s, {"STATEFP": f"{s.fp_code:02d}"}))
        for c in s.children:
            counties.append(_feature(c, {"STATEFP": f"{s.fp_code:02d}", "COUNTYFP": f"{c.fp_code:03d}"}))
            for b in c.children:
                f = b.fips12
                blocks.append(_feature(b, {"STATE_FIPS": f[0:2], "CNTY_FIPS": f[2:5],
                                           "TRACT": f[5:11], "BLKGRP": f[11:12], "FIPS": f}))
    for name, feats in (("states", states), ("counties", counties), ("blocks", blocks)):
        path = os.path.join(out_dir, f"{name}.geojson")
        try:
            with open(path, "w", encoding="utf-8") as fh:
                json.dump({"type": "FeatureCollection", "features": feats}, fh)
                fh.write("\n")
        except OSError:
            raise RuntimeError(f"cannot open for writing: {path}") from None
