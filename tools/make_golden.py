#!/usr/bin/env python3
"""Generate tests/golden/*.npz from the REFERENCE itself (oracle/_ref, the
unmodified /root/reference headers compiled by oracle/Makefile).

Run here (where /root/reference exists):  python tools/make_golden.py
The fixtures pin oracle/oracle.c and the GPU path on machines where the
reference is absent (the GPU box).
"""
from __future__ import annotations

import hashlib
import pathlib
import sys

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import oracle  # noqa: E402
from paper_2005_03156_b200 import synth  # noqa: E402
from paper_2005_03156_b200.fastmap import Soup  # noqa: E402

OUT = ROOT / "tests" / "golden"


def soup_digest(soup: Soup) -> str:
    h = hashlib.sha256()
    for a in (soup.vxy, soup.ring_off, soup.poly_ring):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def star_polygons(rng, n_polys, n_vertices, r_min=0.5, r_max=2.0):
    """Random star polygons (sorted angles, random radii), like the reference
    test generator's shape (tests/oracles.hpp:250-265), restated in numpy."""
    polys = []
    for _ in range(n_polys):
        ang = np.sort(rng.random(n_vertices) * 2 * np.pi)
        rad = r_min + (r_max - r_min) * rng.random(n_vertices)
        polys.append([np.c_[rad * np.cos(ang), rad * np.sin(ang)]])
    return polys


def pip_fixture(rng):
    polys = star_polygons(rng, 40, 31)
    soup = Soup.from_rings(polys)
    pts_all, poly_of, want = [], [], []
    for p, rings in enumerate(polys):
        ring = rings[0]
        n = len(ring)
        pts = list(rng.random((120, 2)) * 5.0 - 2.5)
        for i in range(n):  # on-vertex, on-edge (midpoint), near-edge
            a, b = ring[i], ring[(i + 1) % n]
            pts += [a, 0.5 * (a + b), 0.5 * (a + b) + (1e-13, 0), 0.5 * (a + b) - (1e-13, 0)]
        for q in pts:
            pts_all.append(q)
            poly_of.append(p)
            want.append(oracle.ref_point_in_polygon(rings, float(q[0]), float(q[1])))
    return dict(vxy=soup.vxy, ring_off=soup.ring_off, poly_ring=soup.poly_ring,
                pts=np.asarray(pts_all), poly=np.asarray(poly_of, np.int32),
                inside=np.asarray(want, np.uint8))


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    rng = np.random.default_rng(20260)

    # 1. point_in_polygon bits (geometry.hpp:214-225) incl. on-edge ties
    np.savez_compressed(OUT / "pip_stars.npz", **pip_fixture(rng))

    # 2. reference acceptance fixture shape (acceptance.cpp:75-107):
    #    generate_synthetic(seed 2026, 4x4x25, jitter 0.2) + sample_uniform
    vxy, ro, pr, scb, fips, bbox = oracle.ref_generate_synthetic(2026, 4, 4, 25, 0.2)
    soup = Soup(vxy, ro, pr)
    pts = oracle.ref_sample(False, bbox, 20000, 777)
    m = oracle.RefModel(soup, scb)
    exh = m.exhaustive_assign(pts)
    m.build_index(12, 2)
    ql, _ = m.query_leaves(pts, threads=1)
    np.savez_compressed(OUT / "acceptance_4x4x25.npz", vxy=vxy, ring_off=ro, poly_ring=pr,
                        scb=scb, fips=np.asarray(fips), bbox=bbox, pts=pts,
                        exhaustive=exh, query_leaves=ql)

    # 3. BASELINE config 1 sample: ids from the reference exhaustive_assign
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points(20000, offset=123_456)
    m = oracle.RefModel(soup)
    exh = m.exhaustive_assign(pts)
    m.build_index(12, 4)
    ql, _ = m.query_leaves(pts, threads=1)
    np.savez_compressed(OUT / "c1_sample.npz", pts=pts, exhaustive=exh, query_leaves=ql,
                        soup_sha256=np.asarray(soup_digest(soup)),
                        first_vertices=soup.vxy[:64])

    # 4. adversarial edge cases (tests/edge_cases.py)
    import edge_cases
    soup, pts = edge_cases.build()
    m = oracle.RefModel(soup)
    exh = m.exhaustive_assign(pts)
    np.savez_compressed(OUT / "edge_cases.npz", pts=pts, exhaustive=exh,
                        soup_sha256=np.asarray(soup_digest(soup)))
    fmcb_fixture()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


def fmcb_fixture():
    """5. an FMCB file written by the reference's own save_hierarchy
    (hierarchy.hpp:190-202) over generate_synthetic(seed 11, 2x2x3, jitter
    0.2), plus the reference's collect_leaves view of it."""
    path = OUT / "hier_2x2x3.fmcb"
    oracle.ref_save_synthetic_fmcb(11, 2, 2, 3, 0.2, path)
    vxy, ro, pr, scb, fips, _ = oracle.ref_generate_synthetic(11, 2, 2, 3, 0.2)
    np.savez_compressed(OUT / "hier_2x2x3.npz", vxy=vxy, ring_off=ro, poly_ring=pr, scb=scb,
                        fips=np.asarray(fips, dtype="S12"))
    print(path.name, path.stat().st_size)


if __name__ == "__main__":
    if sys.argv[1:] == ["fmcb"]:
        fmcb_fixture()
    else:
        main()
