"""The CPU oracle against the reference: known-answer tests restated from the
reference suite, the reference-generated golden vectors (tests/golden/),
and -- where oracle/_ref is built -- live comparisons with the reference."""
import pathlib

import numpy as np
import pytest

import oracle
from paper_2005_03156_b200 import synth
from paper_2005_03156_b200.fastmap import Soup

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def unit_square():
    return Soup.from_rings([[[(0, 0), (1, 0), (1, 1), (0, 1)]]])


def square_with_hole():
    return Soup.from_rings([[[(0, 0), (3, 0), (3, 3), (0, 3)], [(1, 1), (2, 1), (2, 2), (1, 2)]]])


def test_kat_unit_square():  # test_geometry.cpp:89-95
    s = unit_square()
    assert oracle.point_in_polygon(s, 0, 0.5, 0.5)
    assert not oracle.point_in_polygon(s, 0, 1.5, 0.5)


def test_kat_hole():  # test_geometry.cpp:97-104
    s = square_with_hole()
    assert not oracle.point_in_polygon(s, 0, 1.5, 1.5)
    assert oracle.point_in_polygon(s, 0, 0.5, 1.5)
    assert not oracle.point_in_polygon(s, 0, 3.5, 1.5)


def test_kat_on_edge_tie_rule():
    # geometry.hpp:166-169: cross == 0 never flips; half-open lo < y <= hi
    s = unit_square()
    assert not oracle.point_in_polygon(s, 0, 1.0, 0.5)   # on the right edge
    assert oracle.point_in_polygon(s, 0, 0.0, 0.5)       # on the left edge (ray crosses right)
    assert oracle.point_in_polygon(s, 0, 0.5, 1.0)       # top edge: y <= hi counts
    assert not oracle.point_in_polygon(s, 0, 0.5, 0.0)   # bottom edge: lo < y fails


def test_golden_pip_bits():
    g = np.load(GOLD / "pip_stars.npz")
    soup = Soup(g["vxy"], g["ring_off"], g["poly_ring"])
    got = np.array([oracle.point_in_polygon(soup, int(p), float(x), float(y))
                    for (x, y), p in zip(g["pts"], g["poly"])], dtype=np.uint8)
    assert np.array_equal(got, g["inside"])


def test_golden_acceptance_fixture():
    g = np.load(GOLD / "acceptance_4x4x25.npz")
    soup = Soup(g["vxy"], g["ring_off"], g["poly_ring"])
    assert np.array_equal(oracle.assign(soup, g["pts"]), g["exhaustive"])
    assert np.array_equal(oracle.exhaustive_assign(soup, g["pts"][:3000]), g["exhaustive"][:3000])
    # valid tiling: the reference's own fast path agrees with exhaustive semantics
    assert np.array_equal(g["query_leaves"], g["exhaustive"])


def test_golden_c1_sample():
    g = np.load(GOLD / "c1_sample.npz")
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    import make_golden_digest
    assert make_golden_digest.digest(soup) == str(g["soup_sha256"]), "c1 generator changed"
    pts = cfg.make_points(20000, offset=123_456)
    assert np.array_equal(pts, g["pts"])
    assert np.array_equal(oracle.assign(soup, pts), g["exhaustive"])


def test_golden_edge_cases():
    import edge_cases
    import make_golden_digest
    g = np.load(GOLD / "edge_cases.npz")
    soup, pts = edge_cases.build()
    assert make_golden_digest.digest(soup) == str(g["soup_sha256"])
    want = g["exhaustive"].copy()
    # exhaustive_assign has no lon/lat domain filter; query_leaves does
    # (cell_index.hpp:549-552) -- the product follows query_leaves there
    outside = ~((np.abs(pts[:, 0]) <= 180) & (np.abs(pts[:, 1]) <= 90))
    want[outside] = -1
    assert np.array_equal(oracle.exhaustive_assign(soup, pts), want)
    assert np.array_equal(oracle.assign(soup, pts), want)


def test_bucketed_equals_exhaustive_on_configs():
    for name in ("c1", "c2"):
        cfg = synth.config(name)
        soup = cfg.make_soup()
        pts = cfg.make_points(2000 if name == "c1" else 300, offset=99)
        assert np.array_equal(oracle.assign(soup, pts), oracle.exhaustive_assign(soup, pts))


@needs_ref
def test_live_reference_pip_random_and_on_edge():
    rng = np.random.default_rng(5)
    for _ in range(20):
        n = int(rng.integers(3, 60))
        ang = np.sort(rng.random(n) * 2 * np.pi)
        rad = 0.5 + 1.5 * rng.random(n)
        ring = np.c_[rad * np.cos(ang), rad * np.sin(ang)]
        soup = Soup.from_rings([[ring]])
        qs = list(rng.random((50, 2)) * 5 - 2.5) + list(ring) + \
            [0.5 * (ring[i] + ring[(i + 1) % n]) for i in range(n)]
        for q in qs:
            assert oracle.point_in_polygon(soup, 0, q[0], q[1]) == \
                oracle.ref_point_in_polygon([ring], q[0], q[1])


@needs_ref
def test_live_reference_exhaustive_on_c4_sample():
    cfg = synth.config("c4")
    soup = cfg.make_soup()
    pts = cfg.make_points(120, soup=soup, offset=7)
    m = oracle.RefModel(soup)
    assert np.array_equal(m.exhaustive_assign(pts), oracle.assign(soup, pts))


@needs_ref
def test_reference_query_leaves_vs_exhaustive_disagreement_is_bounded():
    """SURVEY.md sec. 0 finding 2: on non-simple input the reference's fast
    path may differ from exhaustive semantics; the product follows
    exhaustive semantics.  On config 1 the difference is at most a handful."""
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points(50_000)
    m = oracle.RefModel(soup)
    m.build_index(12, 4)
    ql, _ = m.query_leaves(pts, threads=2)
    want = oracle.assign(soup, pts)
    assert (ql != want).sum() <= 10
