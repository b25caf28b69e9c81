"""The index builder, checked on the CPU: a host-only index (device=-1) is
exported and walked by tests/index_walk.py (a Python restatement of the
query kernel's record walk) and compared with the oracle bit for bit."""
import numpy as np
import pytest

import edge_cases
import index_walk
import oracle
from paper_2005_03156_b200 import fastmap, synth


def walk(soup, pts, **params):
    idx = fastmap.build_index(soup, fastmap.CoverParams(**params), device=-1)
    ex = idx.export()
    return index_walk.walk(ex, pts), idx, ex


def test_c1_index_exact():
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points(100_000, offset=777)
    got, idx, ex = walk(soup, pts)
    assert np.array_equal(got, oracle.assign(soup, pts))
    st = idx.stats()
    assert st["cells_boundary"] > 0 and st["cells_hit"] > st["cells_boundary"]


@pytest.mark.parametrize("name,m", [("c2", 6), ("c2", 14), ("c4", 24), ("c3mini", 16)])
def test_large_config_index_exact_sampled(name, m):
    cfg = synth.config(name)
    soup = cfg.make_soup()
    pts = cfg.make_points(8_000, soup=soup, offset=12345)
    got, _, _ = walk(soup, pts, cells_per_polygon=m)
    assert np.array_equal(got, oracle.assign(soup, pts))


@pytest.mark.parametrize("grid", [(1, 1), (2, 3), (7, 5), (97, 13), (400, 300)])
def test_edge_cases_every_resolution(grid):
    soup, pts = edge_cases.build()
    got, _, ex = walk(soup, pts, nx=grid[0], ny=grid[1])
    assert np.array_equal(got, oracle.exhaustive_assign(soup, pts))


def test_edge_cases_use_wide_and_split_records():
    soup, pts = edge_cases.build()
    _, _, ex = walk(soup, pts, nx=1, ny=1)
    kinds = index_walk.record_kinds(ex)
    assert kinds["split"] >= 1 and kinds["overflow"] >= 1
    got, _, _ = walk(soup, pts, nx=1, ny=1)
    assert np.array_equal(got, oracle.exhaustive_assign(soup, pts))


def test_acceptance_fixture_index_exact():
    import pathlib
    g = np.load(pathlib.Path(__file__).parent / "golden" / "acceptance_4x4x25.npz")
    soup = fastmap.Soup(g["vxy"], g["ring_off"], g["poly_ring"])
    got, _, _ = walk(soup, g["pts"])
    assert np.array_equal(got, g["exhaustive"])


def test_empty_soup_and_zero_ring_polygons():
    empty = fastmap.Soup.from_rings([])
    got, idx, _ = walk(empty, np.array([[0.0, 0.0], [10.0, 10.0]]))
    assert (got == -1).all()
    soup = fastmap.Soup.from_rings([[], [[(0, 0), (1, 0), (1, 1), (0, 1)]], []])
    pts = np.array([[0.5, 0.5], [2.0, 2.0], [0.0, 0.0]])
    got, _, _ = walk(soup, pts)
    assert np.array_equal(got, oracle.exhaustive_assign(soup, pts))
    assert got[0] == 1


def test_slot_invariants():
    """Leaf slots: ascending distinct candidate ids, masks inside the edge
    range, counts within the slot capacity."""
    import struct
    cfg = synth.config("c1")
    _, _, (grid, arena, g) = walk(cfg.make_soup(), np.zeros((1, 2)))
    recs = np.unique(grid[(grid >= 0x80000000) & (grid != 0xFFFFFFFF)])
    recs = np.random.default_rng(0).choice(recs, min(3000, recs.size), replace=False)
    n_leaf = 0
    n_half = 0
    n_double = 0
    for e in recs.tolist():
        off = (e & 0x1FFFFFFF) * 128
        kind, nv, nc, nb = arena[off:off + 4].tolist()
        assert kind in (1, 2, 3, 4)
        half = bool(e & 0x40000000)
        n_half += half
        assert bool(e & 0x20000000) == (kind == 4)
        if kind == 4:  # double leaf slot: never half, within its capacity
            n_double += 1
            assert not half and 1 <= nc <= 8 and nb <= 4 and nv <= 10
            assert nv > 5 or nc > 4 or nb > 2  # it did not fit a leaf slot
            ids = list(struct.unpack_from("<8i", arena.data, off + 8))[:nc]
            assert ids == sorted(ids) and len(set(ids)) == nc
            continue
        if kind != 1:
            assert half and not arena[off + 64: off + 128].any()
            continue
        n_leaf += 1
        assert 1 <= nc <= 4 and nb <= 2 and nv <= 5
        assert half == (nc <= 2 and ((nv <= 2 and nb <= 1) or (nv == 3 and nb == 0)))
        if half:
            assert not arena[off + 64: off + 128].any()
        ids = (list(struct.unpack_from("<2i", arena.data, off + 8))
               + list(struct.unpack_from("<2i", arena.data, off + 72)))[:nc]
        assert ids == sorted(ids) and len(set(ids)) == nc
        masks = arena[off + 4: off + 6].tolist() + arena[off + 68: off + 70].tolist()
        for mk in masks[:nc]:
            assert mk < (1 << max(nv - 1, 0)) or mk == 0
    assert n_half > 0
    assert n_leaf > 0
    assert n_double > 0  # c1's polygon corners


@pytest.mark.parametrize("grid", [(64, 48), (257, 131), (1000, 999)])
def test_margin_scale_cases_index_exact(grid):
    """Vertices and edges at {0, 0.5, 1, 2, 4} x margin from cell borders,
    points at +-k ulps of the borders, on vertices and edges and 1e-9 ..
    1e-13 cell widths off them (tests/margin_cases.py)."""
    import margin_cases
    soup, pts, g = margin_cases.build(*grid)
    got, idx, _ = walk(soup, pts, nx=grid[0], ny=grid[1])
    st = idx.stats()
    # the cases are built against the builder's own cell borders
    assert st["gx0"] == g["gx0"] and st["gy0"] == g["gy0"]
    assert st["cell_w"] == g["w"] and st["cell_h"] == g["h"] and st["margin"] == g["d"]
    assert st["cells_boundary"] > 0
    assert np.array_equal(got, oracle.exhaustive_assign(soup, pts))
