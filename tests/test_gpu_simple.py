"""The simple engine (simple_mapper.hpp:62-166) on the GPU against the
reference's own assign() on the same FMCB bytes (oracle/_ref): state,
county and block per point and both counters, in relaxed and strict mode,
on reference-generated hierarchies and on adversarial ones (overlapping
bboxes, holes, file bboxes larger than their polygons, points on edges and
vertices)."""
import pathlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import fmcb_writer  # noqa: E402
import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap  # noqa: E402
from paper_2005_03156_b200.fastmap import AssignMode  # noqa: E402

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def probe_points(h, n, seed):
    v = h.soup.vxy
    rng = np.random.default_rng(seed)
    lo, hi = v.min(0) - 0.5, v.max(0) + 0.5
    pts = rng.uniform(lo, hi, (n, 2))
    # vertices, edge midpoints and points just off them
    idx = rng.integers(0, v.shape[0], 2000)
    nxt = np.minimum(idx + 1, v.shape[0] - 1)
    extra = np.concatenate([v[idx], 0.5 * (v[idx] + v[nxt]), v[idx] + 1e-12])
    return np.ascontiguousarray(np.concatenate([pts, extra]))


def test_non_finite_points_are_unassigned(tmp_path):
    """The reference CLI drops non-finite rows before assign()
    (tools/fastmap.cpp:240-251; its bbox_membership sorts by lon, which NaN
    leaves unordered).  Here they are simply unresolved in both modes."""
    p = tmp_path / "adv.fmcb"
    fmcb_writer.write_fmcb(p, fmcb_writer.random_hierarchy(1))
    eng = fastmap.SimpleEngine(fastmap.load_hierarchy(p))
    pts = np.array([[np.nan, 0.0], [0.0, np.inf], [np.inf, np.nan], [-np.inf, 1.0]])
    for mode in (AssignMode.relaxed, AssignMode.strict):
        r = eng.assign(pts, mode)
        assert (r.state == -1).all() and (r.block == -1).all()


def check_against_reference(path, pts):
    h = fastmap.load_hierarchy(path)
    eng = fastmap.SimpleEngine(h)
    for mode in (AssignMode.relaxed, AssignMode.strict):
        got = eng.assign(pts, mode)
        st, co, bl, cnt = oracle.ref_simple_assign(path, pts, mode == AssignMode.strict)
        assert np.array_equal(got.state, st), mode
        assert np.array_equal(got.county, co), mode
        assert np.array_equal(got.block, bl), mode
        assert (got.counters.pip_point_evaluations, got.counters.pip_calls) == cnt, mode
        d = torch.from_numpy(pts).cuda()
        ds, dc, db = eng.assign(d, mode, counters=False)
        assert np.array_equal(db.cpu().numpy(), bl) and np.array_equal(ds.cpu().numpy(), st)
    return got


def test_kat_relaxed_falls_back_to_highest_candidate(tmp_path):
    # test_simple_mapper.cpp:104-142
    p = tmp_path / "tri.fmcb"
    fmcb_writer.write_fmcb(p, fmcb_writer.two_triangles())
    eng = fastmap.SimpleEngine(fastmap.load_hierarchy(p))
    pts = np.array([[1.9, 1.9], [40.0, 40.0]])
    strict = eng.assign(pts, AssignMode.strict)
    assert strict.state[0] == -1
    relaxed = eng.assign(pts, AssignMode.relaxed)
    assert relaxed.state[0] == 1 and relaxed.block[0] == 0
    assert relaxed.state[1] == -1 and strict.state[1] == -1


@needs_ref
@pytest.mark.parametrize("spec", [(3, 2, 2, 9, 0.2), (4, 4, 4, 9, 0.3), (6, 2, 2, 6, 0.25),
                                  (2026, 4, 4, 25, 0.2), (1, 2, 2, 4, 0.0)])
def test_reference_hierarchies(tmp_path, spec):
    p = tmp_path / "h.fmcb"
    oracle.ref_save_synthetic_fmcb(*spec, p)
    h = fastmap.load_hierarchy(p)
    check_against_reference(p, probe_points(h, 30_000, spec[0]))


@needs_ref
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_adversarial_hierarchies(tmp_path, seed):
    p = tmp_path / f"adv{seed}.fmcb"
    fmcb_writer.write_fmcb(p, fmcb_writer.random_hierarchy(seed))
    h = fastmap.load_hierarchy(p)
    got = check_against_reference(p, probe_points(h, 30_000, 100 + seed))
    assert got.counters.pip_point_evaluations > 0


def test_golden_hierarchy_strict_equals_exhaustive():
    """Strict mode on a valid tiling equals exhaustive_assign off the edges
    (test_cell_index.cpp:341-379 / test_simple_mapper.cpp:74-86)."""
    h = fastmap.load_hierarchy(GOLD / "hier_2x2x3.fmcb")
    v = h.soup.vxy
    pts = np.random.default_rng(8).uniform(v.min(0), v.max(0), (50_000, 2))
    res = fastmap.assign(h, pts, AssignMode.strict)
    leaf = oracle.exhaustive_assign(h.soup, pts)
    hit = leaf >= 0
    assert np.array_equal(res.block[hit], h.scb[leaf[hit], 2].astype(np.int32))
    assert np.array_equal(res.county[hit], h.scb[leaf[hit], 1].astype(np.int32))


def test_nested_config_against_reference(tmp_path):
    """The bench hierarchy recipe (c3mini scale): both modes vs the reference;
    strict additionally equals the leaf-exact projection off the edges."""
    from paper_2005_03156_b200 import synth
    cfg = synth.config("c3mini")
    p = tmp_path / "c3mini.fmcb"
    cfg.write_fmcb(p)
    pts = cfg.make_points(200_000)
    if oracle.ref_available():
        check_against_reference(p, pts[:50_000])
    h = fastmap.load_hierarchy(p)
    res = fastmap.assign(h, pts, AssignMode.strict)
    leaf = oracle.assign(h.soup, pts)
    hit = leaf >= 0
    agree = (res.block[hit] == h.scb[leaf[hit], 2].astype(np.int32)).mean()
    assert agree > 0.9999  # differs only for points on shared state/county borders


@needs_ref
def test_hierarchy_straddling_the_world_box(tmp_path):
    """Regions partly outside lon 180: there the level indexes answer -1 by
    query_leaves' world rule (cell_index.hpp:549-552), which assign() does
    not have, so the engine must fall back to the crossing tests."""
    states = fmcb_writer.random_hierarchy(4)
    def shift(node):
        node["rings"] = [[(x + 177.5, y + 87.0) for x, y in r] for r in node["rings"]]
        if node.get("bbox"):
            x0, x1, y0, y1 = node["bbox"]
            node["bbox"] = (x0 + 177.5, x1 + 177.5, y0 + 87.0, y1 + 87.0)
        for c in node.get("children", []):
            shift(c)
    for s in states:
        shift(s)
    p = tmp_path / "edge.fmcb"
    fmcb_writer.write_fmcb(p, states)
    h = fastmap.load_hierarchy(p)
    pts = probe_points(h, 30_000, 9)
    assert (pts[:, 0] > 180.0).mean() > 0.1 and (pts[:, 1] > 90.0).mean() > 0.1
    got = check_against_reference(p, pts)
    assert (got.state[pts[:, 0] > 180.0] >= 0).any()  # assigned outside the world box
