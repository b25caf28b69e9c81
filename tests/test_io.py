"""The artifact and IO boundary, on CPU: the FMCB
hierarchy reader against files written by the reference's own
save_hierarchy (hierarchy.hpp:190-202) and against its load_hierarchy
verdicts on damaged files; the raw f64 points reader (io.hpp:154-167); the
assignment CSV (tools/fastmap.cpp:288-301); index save/load of host-only
indexes."""
import pathlib
import struct

import numpy as np
import pytest

import oracle
from paper_2005_03156_b200 import fastmap, synth

GOLD = pathlib.Path(__file__).resolve().parent / "golden"
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def same_leaves(h, vxy, ro, pr, scb, fips):
    assert np.array_equal(h.soup.vxy, vxy)
    assert np.array_equal(h.soup.ring_off, ro)
    assert np.array_equal(h.soup.poly_ring, pr)
    assert np.array_equal(h.scb, scb)
    assert [f.decode() if isinstance(f, bytes) else f for f in h.fips12] == \
        [f.decode() if isinstance(f, bytes) else f for f in fips]


def test_golden_fmcb_matches_reference_leaves():
    h = fastmap.load_hierarchy(GOLD / "hier_2x2x3.fmcb")
    g = np.load(GOLD / "hier_2x2x3.npz")
    assert (h.n_states, h.n_counties, h.n_leaves) == (2, 4, 12)
    same_leaves(h, g["vxy"], g["ring_off"], g["poly_ring"], g["scb"], list(g["fips"]))


@needs_ref
def test_reference_written_fmcb_round_trip(tmp_path):
    path = tmp_path / "h.fmcb"
    oracle.ref_save_synthetic_fmcb(2026, 4, 4, 25, 0.2, path)  # acceptance.cpp fixture shape
    h = fastmap.load_hierarchy(path)
    vxy, ro, pr, scb, fips, _ = oracle.ref_generate_synthetic(2026, 4, 4, 25, 0.2)
    assert h.n_leaves == 400
    same_leaves(h, vxy, ro, pr, scb, fips)


def damaged(tmp_path, name, data: bytes):
    p = tmp_path / name
    p.write_bytes(data)
    return p


def fmcb_cases(tmp_path):
    raw = (GOLD / "hier_2x2x3.fmcb").read_bytes()
    # first state node starts at byte 30: i64 fp, 4 f64 bbox, u32 n_vertices
    nv = struct.unpack_from("<I", raw, 30 + 8 + 32)[0]
    ring_pos = 30 + 8 + 32 + 4 + 16 * nv + 4  # first ring start of the first state
    bad_ring = bytearray(raw)
    struct.pack_into("<I", bad_ring, ring_pos, nv + 5)  # ring start past the vertices
    short_ring = bytearray(raw)
    struct.pack_into("<I", short_ring, ring_pos, nv - 2)  # a 2-vertex ring
    counts = bytearray(raw)
    struct.pack_into("<Q", counts, 22, 13)  # 13 blocks declared, 12 present
    return {
        "ok": (raw, 0),
        "bad_magic": (b"FMCX" + raw[4:], 1),
        "bad_version": (raw[:4] + struct.pack("<H", 2) + raw[6:], 1),
        "truncated": (raw[:len(raw) // 2], 1),
        "corrupt_ring": (bytes(bad_ring), 1),
        "short_ring": (bytes(short_ring), 2),
        "count_mismatch": (bytes(counts), 1),
    }


def test_fmcb_errors_map_like_the_reference(tmp_path):
    expect_exc = {0: None, 1: RuntimeError, 2: ValueError}
    for name, (data, want) in fmcb_cases(tmp_path).items():
        p = damaged(tmp_path, name, data)
        if oracle.ref_available():  # the reference's own verdict on the same bytes
            assert oracle.ref_load_fmcb_status(p) == want, name
        if want == 0:
            assert fastmap.load_hierarchy(p).n_leaves == 12
        else:
            with pytest.raises(expect_exc[want]):
                fastmap.load_hierarchy(p)
    with pytest.raises(RuntimeError, match="cannot open"):
        fastmap.load_hierarchy(tmp_path / "missing.fmcb")


def test_read_points_f64(tmp_path):
    pts = np.array([[-100.5, 40.25], [np.nan, 1.0], [1e300, -1e-300]], dtype="<f8")
    p = tmp_path / "pts.f64"
    pts.tofile(p)
    got = fastmap.read_points_f64(p)
    assert got.shape == (3, 2)
    assert np.array_equal(got[[0, 2]], pts[[0, 2]]) and np.isnan(got[1, 0])
    (tmp_path / "empty.f64").write_bytes(b"")
    assert fastmap.read_points_f64(tmp_path / "empty.f64").shape == (0, 2)
    (tmp_path / "odd.f64").write_bytes(pts.tobytes()[:40])
    with pytest.raises(RuntimeError, match="truncated"):
        fastmap.read_points_f64(tmp_path / "odd.f64")


def test_assign_csv_format(tmp_path):
    h = fastmap.load_hierarchy(GOLD / "hier_2x2x3.fmcb")
    pts = np.array([[0.1, 0.2], [np.inf, 0.0], [-1.0 / 3.0, 2.5e-7], [5.0, 5.0]])
    ids = np.array([3, 0, 11, -1], dtype=np.int32)
    p = tmp_path / "out.csv"
    fastmap.write_assign_csv(p, pts, ids, h)
    fips = [f.decode() for f in h.fips12]
    want = ["idx,lon,lat,fips",
            f"0,{'%.17g' % 0.1},{'%.17g' % 0.2},{fips[3]}",
            f"2,{'%.17g' % (-1.0 / 3.0)},{'%.17g' % 2.5e-7},{fips[11]}",
            f"3,{'%.17g' % 5.0},{'%.17g' % 5.0},"]
    assert p.read_text().splitlines() == want


def test_index_save_load_host_only(tmp_path):
    soup = synth.config("c1").make_soup()
    idx = fastmap.build_index(soup, device=-1)
    path = tmp_path / "c1.fmgi"
    idx.save(path)
    back = fastmap.load_index(path, device=-1)
    a, b = idx.export(), back.export()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2]
    sa, sb = idx.stats(), back.stats()
    for k in ("n_polys", "nx", "ny", "cells_boundary", "slots_total", "slots_phase1"):
        assert sa[k] == sb[k], k
    raw = path.read_bytes()
    (tmp_path / "bad.fmgi").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(RuntimeError, match="bad magic"):
        fastmap.load_index(tmp_path / "bad.fmgi", device=-1)
    (tmp_path / "short.fmgi").write_bytes(raw[: len(raw) - 100])
    with pytest.raises(RuntimeError, match="truncated"):
        fastmap.load_index(tmp_path / "short.fmgi", device=-1)


def test_hierarchy_index_build_host_only():
    h = fastmap.load_hierarchy(GOLD / "hier_2x2x3.fmcb")
    idx = fastmap.build_cover(h, device=-1)
    assert idx.stats()["n_polys"] == 12


def test_python_written_fmcb_loads_like_the_reference(tmp_path):
    import fmcb_writer
    p = tmp_path / "adv.fmcb"
    states = fmcb_writer.random_hierarchy(5)
    fmcb_writer.write_fmcb(p, states)
    if oracle.ref_available():
        assert oracle.ref_load_fmcb_status(p) == 0
    h = fastmap.load_hierarchy(p)
    assert (h.n_states, h.n_counties, h.n_leaves) == (3, 9, 36)
    leaves = [b for s in states for c in s["children"] for b in c["children"]]
    assert [f.decode() for f in h.fips12] == [b["fips"] for b in leaves]
    for k, b in enumerate(leaves):  # rings in file order, collect_leaves order
        got = h.soup.polygon(k)
        assert len(got) == len(b["rings"])
        for r, want in zip(got, b["rings"]):
            assert np.array_equal(r, np.asarray(want, dtype=np.float64))
