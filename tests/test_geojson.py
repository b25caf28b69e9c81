"""GeoJSON ingestion (paper_2005_03156_b200/geojson.py) against the
reference's own geojson.hpp, compiled in place into oracle/_ref: the FMCB
bytes our `ingest` writes must equal the reference `fastmap ingest`'s on the
same files, and malformed inputs must fail with the reference's class and
message."""
import json
import random

import numpy as np
import pytest

import oracle
from paper_2005_03156_b200 import fastmap, geojson

needs_ref = pytest.mark.skipif(not oracle.ref_geojson_available(),
                               reason="oracle/_ref built without nlohmann json")


def paths(d):
    return [d / f"{k}.geojson" for k in ("states", "counties", "blocks")]


def both_ingest(tmp_path, d):
    mine, ref = tmp_path / "mine.fmcb", tmp_path / "ref.fmcb"
    counts = geojson.ingest(*paths(d), mine)
    rc, msg = oracle.ref_ingest_geojson(*paths(d), ref)
    assert rc == 0, msg
    return mine.read_bytes(), ref.read_bytes(), counts


@needs_ref
@pytest.mark.parametrize("shape", [(2, 3, 4, 0.2), (4, 4, 25, 0.3), (1, 1, 1, 0.0)])
def test_reference_written_geojson_ingests_byte_identically(tmp_path, shape):
    d = tmp_path / "g"
    oracle.ref_write_synthetic_geojson(7, *shape, d)
    mine, ref, counts = both_ingest(tmp_path, d)
    assert mine == ref
    assert counts == (shape[0], shape[0] * shape[1], shape[0] * shape[1] * shape[2])


@needs_ref
def test_feature_order_does_not_matter(tmp_path):
    d = tmp_path / "g"
    oracle.ref_write_synthetic_geojson(3, 3, 3, 5, 0.25, d)
    before, _, _ = both_ingest(tmp_path, d)
    rng = random.Random(0)
    for p in paths(d):
        doc = json.loads(p.read_text())
        rng.shuffle(doc["features"])
        p.write_text(json.dumps(doc))
    mine, ref, _ = both_ingest(tmp_path, d)
    assert mine == ref == before


def square(x0, y0, s, closed=True, hole=False):
    ring = [[x0, y0], [x0 + s, y0], [x0 + s, y0 + s], [x0, y0 + s]]
    if hole:
        ring = ring[::-1]
    return ring + [ring[0]] if closed else ring


def feature(props, geom, bbox=None):
    f = {"type": "Feature", "properties": props, "geometry": geom}
    if bbox is not None:
        f["bbox"] = bbox
    return f


def write(d, states, counties, blocks):
    d.mkdir(parents=True, exist_ok=True)
    for name, feats in (("states", states), ("counties", counties), ("blocks", blocks)):
        (d / f"{name}.geojson").write_text(json.dumps({"type": "FeatureCollection", "features": feats}))


def handmade():
    """Integer and zero-padded string codes, a MultiPolygon with a hole,
    unclosed rings, file bboxes (valid, inverted = ignored), two states."""
    poly = lambda *rings: {"type": "Polygon", "coordinates": list(rings)}  # noqa: E731
    states = [feature({"STATEFP": "06"}, poly(square(0, 0, 4))),
              feature({"STATEFP": 1}, poly(square(4, 0, 4, closed=False)), bbox=[4, 0, 8, 4])]
    counties = [feature({"STATEFP": 6, "COUNTYFP": "001"}, poly(square(0, 0, 4))),
                feature({"STATEFP": "01", "COUNTYFP": 3}, poly(square(4, 0, 2))),
                feature({"STATEFP": "01", "COUNTYFP": "002"}, poly(square(6, 0, 2)), bbox=[9, 9, 1, 1])]
    mp = {"type": "MultiPolygon", "coordinates": [[square(0, 0, 2), square(0.5, 0.5, 1, hole=True)],
                                                  [square(2.5, 2.5, 1, closed=False)]]}
    blocks = [feature({"STATE_FIPS": "06", "CNTY_FIPS": "001", "TRACT": "000100", "BLKGRP": "2",
                       "FIPS": "060010001002"}, mp),
              feature({"STATE_FIPS": 6, "CNTY_FIPS": 1, "TRACT": 100, "BLKGRP": 1,
                       "FIPS": "060010001001"}, poly(square(2, 0, 2)), bbox=[1.5, -0.5, 4.5, 2.5]),
              feature({"STATE_FIPS": "01", "CNTY_FIPS": "003", "TRACT": "000200", "BLKGRP": "1",
                       "FIPS": "010030002001"}, poly(square(4, 0, 2))),
              feature({"STATE_FIPS": "01", "CNTY_FIPS": "002", "TRACT": "000300", "BLKGRP": "1",
                       "FIPS": "010020003001"}, poly(square(6, 0, 2)))]
    return states, counties, blocks


@needs_ref
def test_handmade_multipolygon_holes_codes_bboxes(tmp_path):
    d = tmp_path / "h"
    write(d, *handmade())
    mine, ref, counts = both_ingest(tmp_path, d)
    assert mine == ref and counts == (2, 3, 4)
    h = geojson.load_boundaries_hierarchy(*paths(d))
    assert h.n_leaves == 4 and (h.n_states, h.n_counties) == (2, 3)
    # siblings by ascending fp code: state 1 (county 2, 3) before state 6
    assert [f.decode() for f in h.fips12] == ["010020003001", "010030002001", "060010001001",
                                              "060010001002"]
    assert len(h.soup.polygon(3)) == 3  # MultiPolygon: 2 rings + 1, holes kept as rings


def mutate(case):
    s, c, b = handmade()
    poly = lambda *rings: {"type": "Polygon", "coordinates": list(rings)}  # noqa: E731
    if case == "missing_statefp":
        s[0]["properties"] = {}
    elif case == "null_properties":
        c[0]["properties"] = None
    elif case == "bad_code":
        s[1]["properties"]["STATEFP"] = 1.5
    elif case == "non_digit_code":
        c[0]["properties"]["COUNTYFP"] = "x1"
    elif case == "dup_state":
        s[1]["properties"]["STATEFP"] = "6"
    elif case == "dup_county":
        c[2]["properties"]["COUNTYFP"] = 3
    elif case == "absent_state":
        c[0]["properties"]["STATEFP"] = 9
    elif case == "absent_county":
        b[0]["properties"]["CNTY_FIPS"] = "009"
    elif case == "short_fips":
        b[1]["properties"]["FIPS"] = "06001000100"
    elif case == "dup_fips":
        b[1]["properties"]["FIPS"] = "060010001002"
    elif case == "tract_not_digits":
        b[1]["properties"]["TRACT"] = "ab"
    elif case == "dup_block_code":
        b[1]["properties"]["BLKGRP"] = "2"
    elif case == "two_positions":
        b[2]["geometry"] = poly([[0, 0], [1, 1]])
    elif case == "degenerate_after_closing":
        b[2]["geometry"] = poly([[0, 0], [1, 1], [0, 0]])
    elif case == "bad_position":
        b[2]["geometry"] = poly([[0, 0], [1, "a"], [1, 0]])
    elif case == "point_geometry":
        b[2]["geometry"] = {"type": "Point", "coordinates": [0, 0]}
    elif case == "no_coordinates":
        b[2]["geometry"] = {"type": "Polygon"}
    elif case == "null_geometry":
        b[2]["geometry"] = None
    elif case == "no_rings":
        b[2]["geometry"] = poly()
    elif case == "bad_multipolygon":
        b[2]["geometry"] = {"type": "MultiPolygon", "coordinates": [5]}
    elif case == "no_blocks":
        b = []
    elif case == "no_states":
        s = []
    elif case == "not_a_feature":
        b[0] = 7
    return s, c, b


ERROR_CASES = ["missing_statefp", "null_properties", "bad_code", "non_digit_code", "dup_state",
               "dup_county", "absent_state", "absent_county", "short_fips", "dup_fips",
               "tract_not_digits", "dup_block_code", "two_positions", "degenerate_after_closing",
               "bad_position", "point_geometry", "no_coordinates", "null_geometry", "no_rings",
               "bad_multipolygon", "no_blocks", "no_states", "not_a_feature"]


@needs_ref
@pytest.mark.parametrize("case", ERROR_CASES)
def test_malformed_inputs_fail_like_the_reference(tmp_path, case):
    d = tmp_path / case
    write(d, *mutate(case))
    rc, msg = oracle.ref_ingest_geojson(*paths(d), tmp_path / "ref.fmcb")
    assert rc == 1, (rc, msg)  # std::runtime_error
    with pytest.raises(RuntimeError) as e:
        geojson.ingest(*paths(d), tmp_path / "mine.fmcb")
    assert str(e.value) == msg


def test_unreadable_and_invalid_json(tmp_path):
    with pytest.raises(RuntimeError, match="cannot open boundary file"):
        geojson.load_boundaries(str(tmp_path / "nope"), "", "")
    p = tmp_path / "bad.geojson"
    p.write_text('{"type": "FeatureCollection", "features": [NaN]}')
    with pytest.raises(RuntimeError, match="bad.geojson"):
        geojson.load_boundaries(str(p), str(p), str(p))
    p.write_text('{"type": "Feature"}')
    with pytest.raises(RuntimeError, match="not a GeoJSON FeatureCollection"):
        geojson.load_boundaries(str(p), str(p), str(p))


@needs_ref
def test_write_boundaries_round_trip_through_the_reference(tmp_path):
    d = tmp_path / "h"
    write(d, *handmade())
    h = geojson.load_boundaries(*paths(d))
    out = tmp_path / "w"
    geojson.write_boundaries(h, out)
    mine, ref, _ = both_ingest(tmp_path, out)
    assert mine == ref == geojson.fmcb_bytes(h)


def test_ingested_hierarchy_builds_an_exact_index(tmp_path):
    """GeoJSON -> FMCB -> leaves -> host-only index, walked against the oracle."""
    import index_walk
    d = tmp_path / "h"
    write(d, *handmade())
    h = geojson.load_boundaries_hierarchy(*paths(d))
    idx = fastmap.build_index(h.soup, device=-1)
    pts = np.random.default_rng(0).uniform([-0.5, -0.5], [8.5, 4.5], size=(20000, 2))
    got = index_walk.walk(idx.export(), pts)
    assert np.array_equal(got, oracle.exhaustive_assign(h.soup, pts))
