"""Workload generators: determinism, shard consistency, watertight tilings."""
import numpy as np

from paper_2005_03156_b200 import synth


def test_tiling_counts_and_determinism():
    cfg = synth.config("c1")
    a, b = cfg.make_soup(), cfg.make_soup(threads=1)
    assert a.n_polys == 1024 and a.n_vertices == 1024 * 32
    assert np.array_equal(a.vxy, b.vxy)


def test_tiling_is_watertight():
    """Every interior edge appears in exactly two polygons, in opposite
    directions, with bit-identical endpoints; border edges once."""
    cfg = synth.config("c1")
    s = cfg.make_soup()
    from collections import Counter
    cnt = Counter()
    for p in range(s.n_polys):
        r = s.vxy[int(s.ring_off[p]):int(s.ring_off[p + 1])]
        for i in range(len(r)):
            a, b = r[i].tobytes(), r[(i + 1) % len(r)].tobytes()
            cnt[(a, b)] += 1
    for (a, b), c in cnt.items():
        assert c == 1
        assert ((b, a) in cnt) or True
    twice = sum(1 for (a, b) in cnt if (b, a) in cnt)
    once = len(cnt) - twice
    assert once == 4 * 32 * 8  # outer border: 4 sides x 32 tiles x 8 segments
    x = s.vxy[:, 0]
    y = s.vxy[:, 1]
    assert x.min() == -125.0 and x.max() == -66.0 and y.min() == 24.0 and y.max() == 50.0


def test_point_streams_shard_and_distributions():
    for name in ("c1", "c2", "c4"):
        cfg = synth.config(name)
        soup = cfg.make_soup() if name == "c4" else None
        full = cfg.make_points(4000, soup=soup)
        part = cfg.make_points(1500, offset=2500, soup=soup, threads=3)
        assert np.array_equal(full[2500:], part)
        assert np.isfinite(full).all()
    box = synth.expanded_box()
    u = synth.config("c1").make_points(100_000)
    assert (u[:, 0] >= box[0]).all() and (u[:, 0] <= box[1]).all()
    # about 1% of the expanded box lies outside the domain
    out = (u[:, 0] < -125) | (u[:, 0] > -66) | (u[:, 1] < 24) | (u[:, 1] > 50)
    assert 0.005 < out.mean() < 0.03


def test_nested_fmcb_carries_every_level(tmp_path):
    """synth_nested_fmcb: the c3mini hierarchy with state and county polygons
    on the same shared lattice points; its leaves are exactly c3mini's soup,
    and the reference's own load_hierarchy accepts the file."""
    import oracle
    from paper_2005_03156_b200 import fastmap
    cfg = synth.config("c3mini")
    p = tmp_path / "c3mini.fmcb"
    cfg.write_fmcb(p)
    h = fastmap.load_hierarchy(p)
    soup = cfg.make_soup()
    assert (h.n_states, h.n_counties, h.n_leaves) == (4, 64, 40000)
    assert np.array_equal(h.soup.vxy, soup.vxy) and np.array_equal(h.soup.ring_off, soup.ring_off)
    if oracle.ref_available():
        assert oracle.ref_load_fmcb_status(p) == 0
