"""The IO boundary on the GPU: indexes saved and reloaded answer exactly
like the originals (exact and fast-approx); an FMCB hierarchy feeds the
index build and query_leaves maps leaf ids to (state, county, block)."""
import pathlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap, synth  # noqa: E402
from paper_2005_03156_b200.fastmap import CoverMode, CoverParams  # noqa: E402

GOLD = pathlib.Path(__file__).resolve().parent / "golden"


def test_device_index_save_load_identical(tmp_path):
    cfg = synth.config("c2")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, device=0)
    path = tmp_path / "c2.fmgi"
    idx.save(path)
    back = fastmap.load_index(path, device=0)
    a, b = idx.export(), back.export()
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    sa, sb = idx.stats(), back.stats()
    assert sa["query_block_log2"] == sb["query_block_log2"] == 2
    assert sa["query_grid_bytes"] == sb["query_grid_bytes"]
    pts = cfg.make_points(1_000_000, offset=3)
    d = torch.from_numpy(pts).cuda()
    got = back.project(d).cpu().numpy()
    assert np.array_equal(got, idx.project(d).cpu().numpy())
    assert np.array_equal(got[:20000], oracle.assign(soup, pts[:20000]))


def test_approx_index_save_load(tmp_path):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, CoverParams(mode=CoverMode.approx, epsilon=0.005), device=0)
    path = tmp_path / "c1a.fmgi"
    idx.save(path)
    back = fastmap.load_index(path, device=0)
    assert back.params.mode == CoverMode.approx and back.stats()["approx_epsilon"] == 0.005
    pts = cfg.make_points(500_000, offset=9)
    d = torch.from_numpy(pts).cuda()
    assert np.array_equal(back.project(d, mode=CoverMode.approx).cpu().numpy(),
                          idx.project(d, mode=CoverMode.approx).cpu().numpy())


def test_fmcb_hierarchy_build_and_query(tmp_path):
    h = fastmap.load_hierarchy(GOLD / "hier_2x2x3.fmcb")
    idx = fastmap.build_cover(h, device=0)
    v = h.soup.vxy
    rng = np.random.default_rng(4)
    pts = np.c_[rng.uniform(v[:, 0].min() - 1, v[:, 0].max() + 1, 200_000),
                rng.uniform(v[:, 1].min() - 1, v[:, 1].max() + 1, 200_000)]
    res = fastmap.query_leaves(idx, h, pts)
    want = oracle.exhaustive_assign(h.soup, pts)
    assert np.array_equal(res.leaf, want)
    hit = want >= 0
    assert np.array_equal(res.block[hit], h.scb[want[hit], 2].astype(np.int32))
    assert np.array_equal(res.state[hit], h.scb[want[hit], 0].astype(np.int32))
    assert (res.state[~hit] == -1).all()
    out = tmp_path / "assign.csv"
    fastmap.write_assign_csv(out, pts[:1000], res.leaf[:1000], h)
    rows = out.read_text().splitlines()
    assert rows[0] == "idx,lon,lat,fips" and len(rows) == 1001
