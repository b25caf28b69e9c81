"""The GPU index builder against the host builder: byte-identical grid,
slot and overflow arrays (same classification arithmetic, same slot order),
and parity of queries on GPU-built indexes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import edge_cases  # noqa: E402
import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap, synth  # noqa: E402


def both(soup, **params):
    """Host builder and GPU builder, both into device indexes (so both get the
    same query-layout pass: block-major phase-1 slot numbering)."""
    p = fastmap.CoverParams(**params)
    h = fastmap.build_index(soup, p, device=0, on_gpu=False)
    g = fastmap.build_index(soup, p, device=0)
    return h, g


def assert_identical(h, g):
    hg, ha, hgeo = h.export()
    gg, ga, ggeo = g.export()
    assert hgeo == ggeo
    assert np.array_equal(hg, gg), f"grid differs in {(hg != gg).sum()} cells"
    assert ha.shape == ga.shape, (ha.shape, ga.shape)
    assert np.array_equal(ha, ga), f"arena differs in {(ha != ga).sum()} bytes"
    assert g.stats()["built_on_gpu"] == 1 and h.stats()["built_on_gpu"] == 0


@pytest.mark.parametrize("name,m", [("c1", 0), ("c1", 7), ("c2", 0), ("c4", 0), ("c3mini", 20)])
def test_gpu_build_identical_to_host(name, m):
    cfg = synth.config(name)
    soup = cfg.make_soup()
    h, g = both(soup, cells_per_polygon=m)
    assert_identical(h, g)


@pytest.mark.parametrize("grid", [(1, 1), (2, 3), (7, 5), (97, 13), (400, 300)])
def test_gpu_build_identical_edge_cases(grid):
    soup, pts = edge_cases.build()
    h, g = both(soup, nx=grid[0], ny=grid[1])
    assert_identical(h, g)
    d = torch.from_numpy(pts).cuda()
    got = g.project(d).cpu().numpy()
    assert np.array_equal(got, oracle.exhaustive_assign(soup, pts))


def test_c3mini_parity_on_gpu_built_index():
    cfg = synth.config("c3mini")
    soup = cfg.make_soup()
    pts = cfg.make_points(2_000_000)
    idx = fastmap.build_index(soup, device=0)
    got = idx.project(torch.from_numpy(pts).cuda()).cpu().numpy()
    assert np.array_equal(got, oracle.assign(soup, pts))


def test_block_major_renumbering_preserves_the_index():
    """The device-side slot renumbering (block-major phase-1 order) is a pure
    relabelling: walking the host-only (row-major) and the device index
    gives the same answers."""
    import index_walk
    cfg = synth.config("c2")
    soup = cfg.make_soup()
    h = fastmap.build_index(soup, device=-1)
    g = fastmap.build_index(soup, device=0)
    assert g.stats()["query_block_log2"] == 2  # 4x4 blocks, compact sub-blocks
    pts = cfg.make_points(100_000, offset=31)
    wh = index_walk.walk(h.export(), pts)
    wg = index_walk.walk(g.export(), pts)
    assert np.array_equal(wh, wg)
    assert np.array_equal(g.project(torch.from_numpy(pts).cuda()).cpu().numpy(), wh)
