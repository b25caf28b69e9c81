"""Margin-scale exactness on the GPU:
vertices and edges at {0, 0.5, 1, 2, 4} x the classification margin d from
cell borders over several grid sizes, points at +-k ulps of cell borders, on
vertices and edges and 1e-9 .. 1e-13 cell widths off edges -- through both
query paths, against the oracle's exhaustive_assign (synthetic.hpp:193-205;
tie rule geometry.hpp:166-174)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import margin_cases  # noqa: E402
import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap, synth  # noqa: E402


def run(idx, pts, path):
    idx.set_query_path(path)
    d = torch.from_numpy(np.ascontiguousarray(pts)).to("cuda:0")
    out = idx.project(d)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("grid", [(64, 48), (257, 131), (1000, 999), (4093, 2039)])
def test_margin_scale_cases(grid):
    soup, pts, g = margin_cases.build(*grid, n_polys=240)
    idx = fastmap.build_index(soup, fastmap.CoverParams(nx=grid[0], ny=grid[1]), device=0)
    st = idx.stats()
    assert st["cell_w"] == g["w"] and st["gx0"] == g["gx0"] and st["margin"] == g["d"]
    want = oracle.exhaustive_assign(soup, pts)
    for path in ("stream", "binned"):
        got = run(idx, pts, path)
        assert int((got != want).sum()) == 0, path
    # answers are non-trivial: some points inside interior polygons, some in the frame
    frame = soup.n_polys - 1
    assert ((want >= 0) & (want < frame)).sum() > 1000 and (want == frame).sum() > 1000


def test_c4_points_within_1e9_to_1e13_cells_of_edges():
    cfg = synth.config("c4")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, device=0)
    st = idx.stats()
    pts = margin_cases.near_edge_points(soup, 400_000, st["cell_w"], seed=4)
    want = oracle.assign(soup, pts)
    for path in ("stream", "binned"):
        got = run(idx, pts, path)
        assert int((got != want).sum()) == 0, path
