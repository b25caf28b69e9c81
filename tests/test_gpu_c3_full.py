"""The full config-3 index on the GPU: the 12.5M-leaf
nested tiling (300M vertices; ~47 GB of slots), 4M clustered points of the
benchmark stream plus 1M uniform points and points on / next to leaf
vertices, through both query paths, bit-exact against the CPU oracle
(exhaustive_assign semantics, synthetic.hpp:193-205).  About 2 minutes:
the soup, the index build and the 4M-point oracle pass dominate."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import margin_cases  # noqa: E402
import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap, synth  # noqa: E402


def test_c3_full_index_bit_exact():
    cfg = synth.config("c3")
    soup = cfg.make_soup()
    assert soup.n_polys == 12_500_000
    idx = fastmap.build_index(soup, device=0)
    st = idx.stats()
    assert st["cells_boundary"] > 0.3 * st["nx"] * st["ny"] and st["cells_split"] > 0
    rng = np.random.default_rng(3)
    clustered = cfg.make_points(4_000_000, soup=soup, offset=123_456_789)
    uniform = np.stack([rng.uniform(-125.3, -65.7, 1_000_000), rng.uniform(23.87, 50.13, 1_000_000)], 1)
    near = margin_cases.near_edge_points(soup, 500_000, st["cell_w"], seed=3)
    pts = np.ascontiguousarray(np.concatenate([clustered, uniform, near]))
    want = oracle.assign(soup, pts)
    d = torch.from_numpy(pts).to("cuda:0")
    for path in ("stream", "binned"):
        idx.set_query_path(path)
        out = idx.project(d)
        torch.cuda.synchronize()
        got = out.cpu().numpy()
        assert int((got != want).sum()) == 0, path
    assert (want >= 0).mean() > 0.8 and (want == -1).sum() > 0
    idx.close()
