"""Fast-approx mode (CoverMode::approx, cell_index.hpp:558-560) on the GPU,
checked the way the reference checks it (test_cell_index.cpp:381-435,
acceptance.cpp:220-253): zero crossing tests, every disagreement with the
exact answer has a deemed leaf within epsilon of the point
(tests/oracles.hpp:92-95 distance), exact queries on the approx cover stay
exact, and approx queries on an exact-only cover raise."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2005_03156_b200 import _native as N, fastmap, synth  # noqa: E402
from paper_2005_03156_b200.fastmap import CoverMode, CoverParams  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def check_approx(soup, pts, got, want, eps, max_checks=4000):
    dis = np.nonzero(got != want)[0]
    assert (got[dis] >= 0).all(), "a disagreement without a deemed leaf"
    rng = np.random.default_rng(0)
    sample = dis if dis.size <= max_checks else rng.choice(dis, max_checks, replace=False)
    worst = 0.0
    for i in sample:
        d = oracle.point_polygon_distance(soup, int(got[i]), float(pts[i, 0]), float(pts[i, 1]))
        worst = max(worst, d)
    assert worst <= eps, worst
    return dis.size, worst


@pytest.mark.parametrize("name,eps,n", [("c1", 0.02, 1_000_000), ("c3mini", 0.02, 500_000),
                                        ("c4", 0.05, 300_000),
                                        # fine grid > 48 MB: two-level covers with 4x4
                                        # and 8x8 blocks (palette + full sub-blocks)
                                        ("c1", 0.005, 1_000_000), ("c1", 0.0025, 1_000_000)])
def test_approx_error_bound_and_zero_tests(dev, name, eps, n):
    cfg = synth.config(name)
    soup = cfg.make_soup()
    pts = cfg.make_points(n, soup=soup) if name == "c4" else cfg.make_points(n)
    idx = fastmap.build_index(soup, CoverParams(mode=CoverMode.approx, epsilon=eps), device=0)
    st = idx.stats()
    assert st["approx_epsilon"] == eps and st["approx_grid_bytes"] > 0
    if st["grid_bytes"] > 48 << 20:
        assert st["approx_grid_bytes"] < st["grid_bytes"] and st["approx_block_log2"] >= 2
    assert np.hypot(st["cell_w"] + 2 * st["margin"], st["cell_h"] + 2 * st["margin"]) <= eps
    want = oracle.assign(soup, pts)
    d = torch.from_numpy(pts).to(dev)
    ctr = torch.zeros(4, dtype=torch.int64, device=dev)
    got = idx.project(d, counters=ctr, mode=CoverMode.approx).cpu().numpy()
    c = ctr.cpu().numpy()
    assert c[0] == n and c[2] == 0 and c[3] == 0  # no candidate or crossing tests
    n_dis, worst = check_approx(soup, pts, got, want, eps)
    if name != "c4":  # c4 puts half its points within 1e-4 cells of an edge
        assert n_dis < 0.05 * n
    # the host path gives the same answers
    assert np.array_equal(idx.project(pts, mode=CoverMode.approx), got)
    # an exact query against the approximate cover is exact
    assert np.array_equal(idx.project(d).cpu().numpy(), want)


def test_approx_histogram_and_edge_points(dev):
    import edge_cases
    soup, pts = edge_cases.build()
    idx = fastmap.build_index(soup, CoverParams(mode=CoverMode.approx, epsilon=0.05), device=0)
    got = idx.project(pts, mode=CoverMode.approx)
    want = oracle.assign(soup, pts)
    outside = ~((np.abs(pts[:, 0]) <= 180) & (np.abs(pts[:, 1]) <= 90))  # incl. NaN
    assert (got[outside] == -1).all()
    check_approx(soup, pts, got, want, 0.05)
    hist = torch.zeros(soup.n_polys, dtype=torch.int64, device=dev)
    g2 = idx.project(torch.from_numpy(pts).to(dev), hist=hist, mode=CoverMode.approx)
    assert np.array_equal(g2.cpu().numpy(), got)
    assert np.array_equal(hist.cpu().numpy(), np.bincount(got[got >= 0], minlength=soup.n_polys))


def test_approx_query_on_exact_cover_raises(dev):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, device=0)
    pts = cfg.make_points(1000)
    with pytest.raises(ValueError, match="approximate-mode cover"):
        idx.project(pts, mode=CoverMode.approx)
    with pytest.raises(ValueError, match="approximate-mode cover"):
        fastmap.query_leaves(idx, soup, pts, CoverMode.approx)
    res = fastmap.query_leaves(fastmap.build_index(
        soup, CoverParams(mode=CoverMode.approx, epsilon=0.05), device=0), soup, pts,
        CoverMode.approx)
    assert res.size() == 1000


def test_query_mode_rejects_unknown_mode(dev):
    cfg = synth.config("c1")
    idx = fastmap.build_index(cfg.make_soup(), device=0)
    pts = cfg.make_points(10)
    out = np.empty(10, dtype=np.int32)
    st = N.lib().fm_query_host_mode(idx.handle, 7, N.ptr(pts, N.C.c_double), 10,
                                    N.ptr(out, N.C.c_int32), None)
    assert st == 1


def test_approx_epsilon_finer_than_the_uniform_grid_is_served_exactly(dev, tmp_path):
    """epsilon = 1e-6 would need > 2^31 uniform approx cells over c1's extent:
    the index is the exact one and approximate queries return the exact
    answers (error 0 <= epsilon, the reference's bound,
    test_cell_index.cpp:381-435); the choice survives save / load."""
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points(500_000, offset=31)
    idx = fastmap.build_index(soup, CoverParams(mode=CoverMode.approx, epsilon=1e-6), device=0)
    st = idx.stats()
    assert st["approx_epsilon"] == 1e-6 and st["approx_grid_bytes"] == 0
    want = oracle.assign(soup, pts)
    d = torch.from_numpy(pts).to(dev)
    assert np.array_equal(idx.project(d, mode=CoverMode.approx).cpu().numpy(), want)
    assert np.array_equal(idx.project(pts, mode=CoverMode.approx), want)
    p = tmp_path / "tiny.fmgi"
    idx.save(p)
    again = fastmap.load_index(p, device=0)
    assert again.stats()["approx_grid_bytes"] == 0
    assert np.array_equal(again.project(pts, mode=CoverMode.approx), want)
