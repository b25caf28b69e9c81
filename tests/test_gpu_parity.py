"""GPU parity: the sm_100a projection (through the C-ABI) against the CPU
oracle, bit-exact, on the BASELINE configs and on edge cases."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap, synth  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch.device("cuda:0")


def project_device(idx, pts, dev):
    d = torch.from_numpy(np.ascontiguousarray(pts)).to(dev)
    out = idx.project(d)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def test_c1_full_million_points_bit_exact(dev):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points()
    idx = fastmap.build_index(soup, device=0)
    got = project_device(idx, pts, dev)
    want = oracle.assign(soup, pts)
    assert np.array_equal(got, want)
    assert (want >= 0).mean() > 0.97 and (want == -1).sum() > 0


@pytest.mark.parametrize("name,n", [("c2", 2_000_000), ("c4", 1_000_000)])
def test_large_configs_sampled_bit_exact(dev, name, n):
    cfg = synth.config(name)
    soup = cfg.make_soup()
    pts = cfg.make_points(n, soup=soup)
    idx = fastmap.build_index(soup, device=0)
    got = project_device(idx, pts, dev)
    want = oracle.assign(soup, pts)
    assert int((got != want).sum()) == 0


def test_host_path_and_histogram(dev):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points(300_000, offset=5_000_000)
    idx = fastmap.build_index(soup, device=0)
    hist = np.zeros(soup.n_polys, dtype=np.int64)
    got = idx.project(pts, hist=hist)
    want = oracle.assign(soup, pts)
    assert np.array_equal(got, want)
    assert np.array_equal(hist, np.bincount(want[want >= 0], minlength=soup.n_polys))
    # device histogram accumulates
    dh = torch.zeros(soup.n_polys, dtype=torch.int64, device=dev)
    d = torch.from_numpy(pts).to(dev)
    idx.project(d, hist=dh)
    idx.project(d, hist=dh)
    torch.cuda.synchronize()
    assert np.array_equal(dh.cpu().numpy(), 2 * hist)


def test_counters(dev):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points(100_000)
    idx = fastmap.build_index(soup, device=0)
    c = torch.zeros(4, dtype=torch.int64, device=dev)
    d = torch.from_numpy(pts).to(dev)
    out = idx.project(d, counters=c)
    torch.cuda.synchronize()
    c = c.cpu().numpy()
    assert c[0] == len(pts) and 0 < c[1] < len(pts) and c[2] >= c[1]
    assert np.array_equal(out.cpu().numpy(), oracle.assign(soup, pts))


def test_edge_cases_bit_exact(dev):
    import edge_cases
    soup, pts = edge_cases.build()
    idx = fastmap.build_index(soup, device=0)
    got = project_device(idx, pts, dev)
    want = oracle.exhaustive_assign(soup, pts)
    assert np.array_equal(got, want)


def test_empty_and_tiny_inputs(dev):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, device=0)
    empty = torch.zeros((0, 2), dtype=torch.float64, device=dev)
    assert idx.project(empty).numel() == 0
    one = np.array([[-100.0, 35.0]])
    assert np.array_equal(project_device(idx, one, dev), oracle.assign(soup, one))
    # no polygons at all: everything is -1
    none = fastmap.Soup.from_rings([])
    idx0 = fastmap.build_index(none, device=0)
    pts = cfg.make_points(1000)
    assert (project_device(idx0, pts, dev) == -1).all()


def test_folded_query_grid_odd_dims(dev):
    """The query-side 2x2 fold of the grid (KParams.blocks/sub) at odd grid
    dimensions (partial edge blocks) gives the flat grid's answers."""
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, fastmap.CoverParams(nx=4097, ny=2049), device=0)
    st = idx.stats()
    assert st["query_block_log2"] == 1 and st["query_grid_bytes"] < st["grid_bytes"]
    pts = cfg.make_points(1_000_000, offset=77)
    assert np.array_equal(project_device(idx, pts, dev), oracle.assign(soup, pts))
    c2 = fastmap.build_index(synth.config("c2").make_soup(), device=0).stats()
    assert c2["query_block_log2"] >= 1


def test_more_than_one_launch_slice(dev):
    """fm_query splits batches into 2^28-point slices (queue scratch bound):
    a batch just past the slice size must match point for point, histogram
    included."""
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, device=0)
    n = (1 << 28) + 4099
    base = cfg.make_points(1 << 20, offset=11)
    d = torch.from_numpy(base).to(dev).repeat((n + base.shape[0] - 1) // base.shape[0], 1)[:n].contiguous()
    hist = torch.zeros(soup.n_polys, dtype=torch.int64, device=dev)
    out = idx.project(d, hist=hist)
    torch.cuda.synchronize()
    want = oracle.assign(soup, base)
    got = out.cpu().numpy()
    reps = np.arange(n) % base.shape[0]
    assert np.array_equal(got, want[reps])
    assert np.array_equal(hist.cpu().numpy(), np.bincount(got[got >= 0], minlength=soup.n_polys))
    del d, out


def test_concurrent_streams_share_an_index(dev):
    """Built indexes are immutable; fm_query on two streams at once gives the
    same answers as one after the other (SURVEY.md sec. 8b threading)."""
    cfg = synth.config("c2")
    soup = cfg.make_soup()
    idx = fastmap.build_index(soup, device=0)
    a = torch.from_numpy(cfg.make_points(3_000_000, offset=1)).to(dev)
    b = torch.from_numpy(cfg.make_points(3_000_000, offset=2)).to(dev)
    ra, rb = idx.project(a), idx.project(b)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    oa = torch.empty_like(ra)
    ob = torch.empty_like(rb)
    for _ in range(3):
        with torch.cuda.stream(s1):
            idx.project(a, out=oa, stream=s1)
        with torch.cuda.stream(s2):
            idx.project(b, out=ob, stream=s2)
    torch.cuda.synchronize()
    assert torch.equal(oa, ra) and torch.equal(ob, rb)


def test_histogram_shared_across_streams_and_host_chunks(dev):
    """The per-launch u32 counters are folded into the caller's int64
    histogram atomically: host-path chunks on 3 streams, and device queries
    on 4 concurrent streams into one histogram, lose no counts."""
    cfg = synth.config("c2")
    soup = cfg.make_soup()
    pts = cfg.make_points(30_000_000, soup=soup, offset=77)  # 4 host chunks of 8M points
    idx = fastmap.build_index(soup, device=0)
    hist = np.zeros(soup.n_polys, dtype=np.int64)
    got = idx.project(pts, hist=hist)
    assert np.array_equal(hist, np.bincount(got[got >= 0], minlength=soup.n_polys))
    d = torch.from_numpy(pts).to(dev)
    dh = torch.zeros(soup.n_polys, dtype=torch.int64, device=dev)
    outs, streams = [], [torch.cuda.Stream(dev) for _ in range(4)]
    torch.cuda.synchronize()
    for k, s in enumerate(streams):
        with torch.cuda.stream(s):
            outs.append(idx.project(d[k * 7_000_000:(k + 1) * 7_000_000], hist=dh, stream=s.cuda_stream))
    torch.cuda.synchronize()
    allout = torch.cat(outs).cpu().numpy()
    assert np.array_equal(allout, got[:28_000_000])
    assert np.array_equal(dh.cpu().numpy(), np.bincount(allout[allout >= 0], minlength=soup.n_polys))


def test_invariance_under_ring_rotation_and_power_of_two_translation(dev):
    """test_geometry.cpp:145-184 through the GPU index: a soup of random
    star polygons, the same soup with every ring's start rotated, and the
    soup plus points translated by (64, -32) give identical answers (the
    translated points off the edges by > 1e-9, as the reference requires)."""
    rng = np.random.default_rng(17)
    rings = []
    for k in range(60):
        c = rng.uniform(-20, 20, 2)
        n = int(rng.integers(5, 40))
        a = np.sort(rng.random(n)) * 2 * np.pi
        r = rng.uniform(0.5, 2.0, n)
        rings.append(np.stack([c[0] + r * np.cos(a), c[1] + r * np.sin(a)], 1))
    pts = rng.uniform(-23, 23, (200_000, 2))
    base_soup = fastmap.Soup.from_rings([[r] for r in rings])
    want = oracle.assign(base_soup, pts)
    got = project_device(fastmap.build_index(base_soup, device=0), pts, dev)
    assert np.array_equal(got, want)
    rot = fastmap.Soup.from_rings([[np.roll(r, 13 % len(r), axis=0)] for r in rings])
    assert np.array_equal(project_device(fastmap.build_index(rot, device=0), pts, dev), want)
    shift = np.array([64.0, -32.0])
    moved = fastmap.Soup.from_rings([[r + shift] for r in rings])
    far = np.ones(len(pts), dtype=bool)
    for r in rings:  # keep points farther than 1e-9 from every edge
        a, b = r, np.roll(r, -1, axis=0)
        for j in range(len(r)):
            d = b[j] - a[j]
            t = np.clip(((pts - a[j]) @ d) / (d @ d), 0, 1)
            far &= np.hypot(*(pts - (a[j] + t[:, None] * d)).T) > 1e-9
    moved_got = project_device(fastmap.build_index(moved, device=0), pts + shift, dev)
    assert np.array_equal(moved_got[far], want[far])
