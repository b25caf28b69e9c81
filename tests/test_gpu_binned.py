"""GPU parity of the binned query path (csrc/binned.cuh, fm_query_path):
points partitioned by index tile, queried tile by tile and gathered back.
Every answer must equal the oracle's -- and the stream path's -- bit for
bit, whatever the tile size, batch shape or output alignment."""
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


def run(idx, pts, dev, path, hist=None, counters=None):
    idx.set_query_path(path)
    d = torch.from_numpy(np.ascontiguousarray(pts)).to(dev)
    out = idx.project(d, hist=hist, counters=counters)
    torch.cuda.synchronize()
    return out.cpu().numpy()


@pytest.mark.parametrize("name,n", [("c1", 1_000_000), ("c2", 3_000_000), ("c4", 2_000_000),
                                    ("c3mini", 2_000_000)])
def test_binned_equals_oracle_and_stream(dev, name, n):
    cfg = synth.config(name)
    soup = cfg.make_soup()
    pts = cfg.make_points(n, soup=soup)
    idx = fastmap.build_index(soup, device=0)
    want = oracle.assign(soup, pts)
    got_b = run(idx, pts, dev, "binned")
    assert int((got_b != want).sum()) == 0
    got_s = run(idx, pts, dev, "stream")
    assert np.array_equal(got_s, got_b)
    assert idx.query_plan(n)["n_tiles"] >= 1


@pytest.mark.parametrize("tile_bytes", [1e3, 2e5, 5e6, 1e9])
def test_binned_tile_sizes(dev, tile_bytes):
    """From thousands of tiny tiles (capped at 4096) to a single tile."""
    cfg = synth.config("c4")
    soup = cfg.make_soup()
    pts = cfg.make_points(1_500_000, soup=soup, offset=3)
    idx = fastmap.build_index(soup, device=0)
    idx.set_query_path("binned", tile_bytes)
    plan = idx.query_plan(len(pts))
    assert plan["path"] == "binned" and 1 <= plan["n_tiles"] <= 4096
    d = torch.from_numpy(pts).to(dev)
    got = idx.project(d).cpu().numpy()
    assert int((got != oracle.assign(soup, pts)).sum()) == 0


def test_binned_edge_cases_nan_and_outside(dev):
    """The adversarial soup (holes, bow-ties, overlaps, on-vertex and on-edge
    points, NaN/Inf, out-of-world points) through the binned path."""
    import edge_cases
    soup, pts = edge_cases.build()
    idx = fastmap.build_index(soup, device=0)
    idx.set_query_path("binned", 1e3)
    reps = np.concatenate([pts] * 50)  # several chunks, many per tile
    got = run(idx, reps, dev, "binned")
    want = oracle.exhaustive_assign(soup, pts)
    assert np.array_equal(got, np.concatenate([want] * 50))


def test_binned_histogram_counters_and_unaligned_output(dev):
    cfg = synth.config("c3mini")
    soup = cfg.make_soup()
    n = 1_000_003  # not a multiple of 4: the gather's scalar tail
    pts = cfg.make_points(n, offset=9)
    idx = fastmap.build_index(soup, device=0)
    want = oracle.assign(soup, pts)
    hist = torch.zeros(soup.n_polys, dtype=torch.int64, device=dev)
    cnt_b = torch.zeros(4, dtype=torch.int64, device=dev)
    got = run(idx, pts, dev, "binned", hist=hist, counters=cnt_b)
    assert np.array_equal(got, want)
    assert np.array_equal(hist.cpu().numpy(), np.bincount(want[want >= 0], minlength=soup.n_polys))
    cnt_s = torch.zeros(4, dtype=torch.int64, device=dev)
    run(idx, pts, dev, "stream", counters=cnt_s)
    # the same work, whatever the order: points, boundary points, candidates, edge tests
    assert np.array_equal(cnt_b.cpu().numpy(), cnt_s.cpu().numpy())
    assert cnt_b[0].item() == n
    # output at an address that is not 16-byte aligned (the gather's scalar path)
    d = torch.from_numpy(pts).to(dev)
    buf = torch.full((n + 1,), -7, dtype=torch.int32, device=dev)
    idx.project(d, out=buf[1:])
    torch.cuda.synchronize()
    assert buf[0].item() == -7 and np.array_equal(buf[1:].cpu().numpy(), want)


def test_auto_path_choice_follows_index_statistics(dev):
    """Auto picks binned for big, mostly-boundary indexes and big batches
    (c3, c4), never for small or mostly true-hit indexes (c1, c2)."""
    c2 = fastmap.build_index(synth.config("c2").make_soup(), device=0)
    assert c2.query_plan(100_000_000)["path"] == "stream"       # 9% boundary cells
    c4 = fastmap.build_index(synth.config("c4").make_soup(), device=0)
    assert c4.query_plan(1000)["path"] == "stream"              # batch too small to reuse tiles
    assert c4.query_plan(200_000_000)["path"] == "binned"       # 6 GB index, 50% boundary cells
    c4.set_query_path("binned")
    assert c4.query_plan(1000)["path"] == "binned"
    c1 = fastmap.build_index(synth.config("c1").make_soup(), device=0)
    assert c1.query_plan(100_000_000)["path"] == "stream"       # L2-sized index
    with pytest.raises(ValueError):
        c1.set_query_path("binned", -1.0)


@pytest.mark.parametrize("name", ["c1", "c2", "c4", "c3mini"])
def test_device_point_streams_equal_host_streams(dev, name):
    """The GPU generator (csrc/synth_gpu.cu) writes the host generator's
    bits for every point index (shared synth_rng.h, no FMA either side)."""
    cfg = synth.config(name)
    soup = cfg.make_soup() if name == "c4" else None
    for off, n in ((0, 100_000), (123_456_789, 50_001)):
        want = cfg.make_points(n, offset=off, soup=soup)
        got = torch.empty((n, 2), dtype=torch.float64, device=dev)
        cfg.make_points_device(got, offset=off, soup=soup)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy(), want)


def _stratum_offsets(n, stride=64):
    """Index of the sampled point of every stratum (binned.cuh stratum_hash)."""
    j = np.arange((n + stride - 1) // stride, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = j * np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(31))) * np.uint64(0xBF58476D1CE4E5B9)
    h = (z >> np.uint64(40)).astype(np.int64)
    lo = j.astype(np.int64) * stride
    w = np.minimum(stride, n - lo)
    return lo + h % w


def test_binned_sample_blind_stream_overflows_and_unplaced(dev):
    """A stream built against the capacity sample: every sampled point is
    spread over the domain, every other point sits in one small box, so that
    box's bin is planned nearly empty.  Its points fill the bin, then the
    overflow bin, and the rest are answered by unplaced_kernel -- ids,
    histogram and counters must still equal the oracle's and the stream
    path's."""
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    n = 2_000_000
    spread = cfg.make_points(n, offset=5)
    rng = np.random.default_rng(3)
    box = np.column_stack([rng.uniform(-96.0, -95.2, n), rng.uniform(36.0, 36.6, n)])
    pts = box.copy()
    s = _stratum_offsets(n)
    pts[s] = spread[s]
    idx = fastmap.build_index(soup, device=0)
    idx.set_query_path("binned", 2e5)
    assert idx.query_plan(n)["n_tiles"] > 16
    want = oracle.assign(soup, pts)
    hist = torch.zeros(soup.n_polys, dtype=torch.int64, device=dev)
    cnt_b = torch.zeros(4, dtype=torch.int64, device=dev)
    got = run(idx, pts, dev, "binned", hist=hist, counters=cnt_b)
    assert int((got != want).sum()) == 0
    assert np.array_equal(hist.cpu().numpy(), np.bincount(want[want >= 0], minlength=soup.n_polys))
    cnt_s = torch.zeros(4, dtype=torch.int64, device=dev)
    run(idx, pts, dev, "stream", counters=cnt_s)
    assert np.array_equal(cnt_b.cpu().numpy(), cnt_s.cpu().numpy())
    assert cnt_b[0].item() == n
