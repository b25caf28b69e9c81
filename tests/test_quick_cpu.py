"""Quick records (csrc/quick.h), checked on the CPU: fm_index_quick_host
runs the kernel's own quick_encode / quick_eval code on a host-only index,
and every answer it certifies must equal the oracle's bit for bit; only
FM_QUICK_UNSURE / FM_QUICK_NONE points may go the exact way."""
import ctypes as C

import numpy as np
import pytest

import edge_cases
import oracle
from paper_2005_03156_b200 import _native as N
from paper_2005_03156_b200 import fastmap, synth

UNSURE, NONE = -3, -4


def quick(soup, pts, **params):
    idx = fastmap.build_index(soup, fastmap.CoverParams(**params), device=-1)
    pts = np.ascontiguousarray(pts, dtype=np.float64)
    out = np.empty(len(pts), dtype=np.int32)
    N.check(N.lib().fm_index_quick_host(idx.handle, N.ptr(pts, C.c_double), len(pts),
                                        N.ptr(out, C.c_int32)), "fm_index_quick_host")
    return out


def near_edge_points(soup, n, seed, scales=(0.0, 1e-13, 1e-10, 1e-7, 1e-5, 1e-3)):
    """Points on and very near random polygon edges (perpendicular offsets
    of the given sizes in degrees, both signs) and exactly on vertices."""
    rng = np.random.default_rng(seed)
    v = soup.vxy
    ro = soup.ring_off.astype(np.int64)
    ring = rng.integers(0, len(ro) - 1, n)
    a = ro[ring] + (rng.integers(0, 1 << 30, n) % (ro[ring + 1] - ro[ring]))
    b = np.where(a + 1 < ro[ring + 1], a + 1, ro[ring])
    t = rng.random(n)
    p = v[a] + t[:, None] * (v[b] - v[a])
    d = v[b] - v[a]
    nrm = np.stack([-d[:, 1], d[:, 0]], 1) / np.maximum(np.hypot(d[:, 0], d[:, 1]), 1e-300)[:, None]
    s = np.asarray(scales)[rng.integers(0, len(scales), n)] * rng.choice([-1.0, 1.0], n)
    p = p + s[:, None] * nrm
    k = n // 10
    p[:k] = v[a[:k]]  # exactly on vertices
    return p


def check(soup, pts, **params):
    got = quick(soup, pts, **params)
    want = oracle.assign(soup, pts)
    sure = got >= -1
    bad = np.flatnonzero(sure & (got != want))
    assert bad.size == 0, (bad[:10], got[bad[:10]], want[bad[:10]], pts[bad[:10]])
    return got


@pytest.mark.parametrize("m,min_sure", [(0.0, 0.9), (8.0, 0.9), (4.0, 0.75)])
def test_c1_quick_answers_match_oracle(m, min_sure):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = cfg.make_points(200_000, offset=4242)
    got = check(soup, pts, cells_per_polygon=m)
    # a certified answer for nearly every point
    assert (got == UNSURE).mean() < 2e-3
    assert (got >= -1).mean() > min_sure


@pytest.mark.parametrize("m", [0.0, 8.0])
def test_c1_near_edge_points(m):
    cfg = synth.config("c1")
    soup = cfg.make_soup()
    pts = near_edge_points(soup, 100_000, seed=7)
    got = check(soup, pts, cells_per_polygon=m)
    # points within ~1e-7 deg of an edge cannot be certified; farther ones are
    assert (got == UNSURE).mean() < 0.8
    assert (got >= -1).sum() > 1_000


@pytest.mark.parametrize("name,m", [("c2", 8.0), ("c4", 12.0), ("c3mini", 16.0)])
def test_large_configs_quick_sampled(name, m):
    cfg = synth.config(name)
    soup = cfg.make_soup()
    pts = np.concatenate([cfg.make_points(20_000, soup=soup, offset=99),
                          near_edge_points(soup, 10_000, seed=3)])
    check(soup, pts, cells_per_polygon=m)


@pytest.mark.parametrize("grid", [(1, 1), (7, 5), (97, 13), (400, 300)])
def test_edge_cases_quick(grid):
    soup, pts = edge_cases.build()
    got = quick(soup, pts, nx=grid[0], ny=grid[1])
    want = oracle.exhaustive_assign(soup, pts)
    sure = got >= -1
    assert np.array_equal(got[sure], want[sure])


def test_quick_needs_host_index():
    soup = fastmap.Soup.from_rings([[[(0, 0), (1, 0), (1, 1), (0, 1)]]])
    pts = np.zeros((1, 2))
    out = np.empty(1, dtype=np.int32)
    idx = fastmap.build_index(soup, device=-1)
    assert N.lib().fm_index_quick_host(idx.handle, N.ptr(pts, C.c_double), 1,
                                       N.ptr(out, C.c_int32)) == 0
