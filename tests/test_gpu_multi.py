"""The multi-GPU C-ABI entry (fm_multi_*; run_chunked one level up,
parallel.hpp:30-82) on the devices of this box: replicas built per device,
the host batch sharded contiguously, the per-block histogram summed with
ncclAllReduce.  The driver's boxes have one GPU, so this runs with N = 1
(NCCL communicator of one rank) -- the shard arithmetic for N > 1 is
covered on CPU by tests/test_parallel_cpu.py (shard_range)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap, synth  # noqa: E402


def test_multi_index_shards_and_reduces_histogram():
    cfg = synth.config("c2")
    soup = cfg.make_soup()
    devs = list(range(torch.cuda.device_count()))
    mi = fastmap.MultiIndex(soup, devs)
    assert len(mi) == len(devs)
    pts = cfg.make_points(20_000_003, soup=soup, offset=99)  # odd size: ragged shards
    hist = np.zeros(soup.n_polys, dtype=np.int64)
    got = mi.project(pts, hist=hist)
    sample = np.random.default_rng(0).choice(len(pts), 2_000_000, replace=False)
    want = oracle.assign(soup, pts[sample])
    assert np.array_equal(got[sample], want)
    assert np.array_equal(hist, np.bincount(got[got >= 0], minlength=soup.n_polys))
    # the histogram accumulates; the ids equal the single-index host path
    mi.project(pts[:1000], hist=hist)
    single = fastmap.build_index(soup, device=0)
    assert np.array_equal(single.project(pts[:5_000_000]), got[:5_000_000])
    assert hist.sum() == (got >= 0).sum() + (got[:1000] >= 0).sum()
    mi.close()


def test_multi_index_rejects_duplicate_devices():
    soup = synth.config("c1").make_soup()
    with pytest.raises(ValueError, match="distinct"):
        fastmap.MultiIndex(soup, [0, 0])
    with pytest.raises(ValueError, match="out of range"):
        fastmap.MultiIndex(soup, [torch.cuda.device_count()])
