"""GeoJSON -> FMCB -> GPU, end to end: boundaries written by the reference's
own write_boundaries are ingested by paper_2005_03156_b200.geojson, then the
exact leaf index and the simple engine run on the B200 and are checked
against the oracle and the reference's assign() on the same FMCB bytes."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
from paper_2005_03156_b200 import fastmap, geojson  # noqa: E402
from test_gpu_simple import check_against_reference, probe_points  # noqa: E402

needs_ref = pytest.mark.skipif(not oracle.ref_geojson_available(),
                               reason="oracle/_ref built without nlohmann json")


@needs_ref
@pytest.mark.parametrize("spec", [(11, 4, 4, 25, 0.2), (12, 3, 5, 7, 0.3)])
def test_geojson_to_gpu_index_and_simple_engine(tmp_path, spec):
    d = tmp_path / "g"
    oracle.ref_write_synthetic_geojson(*spec, d)
    fm = tmp_path / "h.fmcb"
    geojson.ingest(d / "states.geojson", d / "counties.geojson", d / "blocks.geojson", fm)
    h = fastmap.load_hierarchy(fm)
    pts = probe_points(h, 50_000, spec[0])
    idx = fastmap.build_index_hierarchy(h, device=0)
    got = idx.project(torch.from_numpy(pts).cuda()).cpu().numpy()
    assert np.array_equal(got, oracle.exhaustive_assign(h.soup, pts))
    check_against_reference(fm, pts)
