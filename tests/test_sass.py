"""SASS checks on the shipped library: the fp64 crossing predicate must
never be contracted into DFMA (SURVEY.md sec. 0 finding 1), and the
record staging must use the async-copy path (LDGSTS)."""
import re
import subprocess

import pytest

from paper_2005_03156_b200 import _native as N


@pytest.fixture(scope="module")
def sass():
    out = subprocess.run(["cuobjdump", "-sass", str(N.PRODUCT_SO)], capture_output=True, text=True)
    assert out.returncode == 0, out.stderr
    return out.stdout


def functions(sass):
    parts = re.split(r"\n\s*Function : ", sass)
    return {p.split("\n", 1)[0].strip(): p for p in parts[1:]}


def test_no_dfma_on_the_query_path(sass):
    """The query kernels evaluate the reference predicate: no DFMA at all.
    (The GPU index builder's contrib_kernel contains DFMA only inside the
    IEEE-correctly-rounded fp64 division sequence (div.rn.f64); its results
    are checked byte-for-byte against the host builder in
    tests/test_gpu_build.py.)"""
    fns = functions(sass)
    query = {n: b for n, b in fns.items() if "stream_kernel" in n or "resolve_kernel" in n
             or "resolve_slot_global" in n or "resolve_wide" in n or "resolve_compact" in n}
    assert query, "query kernels not found"
    for n, b in query.items():
        assert "DFMA" not in b, n
    for n, b in fns.items():
        if "DFMA" in b:
            assert "index_gpu" in n and "contrib_kernel" in n, f"unexpected DFMA in {n}"


def test_kernels_present_and_use_fp64_and_async_copy(sass):
    fns = functions(sass)
    names = " ".join(fns)
    assert "stream_kernel" in names and "resolve_kernel" in names
    resolve = [b for n, b in fns.items() if "resolve_kernel" in n]
    assert any("LDGSTS" in b for b in resolve)
    assert any("DMUL" in b and "DADD" in b for b in resolve)
