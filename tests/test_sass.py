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


def test_no_dfma_anywhere(sass):
    assert "DFMA" not in sass


def test_kernels_present_and_use_fp64_and_async_copy(sass):
    fns = functions(sass)
    names = " ".join(fns)
    assert "stream_kernel" in names and "resolve_kernel" in names
    resolve = [b for n, b in fns.items() if "resolve_kernel" in n]
    assert any("LDGSTS" in b for b in resolve)
    assert any("DMUL" in b and "DADD" in b for b in resolve)
