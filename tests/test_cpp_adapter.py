"""The C++ drop-in adapter (include/fastmap_b200/fastmap_gpu.hpp), compiled
against the reference's own headers (oracle/_ref/adapter_check, built by
`make ref` where /root/reference exists)."""
import pathlib
import subprocess

import pytest

BIN = pathlib.Path(__file__).resolve().parent.parent / "oracle" / "_ref" / "adapter_check"
needs_bin = pytest.mark.skipif(not BIN.exists(), reason="adapter_check not built (make ref)")


@needs_bin
def test_adapter_no_gpu_behaviour():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("checks the no-GPU behaviour")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "OK (no GPU)" in r.stdout, r.stdout + r.stderr


@needs_bin
@pytest.mark.gpu
def test_adapter_query_equals_reference_exhaustive_assign():
    r = subprocess.run([str(BIN), "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.startswith("OK"), r.stdout + r.stderr
