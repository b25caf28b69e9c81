"""The C-ABI library: loads, exports every symbol include/fastmap_b200.h
declares, and fails loudly (no CPU fallback) where no GPU is present."""
import ctypes as C
import pathlib
import re
import subprocess

import numpy as np
import pytest
import torch

from paper_2005_03156_b200 import _native as N
from paper_2005_03156_b200 import fastmap, synth

ROOT = pathlib.Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "fastmap_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(fm_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_what_python_binds():
    assert declared_symbols() == sorted(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    nm = subprocess.run(["nm", "-D", "--defined-only", str(N.PRODUCT_SO)],
                        capture_output=True, text=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}\b", nm), f"{name} not exported"


def test_status_strings_and_version():
    lib = N.lib()
    assert lib.fm_status_string(0) == b"ok"
    assert lib.fm_status_string(5) == b"no CUDA device"
    assert b"sm_100a" in lib.fm_version()


def test_library_is_built_for_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.PRODUCT_SO)],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback_without_gpu():
    soup = synth.config("c1").make_soup()
    with pytest.raises(RuntimeError, match="no CUDA device"):
        fastmap.build_index(soup, device=0)
    idx = fastmap.build_index(soup, device=-1)  # host-only index: inspectable, not queryable
    with pytest.raises(RuntimeError, match="host-only"):
        idx.project(np.zeros((4, 2)))


def test_error_mapping_matches_reference_exceptions():
    bad_ring = fastmap.Soup.from_rings([[[(0, 0), (1, 0)]]])
    with pytest.raises(ValueError, match="at least 3 vertices"):  # geometry.hpp:75-77
        fastmap.build_index(bad_ring, device=-1)
    nan = fastmap.Soup.from_rings([[[(0, 0), (1, 0), (np.nan, 1)]]])
    with pytest.raises(ValueError, match="non-finite"):
        fastmap.build_index(nan, device=-1)
    with pytest.raises(ValueError, match="max_level"):  # cell_index.hpp:383-385
        fastmap.build_index(bad_ring, fastmap.CoverParams(max_level=31), device=-1)
    with pytest.raises(ValueError, match="level-30"):  # cell_index.hpp:386-392
        fastmap.validate_cover_params(fastmap.CoverParams(mode=fastmap.CoverMode.approx,
                                                          epsilon=1e-9))
    idx = fastmap.build_index(synth.config("c1").make_soup(), device=-1)
    with pytest.raises(ValueError, match="fanout"):  # cell_index.hpp:454-456
        fastmap.build_trie(idx, 3)
    trie = fastmap.build_trie(idx, 4)
    with pytest.raises(ValueError, match="different hierarchy"):  # cell_index.hpp:536-538
        fastmap.query_leaves(trie, fastmap.Soup.from_rings([[[(0, 0), (1, 0), (1, 1)]]]),
                             np.zeros((1, 2)))
    with pytest.raises(ValueError, match="approximate-mode cover"):  # cell_index.hpp:532-535
        fastmap.query_leaves(trie, synth.config("c1").make_soup(), np.zeros((1, 2)),
                             fastmap.CoverMode.approx)


def test_approx_cover_params_and_resolution():
    """fast-approx covers: the C-ABI validates epsilon like
    validate_cover_params (cell_index.hpp:386-392) and refines the grid until
    every margin-expanded cell diagonal is <= epsilon (cell_index.hpp:313-316)."""
    soup = synth.config("c1").make_soup().contiguous()
    bp = N.BuildParams(device=-1, build_on_gpu=0, approx_epsilon=1e-9)
    h = C.c_void_p()
    st = N.lib().fm_index_build(N.ptr(soup.vxy, C.c_double), N.ptr(soup.ring_off, C.c_uint64),
                                soup.n_rings, N.ptr(soup.poly_ring, C.c_uint64), soup.n_polys,
                                C.byref(bp), C.byref(h))
    assert st == 1 and b"level-30" in N.lib().fm_last_error()
    eps = 0.03
    P = fastmap.CoverParams(mode=fastmap.CoverMode.approx, epsilon=eps)
    idx = fastmap.build_index(soup, P, device=-1)
    s = idx.stats()
    assert s["approx_epsilon"] == eps
    assert np.hypot(s["cell_w"] + 2 * s["margin"], s["cell_h"] + 2 * s["margin"]) <= eps
    assert np.hypot(2 * s["cell_w"], 2 * s["cell_h"]) > eps  # not needlessly fine
    # an explicit resolution is only ever raised to meet epsilon
    fine = fastmap.build_index(soup, fastmap.CoverParams(mode=fastmap.CoverMode.approx, epsilon=eps,
                                                         nx=5000, ny=300), device=-1).stats()
    assert fine["nx"] == 5000 and fine["ny"] == s["ny"]
    # an epsilon finer than a 2^31-cell uniform grid resolves: the exact grid,
    # approximate queries answered exactly (error 0 <= epsilon)
    tiny = fastmap.build_index(soup, fastmap.CoverParams(mode=fastmap.CoverMode.approx,
                                                         epsilon=1e-6), device=-1).stats()
    exact = fastmap.build_index(soup, device=-1).stats()
    assert tiny["approx_epsilon"] == 1e-6 and (tiny["nx"], tiny["ny"]) == (exact["nx"], exact["ny"])


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure")
def test_multi_gpu_entry_fails_loudly_without_a_device():
    soup = synth.config("c1").make_soup()
    with pytest.raises(RuntimeError, match="no CUDA device"):
        fastmap.MultiIndex(soup, [0])
    with pytest.raises(ValueError):
        fastmap.MultiIndex(soup, [])
