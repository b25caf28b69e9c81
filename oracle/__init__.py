"""CPU oracle for the point-to-block projection -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline
/ reference legs may import this package, and only as the checker (or the
timed reference CPU arm), never as a path that produces product answers.

Two layers:
  * ``liboracle.so`` (oracle/oracle.c): a C restatement of the reference's
    predicate and exhaustive_assign semantics (geometry.hpp:170-225,
    synthetic.hpp:193-205, cell_index.hpp:549-552).
  * ``_ref/libfastmap_ref.so`` (oracle/ref_shim.cpp): the UNMODIFIED
    reference headers compiled here, used to pin the restatement and as the
    reference CPU baseline (query_leaves via run_chunked).
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ORACLE_SO = HERE / "liboracle.so"
REF_SO = HERE / "_ref" / "libfastmap_ref.so"

PD = C.POINTER(C.c_double)
PU64 = C.POINTER(C.c_uint64)
PU32 = C.POINTER(C.c_uint32)
PI32 = C.POINTER(C.c_int32)
PU8 = C.POINTER(C.c_uint8)
u64 = C.c_uint64

_orc = None
_ref = None


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def lib():
    global _orc
    if _orc is None:
        if not ORACLE_SO.exists():
            raise RuntimeError(f"{ORACLE_SO} missing: run `make oracle`")
        L = C.CDLL(str(ORACLE_SO))
        L.orc_point_in_polygon.restype = C.c_int
        L.orc_point_in_polygon.argtypes = [C.c_double, C.c_double, PD, PU64, PU64, u64]
        L.orc_exhaustive_assign.restype = None
        L.orc_exhaustive_assign.argtypes = [PD, PU64, PU64, u64, PD, u64, C.c_int, PI32]
        L.orc_assign.restype = None
        L.orc_assign.argtypes = [PD, PU64, PU64, u64, PD, u64, C.c_int, C.c_int, PI32]
        L.orc_count_containing.restype = None
        L.orc_count_containing.argtypes = [PD, PU64, PU64, u64, PD, u64, PI32]
        L.orc_point_polygon_distance.argtypes = [C.c_double, C.c_double, PD, PU64, PU64, u64]
        L.orc_point_polygon_distance.restype = C.c_double
        _orc = L
    return _orc


def ref_available() -> bool:
    return REF_SO.exists()


def ref():
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            raise RuntimeError(f"{REF_SO} missing: build it with `make ref` where /root/reference exists")
        L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_point_in_polygon.restype = C.c_int
        L.ref_point_in_polygon.argtypes = [C.c_double, C.c_double, PD, PU64, u64]
        L.ref_points_in_polygon.restype = C.c_int
        L.ref_points_in_polygon.argtypes = [PD, u64, PD, PU64, u64, PU8]
        L.ref_model_create.restype = C.c_void_p
        L.ref_model_create.argtypes = [PD, PU64, PU64, u64, PU32]
        L.ref_model_destroy.restype = None
        L.ref_model_destroy.argtypes = [C.c_void_p]
        L.ref_exhaustive_assign.restype = C.c_int
        L.ref_exhaustive_assign.argtypes = [C.c_void_p, PD, u64, PI32]
        L.ref_build_index.restype = C.c_int
        L.ref_build_index.argtypes = [C.c_void_p, C.c_int, C.c_int, PD, PU64, PU64]
        L.ref_query_leaves.restype = C.c_int
        L.ref_query_leaves.argtypes = [C.c_void_p, PD, u64, C.c_uint, u64, PI32, PU64, PD]
        L.ref_generate_synthetic.restype = C.c_int
        L.ref_generate_synthetic.argtypes = [u64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                             PU64, PU64, PU64, PD, PU64, PU64, PU32,
                                             C.c_char_p, PD]
        L.ref_sample.restype = C.c_int
        L.ref_sample.argtypes = [C.c_int, PD, u64, u64, PD]
        L.ref_cell_from_point.restype = C.c_int
        L.ref_save_synthetic_fmcb.argtypes = [u64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                              C.c_char_p]
        L.ref_save_synthetic_fmcb.restype = C.c_int
        L.ref_load_fmcb_status.argtypes = [C.c_char_p]
        L.ref_load_fmcb_status.restype = C.c_int
        L.ref_simple_assign_fmcb.argtypes = [C.c_char_p, PD, u64, C.c_int, PI32, PI32, PI32, PU64]
        L.ref_simple_assign_fmcb.restype = C.c_int
        L.ref_cell_from_point.argtypes = [C.c_double, C.c_double, C.c_int, PU64]
        if hasattr(L, "ref_ingest_geojson"):  # built with nlohmann json on the include path
            L.ref_ingest_geojson.argtypes = [C.c_char_p] * 4
            L.ref_ingest_geojson.restype = C.c_int
            L.ref_write_synthetic_geojson.argtypes = [u64, C.c_uint32, C.c_uint32, C.c_uint32,
                                                      C.c_double, C.c_char_p]
            L.ref_write_synthetic_geojson.restype = C.c_int
        _ref = L
    return _ref


def _soup_arrays(soup):
    vxy = np.ascontiguousarray(soup.vxy, dtype=np.float64)
    ro = np.ascontiguousarray(soup.ring_off, dtype=np.uint64)
    pr = np.ascontiguousarray(soup.poly_ring, dtype=np.uint64)
    return vxy, ro, pr


# -- restatement -------------------------------------------------------------

def point_in_polygon(soup, poly: int, px: float, py: float) -> bool:
    vxy, ro, pr = _soup_arrays(soup)
    return bool(lib().orc_point_in_polygon(px, py, _p(vxy, C.c_double), _p(ro, C.c_uint64),
                                           _p(pr, C.c_uint64), poly))


def exhaustive_assign(soup, pts, world_check: bool = True) -> np.ndarray:
    """O(N * P) restatement of synthetic.hpp:193-205 (small cases only)."""
    vxy, ro, pr = _soup_arrays(soup)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    out = np.empty(pts.shape[0], dtype=np.int32)
    lib().orc_exhaustive_assign(_p(vxy, C.c_double), _p(ro, C.c_uint64), _p(pr, C.c_uint64),
                                soup.n_polys, _p(pts, C.c_double), pts.shape[0],
                                1 if world_check else 0, _p(out, C.c_int32))
    return out


def assign(soup, pts, world_check: bool = True, threads: int = 0) -> np.ndarray:
    """Same answers as exhaustive_assign, bbox-bucketed and threaded."""
    vxy, ro, pr = _soup_arrays(soup)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    out = np.empty(pts.shape[0], dtype=np.int32)
    lib().orc_assign(_p(vxy, C.c_double), _p(ro, C.c_uint64), _p(pr, C.c_uint64),
                     soup.n_polys, _p(pts, C.c_double), pts.shape[0],
                     1 if world_check else 0, threads or (os.cpu_count() or 1),
                     _p(out, C.c_int32))
    return out


def count_containing(soup, pts) -> np.ndarray:
    vxy, ro, pr = _soup_arrays(soup)
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    out = np.empty(pts.shape[0], dtype=np.int32)
    lib().orc_count_containing(_p(vxy, C.c_double), _p(ro, C.c_uint64), _p(pr, C.c_uint64),
                               soup.n_polys, _p(pts, C.c_double), pts.shape[0],
                               _p(out, C.c_int32))
    return out


def point_polygon_distance(soup, poly: int, px: float, py: float) -> float:
    """tests/oracles.hpp:92-95: 0 inside, else the nearest-edge distance."""
    vxy, ro, pr = _soup_arrays(soup)
    return float(lib().orc_point_polygon_distance(px, py, _p(vxy, C.c_double), _p(ro, C.c_uint64),
                                                  _p(pr, C.c_uint64), poly))


# -- the reference itself ------------------------------------------------------

class RefModel:
    """Reference leaves + (optionally) its cover/trie, via oracle/_ref."""

    def __init__(self, soup, scb=None):
        self._soup = _soup_arrays(soup)
        vxy, ro, pr = self._soup
        self.n = soup.n_polys
        self._scb = None if scb is None else np.ascontiguousarray(scb, dtype=np.uint32)
        L = ref()
        self._h = L.ref_model_create(_p(vxy, C.c_double), _p(ro, C.c_uint64), _p(pr, C.c_uint64),
                                     self.n, None if self._scb is None else _p(self._scb, C.c_uint32))
        if not self._h:
            raise RuntimeError(L.ref_last_error().decode())

    def __del__(self):
        if getattr(self, "_h", None):
            ref().ref_model_destroy(self._h)
            self._h = None

    def exhaustive_assign(self, pts) -> np.ndarray:
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        out = np.empty(pts.shape[0], dtype=np.int32)
        rc = ref().ref_exhaustive_assign(self._h, _p(pts, C.c_double), pts.shape[0], _p(out, C.c_int32))
        if rc:
            raise RuntimeError(ref().ref_last_error().decode())
        return out

    def build_index(self, max_level: int, levels_per_node: int = 4):
        sec = C.c_double(0)
        ne = C.c_uint64(0)
        tb = C.c_uint64(0)
        rc = ref().ref_build_index(self._h, max_level, levels_per_node, C.byref(sec),
                                   C.byref(ne), C.byref(tb))
        if rc:
            raise RuntimeError(ref().ref_last_error().decode())
        return {"seconds": sec.value, "entries": ne.value, "bytes": tb.value}

    def query_leaves(self, pts, threads: int = 0, chunk: int = 0, want_ids: bool = True):
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
        out = np.empty(pts.shape[0], dtype=np.int32) if want_ids else None
        pe = C.c_uint64(0)
        sec = C.c_double(0)
        rc = ref().ref_query_leaves(self._h, _p(pts, C.c_double), pts.shape[0], threads, chunk,
                                    None if out is None else _p(out, C.c_int32), C.byref(pe),
                                    C.byref(sec))
        if rc:
            raise RuntimeError(ref().ref_last_error().decode())
        return out, {"seconds": sec.value, "pip_point_evaluations": pe.value}


def ref_point_in_polygon(rings, px: float, py: float) -> bool:
    verts = np.ascontiguousarray(np.concatenate([np.asarray(r, np.float64).reshape(-1, 2) for r in rings]))
    off = np.zeros(len(rings) + 1, dtype=np.uint64)
    off[1:] = np.cumsum([len(r) for r in rings])
    rc = ref().ref_point_in_polygon(px, py, _p(verts, C.c_double), _p(off, C.c_uint64), len(rings))
    if rc < 0:
        raise ValueError(ref().ref_last_error().decode())
    return bool(rc)


def ref_generate_synthetic(seed, n_states, counties_per_state, blocks_per_county, jitter):
    """generate_synthetic + collect_leaves -> (vxy, ring_off, poly_ring, scb, fips, bbox)."""
    L = ref()
    npo, nr, nv = C.c_uint64(0), C.c_uint64(0), C.c_uint64(0)
    rc = L.ref_generate_synthetic(seed, n_states, counties_per_state, blocks_per_county, jitter,
                                  C.byref(npo), C.byref(nr), C.byref(nv), None, None, None,
                                  None, None, None)
    if rc:
        raise ValueError(L.ref_last_error().decode())
    vxy = np.zeros((nv.value, 2))
    ro = np.zeros(nr.value + 1, dtype=np.uint64)
    pr = np.zeros(npo.value + 1, dtype=np.uint64)
    scb = np.zeros((npo.value, 3), dtype=np.uint32)
    fips = C.create_string_buffer(12 * npo.value + 1)
    bbox = np.zeros(4)
    rc = L.ref_generate_synthetic(seed, n_states, counties_per_state, blocks_per_county, jitter,
                                  C.byref(npo), C.byref(nr), C.byref(nv), _p(vxy, C.c_double),
                                  _p(ro, C.c_uint64), _p(pr, C.c_uint64), _p(scb, C.c_uint32),
                                  fips, _p(bbox, C.c_double))
    if rc:
        raise ValueError(L.ref_last_error().decode())
    f = fips.raw[:12 * npo.value].decode()
    return vxy, ro, pr, scb, [f[12 * i:12 * i + 12] for i in range(npo.value)], bbox


def ref_sample(clustered: bool, bbox4, n: int, seed: int) -> np.ndarray:
    b = np.ascontiguousarray(bbox4, dtype=np.float64)
    out = np.empty((n, 2))
    rc = ref().ref_sample(1 if clustered else 0, _p(b, C.c_double), n, seed, _p(out, C.c_double))
    if rc:
        raise ValueError(ref().ref_last_error().decode())
    return out


def ref_save_synthetic_fmcb(seed, n_states, counties_per_state, blocks_per_county, jitter, path):
    """The reference's save_hierarchy over its generate_synthetic hierarchy."""
    rc = ref().ref_save_synthetic_fmcb(seed, n_states, counties_per_state, blocks_per_county,
                                       jitter, str(path).encode())
    if rc != 0:
        raise RuntimeError("reference save_hierarchy failed")


def ref_load_fmcb_status(path) -> int:
    """load_hierarchy's verdict: 0 ok, 1 runtime_error, 2 invalid_argument, 3 other."""
    return int(ref().ref_load_fmcb_status(str(path).encode()))


def ref_geojson_available() -> bool:
    return ref_available() and hasattr(ref(), "ref_ingest_geojson")


def ref_ingest_geojson(states, counties, blocks, out_fmcb):
    """The reference's `fastmap ingest` (load_boundaries + save_hierarchy):
    (status, message) -- 0 ok, 1 runtime_error, 2 invalid_argument, 3 other."""
    L = ref()
    rc = L.ref_ingest_geojson(*(str(x).encode() for x in (states, counties, blocks, out_fmcb)))
    return int(rc), (L.ref_last_error().decode() if rc else "")


def ref_write_synthetic_geojson(seed, n_states, counties_per_state, blocks_per_county, jitter, out_dir):
    """The reference's write_boundaries over its generate_synthetic hierarchy."""
    rc = ref().ref_write_synthetic_geojson(seed, n_states, counties_per_state, blocks_per_county,
                                           jitter, str(out_dir).encode())
    if rc != 0:
        raise RuntimeError("reference write_boundaries failed")


def ref_simple_assign(path, pts, strict: bool):
    """The reference's simple engine (simple_mapper.hpp:119-166) on an FMCB file:
    (state, county, block, (pip_point_evaluations, pip_calls))."""
    pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 2)
    n = pts.shape[0]
    st, co, bl = (np.empty(n, dtype=np.int32) for _ in range(3))
    cnt = np.zeros(2, dtype=np.uint64)
    rc = ref().ref_simple_assign_fmcb(str(path).encode(), _p(pts, C.c_double), n, 1 if strict else 0,
                                      _p(st, C.c_int32), _p(co, C.c_int32), _p(bl, C.c_int32),
                                      _p(cnt, C.c_uint64))
    if rc:
        raise RuntimeError("reference assign failed")
    return st, co, bl, (int(cnt[0]), int(cnt[1]))
