"""Host-side mirror of the reference's projection interface, B200-backed.

Names, argument meaning and error behaviour follow the reference headers
(``/root/reference/proj/include/fastmap``) so that code written against the
reference reads the same here:

===========================================  =====================================
reference (file:line)                        here
===========================================  =====================================
``PolygonGeometry`` geometry.hpp:64-87        :class:`PolygonGeometry`
``LeafRegion`` hierarchy.hpp:67-74            :class:`LeafRegion`
``CoverMode`` / ``CoverParams``               :class:`CoverMode` / :class:`CoverParams`
  cell_index.hpp:246-252
``build_cover`` cell_index.hpp:396-405        :func:`build_cover` (GPU cell index)
``build_trie`` cell_index.hpp:453-507         :func:`build_trie` (validates F; no trie
                                              is needed, the grid is direct-mapped)
``query_leaves`` cell_index.hpp:527-590       :func:`query_leaves`
``query`` cell_index.hpp:592-596              :func:`query`
``exhaustive_assign`` synthetic.hpp:193-205   :func:`exhaustive_assign`
``AssignmentResult`` simple_mapper.hpp:39-46  :class:`AssignmentResult`
``index_stats`` cell_index.hpp:616-631        :func:`index_stats`
``load_hierarchy`` hierarchy.hpp:204-223      :func:`load_hierarchy` (FMCB -> leaves)
FMCI save/load cell_index.hpp:641-726         :meth:`CellIndex.save` / :func:`load_index`
``read_points_f64`` io.hpp:154-167            :func:`read_points_f64`
assign CSV tools/fastmap.cpp:288-301          :func:`write_assign_csv`
``load_boundaries`` / ``write_boundaries``   :mod:`paper_2005_03156_b200.geojson`
  geojson.hpp:154-271, :276-353; ``fastmap    (``load_boundaries``, ``ingest``,
  ingest`` tools/fastmap.cpp:163-170          ``write_boundaries``)
``AssignMode``, ``assign`` simple_mapper.hpp  :class:`AssignMode`, :func:`assign` (the simple
  :24, :119-166                               engine on the GPU, :class:`SimpleEngine`)
===========================================  =====================================

Exceptions: ``std::invalid_argument`` -> ``ValueError``,
``std::runtime_error`` -> ``RuntimeError``.  The projection itself runs
only on the GPU (``libfastmap_b200.so``); with no CUDA device the query
calls raise ``RuntimeError`` -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import enum
import math
from dataclasses import dataclass, field
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native as N

K_MAX_LEVEL = 30  # CellId::kMaxLevel, cell_index.hpp:35


# ---------------------------------------------------------------------------
# geometry and leaf tables
# ---------------------------------------------------------------------------

class PolygonGeometry:
    """Multi-ring polygon as node lists (geometry.hpp:64-87)."""

    def __init__(self) -> None:
        self.rings: list[np.ndarray] = []

    def add_ring(self, ring) -> None:
        r = np.ascontiguousarray(np.asarray(ring, dtype=np.float64).reshape(-1, 2))
        if r.shape[0] < 3:
            raise ValueError("polygon ring needs at least 3 vertices")  # geometry.hpp:75-77
        self.rings.append(r)

    def empty(self) -> bool:
        return not self.rings

    def edge_count(self) -> int:
        return sum(r.shape[0] for r in self.rings)


@dataclass
class LeafRegion:
    """Flattened leaf record (hierarchy.hpp:67-74)."""
    state: int = 0
    county: int = 0
    block: int = 0
    geometry: Optional[PolygonGeometry] = None
    fips12: Optional[str] = None


@dataclass
class Soup:
    """Polygon soup in the C-ABI layout (include/fastmap_b200.h)."""
    vxy: np.ndarray        # (V, 2) float64 lon, lat
    ring_off: np.ndarray   # (R + 1,) uint64
    poly_ring: np.ndarray  # (P + 1,) uint64

    @property
    def n_polys(self) -> int:
        return int(self.poly_ring.shape[0] - 1)

    @property
    def n_rings(self) -> int:
        return int(self.ring_off.shape[0] - 1)

    @property
    def n_vertices(self) -> int:
        return int(self.vxy.shape[0])

    def contiguous(self) -> "Soup":
        return Soup(np.ascontiguousarray(self.vxy, dtype=np.float64),
                    np.ascontiguousarray(self.ring_off, dtype=np.uint64),
                    np.ascontiguousarray(self.poly_ring, dtype=np.uint64))

    def polygon(self, p: int) -> list[np.ndarray]:
        rings = []
        for r in range(int(self.poly_ring[p]), int(self.poly_ring[p + 1])):
            rings.append(self.vxy[int(self.ring_off[r]):int(self.ring_off[r + 1])])
        return rings

    @staticmethod
    def from_rings(polys: Sequence[Sequence[Iterable]]) -> "Soup":
        """``polys[p]`` is a list of rings; a ring is a sequence of (lon, lat)."""
        verts, ring_off, poly_ring = [], [0], [0]
        for rings in polys:
            for ring in rings:
                r = np.asarray(ring, dtype=np.float64).reshape(-1, 2)
                verts.append(r)
                ring_off.append(ring_off[-1] + r.shape[0])
            poly_ring.append(len(ring_off) - 1)
        vxy = np.concatenate(verts) if verts else np.zeros((0, 2))
        return Soup(np.ascontiguousarray(vxy), np.asarray(ring_off, dtype=np.uint64),
                    np.asarray(poly_ring, dtype=np.uint64))


def leaves_to_soup(leaves: Sequence[LeafRegion]) -> Soup:
    polys = []
    for lf in leaves:
        g = lf.geometry
        polys.append([] if g is None else list(g.rings))
    return Soup.from_rings(polys)


class Hierarchy:
    """An FMCB region hierarchy flattened to its leaves (``load_hierarchy``,
    hierarchy.hpp:204-223, then ``collect_leaves``, hierarchy.hpp:76-91):
    the leaf soup, per-leaf (state, county, block) and 12-char FIPS codes.
    Owns the native ``fm_hierarchy`` handle (used by :func:`write_assign_csv`)."""

    def __init__(self, handle: C.c_void_p) -> None:
        self._h = handle
        L = N.lib()
        v = [C.c_uint64(0) for _ in range(5)]
        N.check(L.fm_hierarchy_sizes(handle, *[C.byref(x) for x in v]), "fm_hierarchy_sizes")
        self.n_states, self.n_counties, n_leaves, n_rings, n_verts = (x.value for x in v)
        vxy = np.zeros((n_verts, 2), dtype=np.float64)
        ro = np.zeros(n_rings + 1, dtype=np.uint64)
        pr = np.zeros(n_leaves + 1, dtype=np.uint64)
        self.scb = np.zeros((n_leaves, 3), dtype=np.uint32)
        fips = C.create_string_buffer(12 * n_leaves + 1)
        N.check(L.fm_hierarchy_leaves(handle, N.ptr(vxy, C.c_double), N.ptr(ro, C.c_uint64),
                                      N.ptr(pr, C.c_uint64), N.ptr(self.scb, C.c_uint32), fips),
                "fm_hierarchy_leaves")
        self.soup = Soup(vxy, ro, pr)
        self.fips12 = np.frombuffer(fips.raw[:12 * n_leaves], dtype="S12").copy()

    @property
    def n_leaves(self) -> int:
        return self.soup.n_polys

    def __del__(self) -> None:
        if getattr(self, "_h", None):
            lib = N.lib() if N is not None else None
            if lib is not None:
                lib.fm_hierarchy_destroy(self._h)
            self._h = None


def load_hierarchy(path: str) -> Hierarchy:
    """Read an FMCB file (the reference's ``save_hierarchy`` format)."""
    h = C.c_void_p()
    N.check(N.lib().fm_hierarchy_load(str(path).encode(), C.byref(h)), "fm_hierarchy_load")
    return Hierarchy(h)


def read_points_f64(path: str) -> np.ndarray:
    """Raw little-endian f64 (lon, lat) pairs -> (n, 2) float64 (io.hpp:154-167)."""
    L = N.lib()
    n = C.c_uint64(0)
    N.check(L.fm_read_points_f64(str(path).encode(), None, C.byref(n)), "fm_read_points_f64")
    pts = np.zeros((n.value, 2), dtype=np.float64)
    N.check(L.fm_read_points_f64(str(path).encode(), N.ptr(pts, C.c_double), C.byref(n)),
            "fm_read_points_f64")
    return pts


def write_assign_csv(path: str, points: np.ndarray, ids: np.ndarray, hierarchy: Hierarchy) -> None:
    """The reference CLI's ``idx,lon,lat,fips`` output (tools/fastmap.cpp:288-301)."""
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
    ids = np.ascontiguousarray(ids, dtype=np.int32)
    if ids.shape[0] != pts.shape[0]:
        raise ValueError("one id per point")
    N.check(N.lib().fm_write_assign_csv(str(path).encode(), N.ptr(pts, C.c_double), pts.shape[0],
                                        N.ptr(ids, C.c_int32), hierarchy._h), "fm_write_assign_csv")


# ---------------------------------------------------------------------------
# parameters, results
# ---------------------------------------------------------------------------

class CoverMode(enum.IntEnum):
    exact = 0
    approx = 1


def level_diagonal(lvl: int) -> float:
    scale = math.ldexp(1.0, lvl)
    return math.hypot(360.0 / scale, 180.0 / scale)  # cell_index.hpp:152-155


@dataclass
class CoverParams:
    """CoverParams (cell_index.hpp:248-252) plus the grid knobs of fm_build_params.

    ``max_level``/``epsilon`` are validated exactly like
    ``validate_cover_params`` (cell_index.hpp:382-394); the GPU index is exact
    at every max_level (its resolution is set by ``cells_per_polygon``)."""
    max_level: int = 30
    mode: CoverMode = CoverMode.exact
    epsilon: float = 0.0
    cells_per_polygon: float = 0.0
    nx: int = 0
    ny: int = 0
    margin: float = 0.0
    threads: int = 0


def validate_cover_params(p: CoverParams) -> None:
    if p.max_level < 0 or p.max_level > K_MAX_LEVEL:
        raise ValueError("max_level must be in [0, 30]")
    if p.mode == CoverMode.approx:
        floor = level_diagonal(K_MAX_LEVEL)
        if not (p.epsilon > 0.0) or p.epsilon < floor:
            raise ValueError(
                f"approx epsilon must be at least the level-30 cell diagonal ({floor:f} degrees)")


@dataclass
class AssignCounters:
    pip_point_evaluations: int = 0  # simple_mapper.hpp:26-35
    pip_calls: int = 0


@dataclass
class AssignmentResult:
    """Per-point (state, county, block), -1 when unresolved (simple_mapper.hpp:39-46)."""
    state: np.ndarray
    county: np.ndarray
    block: np.ndarray
    counters: AssignCounters = field(default_factory=AssignCounters)
    leaf: Optional[np.ndarray] = None  # leaf id per point (collect_leaves position)

    def size(self) -> int:
        return int(self.state.shape[0])


# ---------------------------------------------------------------------------
# the GPU index
# ---------------------------------------------------------------------------

class CellIndex:
    """Owner of an ``fm_index*`` (the analogue of CellCover + TrieIndex)."""

    def __init__(self, handle: C.c_void_p, n_leaves: int, params: CoverParams,
                 device: int) -> None:
        self._h = handle
        self.n_leaves = n_leaves
        self.params = params
        self.device = device
        self.levels_per_node = 1

    def __del__(self) -> None:
        self.close()

    def close(self) -> None:
        if getattr(self, "_h", None):
            lib = N.lib() if N is not None else None
            if lib is not None:
                lib.fm_index_destroy(self._h)
            self._h = None

    @property
    def handle(self) -> C.c_void_p:
        if not self._h:
            raise ValueError("index is closed")
        return self._h

    def stats(self) -> dict:
        s = N.IndexStats()
        N.check(N.lib().fm_index_stats_get(self.handle, C.byref(s)), "fm_index_stats_get")
        return s.as_dict()

    def export(self):
        """(grid u32[ny*nx], arena u8[], geometry dict) -- host copies."""
        L = N.lib()
        gl, al = C.c_uint64(0), C.c_uint64(0)
        geo = np.zeros(16, dtype=np.float64)
        N.check(L.fm_index_export(self.handle, None, C.byref(gl), None, C.byref(al),
                                  N.ptr(geo, C.c_double)), "fm_index_export")
        grid = np.zeros(gl.value, dtype=np.uint32)
        arena = np.zeros(al.value, dtype=np.uint8)
        N.check(L.fm_index_export(self.handle, N.ptr(grid, C.c_uint32), C.byref(gl),
                                  N.ptr(arena, C.c_uint8), C.byref(al), N.ptr(geo, C.c_double)),
                "fm_index_export")
        keys = ("gx0", "gx1", "gy0", "gy1", "w", "h", "inv_w", "inv_h", "nx", "ny",
                "margin", "n_polys", "slot_bytes")
        g = dict(zip(keys, geo.tolist()))
        g["slot_bytes"] = int(g["slot_bytes"])
        g["nx"] = int(g["nx"])
        g["ny"] = int(g["ny"])
        g["n_polys"] = int(g["n_polys"])
        return grid, arena, g

    def set_query_path(self, path: str = "auto", tile_bytes: float = 0.0) -> None:
        """Exact-mode query path: "auto" (default), "stream" or "binned"
        (fm_index_set_query_path; the answers are the same on every path)."""
        code = {"auto": N.PATH_AUTO, "stream": N.PATH_STREAM, "binned": N.PATH_BINNED}[path]
        N.check(N.lib().fm_index_set_query_path(self.handle, code, float(tile_bytes)),
                "fm_index_set_query_path")

    def query_plan(self, n: int) -> dict:
        """The path a batch of n points takes, and the binned path's tiles."""
        p, ts, nt = C.c_int(0), C.c_int32(0), C.c_int32(0)
        N.check(N.lib().fm_index_query_plan(self.handle, int(n), C.byref(p), C.byref(ts),
                                            C.byref(nt)), "fm_index_query_plan")
        return {"path": "binned" if p.value == N.PATH_BINNED else "stream",
                "tile_log2": ts.value, "n_tiles": nt.value}

    def save(self, path: str) -> None:
        """Persist the built index (FMCI analogue); reload with :func:`load_index`."""
        N.check(N.lib().fm_index_save(self.handle, str(path).encode()), "fm_index_save")

    # -- projection ---------------------------------------------------------
    def project(self, points, out=None, hist=None, counters=None, stream=None,
                mode: "CoverMode" = None):
        """Leaf id per point.

        ``mode``: CoverMode.exact (default) or CoverMode.approx (an index built
        with an approx-mode CoverParams; deemed leaves for boundary cells).

        ``points``: a CUDA ``torch.Tensor`` (n, 2) float64 on the index's device
        (asynchronous, on ``stream`` or the current torch stream), or a numpy
        (n, 2) float64 array (host path: pipelined copies; synchronous).
        ``hist``: optional int64 per-leaf counters, accumulated into.
        """
        L = N.lib()
        m = int(CoverMode.exact if mode is None else mode)
        if isinstance(points, np.ndarray):
            pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
            n = pts.shape[0]
            if out is None:
                out = np.empty(n, dtype=np.int32)
            hp = None
            if hist is not None:
                assert hist.dtype == np.int64 and hist.flags.c_contiguous
                hp = N.ptr(hist, C.c_int64)
            N.check(L.fm_query_host_mode(self.handle, m, N.ptr(pts, C.c_double), n,
                                         N.ptr(out, C.c_int32), hp), "fm_query_host")
            return out
        import torch  # device path
        if not (isinstance(points, torch.Tensor) and points.is_cuda):
            raise TypeError("points must be a numpy array or a CUDA torch tensor")
        if points.dtype != torch.float64 or not points.is_contiguous():
            raise ValueError("device points must be contiguous float64 (n, 2)")
        n = points.numel() // 2
        if out is None:
            out = torch.empty(n, dtype=torch.int32, device=points.device)
        if stream is None:
            stream = torch.cuda.current_stream(points.device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        N.check(L.fm_query_mode(self.handle, m, C.c_void_p(points.data_ptr()), n,
                           C.c_void_p(out.data_ptr()),
                           C.c_void_p(hist.data_ptr()) if hist is not None else None,
                           C.c_void_p(counters.data_ptr()) if counters is not None else None,
                           C.c_void_p(stream)), "fm_query")
        return out


def build_index(soup: Soup, params: Optional[CoverParams] = None, device: int = 0,
                on_gpu: bool = True) -> CellIndex:
    """fm_index_build over a soup.  ``device=-1`` builds a host-only index
    (inspection/export only; queries on it raise).  ``on_gpu=False`` runs the
    host builder and uploads the result (same arrays as the GPU builder)."""
    params = params or CoverParams()
    validate_cover_params(params)
    s = soup.contiguous()
    bp = N.BuildParams(cells_per_polygon=float(params.cells_per_polygon),
                       nx=int(params.nx), ny=int(params.ny), margin=float(params.margin),
                       device=int(device), build_on_gpu=1 if (device >= 0 and on_gpu) else 0,
                       threads=int(params.threads),
                       approx_epsilon=float(params.epsilon) if params.mode == CoverMode.approx
                       else 0.0)
    h = C.c_void_p()
    st = N.lib().fm_index_build(N.ptr(s.vxy, C.c_double), N.ptr(s.ring_off, C.c_uint64),
                                s.n_rings, N.ptr(s.poly_ring, C.c_uint64), s.n_polys,
                                C.byref(bp), C.byref(h))
    N.check(st, "fm_index_build")
    return CellIndex(h, s.n_polys, params, device)


class MultiIndex:
    """Owner of an ``fm_multi*``: one index replica per GPU of this process
    and the sharded host-buffer query (run_chunked one level up,
    parallel.hpp:30-82).  ``project`` splits a host batch into contiguous,
    balanced shards, one per device, and sums the optional histogram with
    one ncclAllReduce."""

    def __init__(self, soup: Soup, devices: Sequence[int], params: Optional[CoverParams] = None):
        params = params or CoverParams()
        validate_cover_params(params)
        s = soup.contiguous()
        self._keep = s
        self.n_leaves = s.n_polys
        self.devices = [int(d) for d in devices]
        bp = N.BuildParams(cells_per_polygon=float(params.cells_per_polygon), nx=int(params.nx),
                           ny=int(params.ny), margin=float(params.margin), device=0,
                           build_on_gpu=1, threads=int(params.threads),
                           approx_epsilon=float(params.epsilon) if params.mode == CoverMode.approx
                           else 0.0)
        devs = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        self._h = None
        N.check(N.lib().fm_multi_build(N.ptr(s.vxy, C.c_double), N.ptr(s.ring_off, C.c_uint64),
                                       s.n_rings, N.ptr(s.poly_ring, C.c_uint64), s.n_polys,
                                       C.byref(bp), devs, len(self.devices), C.byref(h)),
                "fm_multi_build")
        self._h = h

    def __del__(self) -> None:
        self.close()

    def close(self) -> None:
        if getattr(self, "_h", None):
            if N is not None:
                N.lib().fm_multi_destroy(self._h)
            self._h = None

    def __len__(self) -> int:
        return N.lib().fm_multi_size(self._h)

    def replica_stats(self, k: int) -> dict:
        s = N.IndexStats()
        N.check(N.lib().fm_index_stats_get(N.lib().fm_multi_replica(self._h, int(k)), C.byref(s)),
                "fm_index_stats_get")
        return s.as_dict()

    def project(self, points: np.ndarray, out: Optional[np.ndarray] = None,
                hist: Optional[np.ndarray] = None, mode: "CoverMode" = None) -> np.ndarray:
        """Leaf id per point of a HOST (n, 2) float64 batch; ``hist`` (int64
        per leaf) is accumulated into."""
        if not self._h:
            raise ValueError("index is closed")
        pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
        n = pts.shape[0]
        if out is None:
            out = np.empty(n, dtype=np.int32)
        hp = None
        if hist is not None:
            assert hist.dtype == np.int64 and hist.flags.c_contiguous and hist.size == self.n_leaves
            hp = N.ptr(hist, C.c_int64)
        m = int(CoverMode.exact if mode is None else mode)
        N.check(N.lib().fm_multi_query_host(self._h, m, N.ptr(pts, C.c_double), n,
                                            N.ptr(out, C.c_int32), hp), "fm_multi_query_host")
        return out


def load_index(path: str, device: int = 0, params: Optional[CoverParams] = None) -> CellIndex:
    """An index saved by :meth:`CellIndex.save`, onto ``device`` (-1 = host-only)."""
    h = C.c_void_p()
    N.check(N.lib().fm_index_load(str(path).encode(), int(device), C.byref(h)), "fm_index_load")
    s = N.IndexStats()
    N.check(N.lib().fm_index_stats_get(h, C.byref(s)), "fm_index_stats_get")
    if params is None:
        eps = float(s.approx_epsilon)
        params = CoverParams(mode=CoverMode.approx if eps > 0 else CoverMode.exact, epsilon=eps)
    return CellIndex(h, int(s.n_polys), params, device)


def build_index_hierarchy(h: Hierarchy, params: Optional[CoverParams] = None,
                          device: int = 0) -> CellIndex:
    """fm_index_build_hierarchy: the index over an FMCB hierarchy's leaves."""
    params = params or CoverParams()
    validate_cover_params(params)
    bp = N.BuildParams(cells_per_polygon=float(params.cells_per_polygon),
                       nx=int(params.nx), ny=int(params.ny), margin=float(params.margin),
                       device=int(device), build_on_gpu=1 if device >= 0 else 0,
                       threads=int(params.threads),
                       approx_epsilon=float(params.epsilon) if params.mode == CoverMode.approx
                       else 0.0)
    out = C.c_void_p()
    N.check(N.lib().fm_index_build_hierarchy(h._h, C.byref(bp), C.byref(out)),
            "fm_index_build_hierarchy")
    return CellIndex(out, h.n_leaves, params, device)


def build_cover(leaves, params: Optional[CoverParams] = None, device: int = 0) -> CellIndex:
    """build_cover(leaves, params) (cell_index.hpp:396-405) -> GPU cell index.

    ``leaves`` is a sequence of :class:`LeafRegion` or a :class:`Soup`."""
    if isinstance(leaves, Hierarchy):
        return build_index_hierarchy(leaves, params, device)
    soup = leaves if isinstance(leaves, Soup) else leaves_to_soup(leaves)
    return build_index(soup, params, device)


class TrieIndex:
    """What build_trie returns: the index plus the requested fanout.  The
    grid is direct-mapped, so lookups take one probe for any F."""

    def __init__(self, cover: CellIndex, levels_per_node: int) -> None:
        self.cover = cover
        self.levels_per_node = levels_per_node
        self.fanout = 1 << (2 * levels_per_node)


def build_trie(cover: CellIndex, levels_per_node: int) -> TrieIndex:
    if levels_per_node not in (1, 2, 4):  # cell_index.hpp:454-456
        raise ValueError("trie fanout must be 1, 2 or 4 levels per node")
    return TrieIndex(cover, levels_per_node)


def _leaf_table(leaves) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    if isinstance(leaves, Hierarchy):
        t = leaves.scb.astype(np.int32)
        return t[:, 0].copy(), t[:, 1].copy(), t[:, 2].copy()
    if isinstance(leaves, Soup):
        n = leaves.n_polys
        return (np.zeros(n, np.int32), np.zeros(n, np.int32), np.arange(n, dtype=np.int32))
    st = np.fromiter((lf.state for lf in leaves), dtype=np.int32, count=len(leaves))
    co = np.fromiter((lf.county for lf in leaves), dtype=np.int32, count=len(leaves))
    bl = np.fromiter((lf.block for lf in leaves), dtype=np.int32, count=len(leaves))
    return st, co, bl


def query_leaves(trie, leaves, points, mode: CoverMode = CoverMode.exact) -> AssignmentResult:
    """query_leaves (cell_index.hpp:527-590): leaf id -> (state, county, block)
    exactly as set_leaf does (cell_index.hpp:515-519)."""
    cover = trie.cover if isinstance(trie, TrieIndex) else trie
    if mode == CoverMode.approx and cover.params.mode != CoverMode.approx:
        raise ValueError("approximate queries require an approximate-mode cover")
    n_leaves = (leaves.n_polys if isinstance(leaves, Soup) else
                leaves.n_leaves if isinstance(leaves, Hierarchy) else len(leaves))
    if cover.n_leaves != n_leaves:
        raise ValueError("cover was built for a different hierarchy")
    ids = cover.project(points, mode=mode)
    if not isinstance(ids, np.ndarray):
        ids = ids.cpu().numpy()
    st, co, bl = _leaf_table(leaves)
    hit = ids >= 0
    res = AssignmentResult(state=np.where(hit, st[np.maximum(ids, 0)], -1).astype(np.int32),
                           county=np.where(hit, co[np.maximum(ids, 0)], -1).astype(np.int32),
                           block=np.where(hit, bl[np.maximum(ids, 0)], -1).astype(np.int32),
                           leaf=ids)
    return res


def query(trie, leaves, points, mode: CoverMode = CoverMode.exact) -> AssignmentResult:
    return query_leaves(trie, leaves, points, mode)


class AssignMode(enum.IntEnum):
    """simple_mapper.hpp:24."""
    relaxed = 0
    strict = 1


class SimpleEngine:
    """The simple engine's device structures for one hierarchy (fm_simple)."""

    def __init__(self, h: Hierarchy, device: int = 0) -> None:
        self._s = None
        s = C.c_void_p()
        N.check(N.lib().fm_simple_build(h._h, int(device), C.byref(s)), "fm_simple_build")
        self._s = s
        self.device = device
        self.hierarchy = h

    def __del__(self) -> None:
        if getattr(self, "_s", None):
            lib = N.lib() if N is not None else None
            if lib is not None:
                lib.fm_simple_destroy(self._s)
            self._s = None

    def assign(self, points, mode: AssignMode = AssignMode.relaxed, counters: Optional[bool] = None,
               out=None, stream=None):
        """Host numpy points -> AssignmentResult (counters on by default).

        CUDA tensor points -> (state, county, block) int32 tensors written on
        ``stream`` (asynchronously).  With ``counters=True`` the call is
        synchronous and returns ``((state, county, block), AssignCounters)``;
        the default for tensors is no counters."""
        L = N.lib()
        cnt = N.AssignCountersC()
        if isinstance(points, np.ndarray):
            cp = C.byref(cnt) if counters is None or counters else None
            pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 2)
            n = pts.shape[0]
            st, co, bl = (np.empty(n, dtype=np.int32) for _ in range(3))
            N.check(L.fm_simple_assign_host(self._s, int(mode), N.ptr(pts, C.c_double), n,
                                            N.ptr(st, C.c_int32), N.ptr(co, C.c_int32),
                                            N.ptr(bl, C.c_int32), cp), "fm_simple_assign_host")
            return AssignmentResult(st, co, bl, AssignCounters(int(cnt.pip_point_evaluations),
                                                               int(cnt.pip_calls)))
        import torch
        if not (isinstance(points, torch.Tensor) and points.is_cuda):
            raise TypeError("points must be a numpy array or a CUDA torch tensor")
        if (points.dtype != torch.float64 or not points.is_contiguous() or points.dim() != 2
                or points.shape[1] != 2):
            raise ValueError("device points must be a contiguous float64 (n, 2) tensor")
        if points.device.index != self.device:
            raise ValueError(f"points are on {points.device}, the engine on cuda:{self.device}")
        n = points.shape[0]
        if out is None:
            out = tuple(torch.empty(n, dtype=torch.int32, device=points.device) for _ in range(3))
        for t in out:
            if (t.dtype != torch.int32 or not t.is_contiguous() or t.numel() < n
                    or t.device != points.device):
                raise ValueError("outputs must be contiguous int32 tensors of n points on the same device")
        if stream is None:
            stream = torch.cuda.current_stream(points.device).cuda_stream
        elif hasattr(stream, "cuda_stream"):
            stream = stream.cuda_stream
        want = bool(counters)
        N.check(L.fm_simple_assign(self._s, int(mode), C.c_void_p(points.data_ptr()), n,
                                   *[C.c_void_p(t.data_ptr()) for t in out],
                                   C.byref(cnt) if want else None,
                                   C.c_void_p(stream)), "fm_simple_assign")
        if want:
            return out, AssignCounters(int(cnt.pip_point_evaluations), int(cnt.pip_calls))
        return out


def assign(h, points, mode: AssignMode = AssignMode.relaxed, device: int = 0) -> AssignmentResult:
    """assign(h, points, mode) (simple_mapper.hpp:119-166) on the GPU."""
    eng = h if isinstance(h, SimpleEngine) else SimpleEngine(h, device)
    return eng.assign(points, mode)


def exhaustive_assign(leaves, points, device: int = 0) -> np.ndarray:
    """exhaustive_assign semantics (synthetic.hpp:193-205), computed on the GPU."""
    idx = build_cover(leaves, CoverParams(), device)
    try:
        ids = idx.project(points)
        return ids if isinstance(ids, np.ndarray) else ids.cpu().numpy()
    finally:
        idx.close()


def index_stats(trie, cover=None) -> dict:
    c = trie.cover if isinstance(trie, TrieIndex) else trie
    return c.stats()
