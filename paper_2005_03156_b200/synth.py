"""The BASELINE.json workload configs as deterministic generators.

Every config is a polygon tiling of the domain lon [-125, -66] x lat [24, 50]
plus a seeded fp64 point stream.  Generation runs in the native
``libfastmap_synth.so`` (counter-based RNG, so any shard of the stream is
reproducible on any rank).  Recipe choices for what BASELINE leaves open are
documented in DESIGN.md sec. 3.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native as N
from .fastmap import Soup

DOMAIN = (-125.0, -66.0, 24.0, 50.0)  # x0, x1, y0, y1


def expanded_box(domain=DOMAIN, frac: float = 0.01):
    """The domain bbox scaled by (1 + frac) about its centre (0.5% per side)."""
    x0, x1, y0, y1 = domain
    dx, dy = 0.5 * frac * (x1 - x0), 0.5 * frac * (y1 - y0)
    return (x0 - dx, x1 + dx, y0 - dy, y1 + dy)


def _threads() -> int:
    return max(1, min(64, os.cpu_count() or 1))


def _dev_args(out, stream):
    """(n, data pointer, cudaStream_t) of a CUDA float64 (n, 2) tensor."""
    import torch
    if not (isinstance(out, torch.Tensor) and out.is_cuda and out.dtype == torch.float64
            and out.is_contiguous() and out.dim() == 2 and out.shape[1] == 2):
        raise ValueError("out must be a contiguous CUDA float64 (n, 2) tensor")
    if stream is None:
        stream = torch.cuda.current_stream(out.device)
    s = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    return out.shape[0], C.c_void_p(out.data_ptr()), C.c_void_p(s)


def _clustered_dev(cfg, out, offset, stream):
    n, ptr, s = _dev_args(out, stream)
    box = np.asarray(expanded_box(), dtype=np.float64)
    dom = np.asarray(DOMAIN, dtype=np.float64)
    rc = N.synth().synth_points_clustered_dev(N.ptr(dom, C.c_double), N.ptr(box, C.c_double), n,
                                              offset, cfg.seed + 1, cfg.n_centres,
                                              cfg.centre_sigma_deg, cfg.zipf_s,
                                              cfg.frac_clustered, ptr, s)
    if rc != 0:
        raise RuntimeError(f"synth_points_clustered_dev failed ({rc})")
    return out


@dataclass(frozen=True)
class TilingConfig:
    name: str
    nx: int
    ny: int
    segs: int
    jitter: float
    sigma: float
    n_points: int
    points: str                 # "uniform" | "clustered" | "near_edge"
    seed: int = 0
    n_centres: int = 2000
    centre_sigma_deg: float = 0.2
    zipf_s: float = 1.1
    frac_clustered: float = 0.9
    frac_near: float = 0.5
    near_eps_cells: float = 1e-4

    @property
    def n_polys(self) -> int:
        return self.nx * self.ny

    @property
    def cell_size(self):
        x0, x1, y0, y1 = DOMAIN
        return ((x1 - x0) / self.nx, (y1 - y0) / self.ny)

    def make_soup(self, threads: Optional[int] = None) -> Soup:
        P = self.nx * self.ny
        V = P * 4 * self.segs
        vxy = np.empty((V, 2), dtype=np.float64)
        ring_off = np.empty(P + 1, dtype=np.uint64)
        poly_ring = np.empty(P + 1, dtype=np.uint64)
        x0, x1, y0, y1 = DOMAIN
        rc = N.synth().synth_tiling(self.nx, self.ny, self.segs, self.jitter, self.sigma,
                                    x0, x1, y0, y1, self.seed, threads or _threads(),
                                    N.ptr(vxy, C.c_double), N.ptr(ring_off, C.c_uint64),
                                    N.ptr(poly_ring, C.c_uint64))
        if rc != 0:
            raise ValueError("synth_tiling failed")
        return Soup(vxy, ring_off, poly_ring)

    def make_points(self, n: Optional[int] = None, offset: int = 0,
                    soup: Optional[Soup] = None, threads: Optional[int] = None,
                    out: Optional[np.ndarray] = None) -> np.ndarray:
        n = self.n_points if n is None else int(n)
        pts = out if out is not None else np.empty((n, 2), dtype=np.float64)
        assert pts.dtype == np.float64 and pts.flags.c_contiguous and pts.shape == (n, 2)
        box = np.asarray(expanded_box(), dtype=np.float64)
        dom = np.asarray(DOMAIN, dtype=np.float64)
        t = threads or _threads()
        L = N.synth()
        if self.points == "uniform":
            rc = L.synth_points_uniform(N.ptr(box, C.c_double), n, offset, self.seed + 1, t,
                                        N.ptr(pts, C.c_double))
        elif self.points == "clustered":
            rc = L.synth_points_clustered(N.ptr(dom, C.c_double), N.ptr(box, C.c_double), n,
                                          offset, self.seed + 1, self.n_centres,
                                          self.centre_sigma_deg, self.zipf_s,
                                          self.frac_clustered, t, N.ptr(pts, C.c_double))
        elif self.points == "near_edge":
            s = (soup or self.make_soup()).contiguous()
            cw, ch = self.cell_size
            rc = L.synth_points_near_edge(N.ptr(s.vxy, C.c_double), N.ptr(s.ring_off, C.c_uint64),
                                          N.ptr(s.poly_ring, C.c_uint64), s.n_polys, cw, ch,
                                          self.near_eps_cells, self.frac_near,
                                          N.ptr(box, C.c_double), n, offset, self.seed + 1, t,
                                          N.ptr(pts, C.c_double))
        else:
            raise ValueError(self.points)
        if rc != 0:
            raise ValueError("point generation failed")
        return pts

    def make_points_device(self, out, offset: int = 0, soup: Optional[Soup] = None,
                           stream=None, soup_device=None):
        """Points [offset, offset + n) of this config's stream written into the
        CUDA float64 (n, 2) tensor ``out`` by the GPU generator -- bit-identical
        to :meth:`make_points` (csrc/synth_rng.h).  ``soup_device``: the soup's
        (vxy, ring_off, poly_ring) as CUDA tensors (near-edge streams; built
        from ``soup`` when omitted)."""
        if self.points == "clustered":
            return _clustered_dev(self, out, offset, stream)
        n, ptr, s = _dev_args(out, stream)
        box = np.asarray(expanded_box(), dtype=np.float64)
        L = N.synth()
        if self.points == "uniform":
            rc = L.synth_points_uniform_dev(N.ptr(box, C.c_double), n, offset, self.seed + 1, ptr, s)
        elif self.points == "near_edge":
            if soup_device is None:
                import torch
                sp = (soup or self.make_soup()).contiguous()
                soup_device = (torch.from_numpy(sp.vxy).to(out.device),
                               torch.from_numpy(sp.ring_off.view(np.int64)).to(out.device),
                               torch.from_numpy(sp.poly_ring.view(np.int64)).to(out.device))
            vd, rd, pd = soup_device
            cw, ch = self.cell_size
            rc = L.synth_points_near_edge_dev(C.c_void_p(vd.data_ptr()), C.c_void_p(rd.data_ptr()),
                                              C.c_void_p(pd.data_ptr()), pd.shape[0] - 1, cw, ch,
                                              self.near_eps_cells, self.frac_near,
                                              N.ptr(box, C.c_double), n, offset, self.seed + 1,
                                              ptr, s)
        else:
            raise ValueError(self.points)
        if rc != 0:
            raise RuntimeError(f"device point generation failed ({rc})")
        return out


@dataclass(frozen=True)
class NestedConfig:
    """BASELINE config 3 (and 5): states -> counties -> blocks, conformal
    nested jittered tilings; leaves are the blocks in collect_leaves order."""
    name: str
    sx: int
    sy: int
    cx: int
    cy: int
    bx: int
    by: int
    segs: int
    jitter: float
    sigma: float
    n_points: int
    seed: int = 0
    n_centres: int = 20_000
    centre_sigma_deg: float = 0.2
    zipf_s: float = 1.1
    frac_clustered: float = 0.9
    points: str = "clustered"

    @property
    def n_polys(self) -> int:
        return self.sx * self.sy * self.cx * self.cy * self.bx * self.by

    def make_soup(self, threads: Optional[int] = None, with_scb: bool = False):
        P = self.n_polys
        vxy = np.empty((P * 4 * self.segs, 2), dtype=np.float64)
        ring_off = np.empty(P + 1, dtype=np.uint64)
        poly_ring = np.empty(P + 1, dtype=np.uint64)
        scb = np.empty((P, 3), dtype=np.uint32)
        x0, x1, y0, y1 = DOMAIN
        rc = N.synth().synth_nested(self.sx, self.sy, self.cx, self.cy, self.bx, self.by,
                                    self.segs, self.jitter, self.sigma, x0, x1, y0, y1,
                                    self.seed, threads or _threads(), N.ptr(vxy, C.c_double),
                                    N.ptr(ring_off, C.c_uint64), N.ptr(poly_ring, C.c_uint64),
                                    N.ptr(scb, C.c_uint32))
        if rc != 0:
            raise ValueError("synth_nested failed")
        soup = Soup(vxy, ring_off, poly_ring)
        return (soup, scb) if with_scb else soup

    def write_fmcb(self, path, threads: Optional[int] = None) -> None:
        """The full three-level hierarchy (states, counties, blocks) as an
        FMCB file -- the simple engine's input (simple_mapper.hpp)."""
        x0, x1, y0, y1 = DOMAIN
        rc = N.synth().synth_nested_fmcb(self.sx, self.sy, self.cx, self.cy, self.bx, self.by,
                                         self.segs, self.jitter, self.sigma, x0, x1, y0, y1,
                                         self.seed, threads or _threads(), str(path).encode())
        if rc != 0:
            raise RuntimeError(f"synth_nested_fmcb failed for {path}")

    def make_points(self, n: Optional[int] = None, offset: int = 0, soup=None,
                    threads: Optional[int] = None, out: Optional[np.ndarray] = None) -> np.ndarray:
        n = self.n_points if n is None else int(n)
        pts = out if out is not None else np.empty((n, 2), dtype=np.float64)
        box = np.asarray(expanded_box(), dtype=np.float64)
        dom = np.asarray(DOMAIN, dtype=np.float64)
        rc = N.synth().synth_points_clustered(N.ptr(dom, C.c_double), N.ptr(box, C.c_double), n,
                                              offset, self.seed + 1, self.n_centres,
                                              self.centre_sigma_deg, self.zipf_s,
                                              self.frac_clustered, threads or _threads(),
                                              N.ptr(pts, C.c_double))
        if rc != 0:
            raise ValueError("point generation failed")
        return pts

    def make_points_device(self, out, offset: int = 0, soup=None, stream=None, soup_device=None):
        """GPU-generated points [offset, offset + n) into the CUDA tensor
        ``out``, bit-identical to :meth:`make_points`."""
        return _clustered_dev(self, out, offset, stream)


CONFIGS = {
    # BASELINE configs[0]: small CPU-runnable case
    "c1": TilingConfig("c1", 32, 32, 8, 0.3, 0.05, 1_000_000, "uniform"),
    # configs[1]: census block-group scale, clustered points (bench workload)
    "c2": TilingConfig("c2", 500, 500, 12, 0.3, 0.05, 100_000_000, "clustered"),
    # configs[3]: strongly concave blocks, half the points near an edge
    "c4": TilingConfig("c4", 400, 250, 50, 0.3, 0.15, 200_000_000, "near_edge"),
    # configs[2]: 10x5 states, 20x20 counties each, 25x25 blocks each (12.5M leaves)
    "c3": NestedConfig("c3", 10, 5, 20, 20, 25, 25, 6, 0.3, 0.05, 1_000_000_000),
    # configs[4]: the c3 index with 8B points (sharded over GPUs) + histogram
    "c5": NestedConfig("c5", 10, 5, 20, 20, 25, 25, 6, 0.3, 0.05, 8_000_000_000),
    # reduced c3 with the same recipe, for parity tests (4 states, 40,000 leaves)
    "c3mini": NestedConfig("c3mini", 2, 2, 4, 4, 25, 25, 6, 0.3, 0.05, 2_000_000),
    # the c3 recipe at 320,000 leaves (50 states x 64 counties x 100 blocks):
    # the simple engine's bench hierarchy (written as FMCB with all levels)
    "c3s": NestedConfig("c3s", 10, 5, 8, 8, 10, 10, 6, 0.3, 0.05, 100_000_000),
}


def config(name: str) -> TilingConfig:
    try:
        return CONFIGS[name]
    except KeyError:
        raise ValueError(f"unknown config {name!r}; have {sorted(CONFIGS)}") from None
