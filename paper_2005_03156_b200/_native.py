"""ctypes bindings to the in-tree native libraries.

``libfastmap_b200.so`` is the product (C-ABI in ``include/fastmap_b200.h``);
``libfastmap_synth.so`` holds the workload generators.  Both are built
in-tree by ``make`` (``__graft_entry__.build()``).  A missing product
library is a hard error: there is no Python or CPU fallback for the
projection.
"""
from __future__ import annotations

import ctypes as C
import os
import pathlib

_PKG = pathlib.Path(__file__).resolve().parent
LIBDIR = _PKG / "_lib"
# FASTMAP_B200_LIB selects an alternate build of the product (tuning sweeps)
PRODUCT_SO = pathlib.Path(os.environ.get("FASTMAP_B200_LIB", LIBDIR / "libfastmap_b200.so"))
SYNTH_SO = LIBDIR / "libfastmap_synth.so"

u64 = C.c_uint64
i64 = C.c_int64
PD = C.POINTER(C.c_double)
PU64 = C.POINTER(C.c_uint64)
PU32 = C.POINTER(C.c_uint32)
PI32 = C.POINTER(C.c_int32)
PI64 = C.POINTER(C.c_int64)
PU8 = C.POINTER(C.c_uint8)

FM_OK = 0
FM_ERR_INVALID_ARGUMENT = 1
FM_ERR_RUNTIME = 2
FM_ERR_DOMAIN = 3
FM_ERR_CUDA = 4
FM_ERR_NO_DEVICE = 5
FM_ERR_OOM = 6


class BuildParams(C.Structure):
    _fields_ = [
        ("cells_per_polygon", C.c_double),
        ("nx", i64),
        ("ny", i64),
        ("margin", C.c_double),
        ("device", C.c_int),
        ("build_on_gpu", C.c_int),
        ("threads", C.c_int),
        ("approx_epsilon", C.c_double),
    ]


class IndexStats(C.Structure):
    _fields_ = [
        ("n_polys", u64), ("n_rings", u64), ("n_vertices", u64), ("n_edges", u64),
        ("nx", i64), ("ny", i64),
        ("cells_empty", u64), ("cells_hit", u64), ("cells_boundary", u64),
        ("grid_bytes", u64), ("arena_bytes", u64), ("geometry_bytes", u64),
        ("record_edges", u64), ("record_cands", u64), ("record_breaks", u64),
        ("max_record_edges", u64), ("max_record_cands", u64),
        ("gx0", C.c_double), ("gx1", C.c_double), ("gy0", C.c_double), ("gy1", C.c_double),
        ("cell_w", C.c_double), ("cell_h", C.c_double), ("margin", C.c_double),
        ("build_seconds", C.c_double),
        ("built_on_gpu", C.c_int32), ("reserved0", C.c_int32),
        ("cells_split", u64), ("slots_phase1", u64), ("slots_total", u64),
        ("approx_epsilon", C.c_double), ("approx_grid_bytes", u64),
        ("query_grid_bytes", u64), ("query_block_log2", C.c_int32),
        ("approx_block_log2", C.c_int32), ("slots_double", u64),
        ("build_phase_seconds", C.c_double * 6),
    ]

    def as_dict(self) -> dict:
        d = {k: getattr(self, k) for k, _ in self._fields_}
        d["build_phase_seconds"] = list(d["build_phase_seconds"])
        return d


class AssignCountersC(C.Structure):
    _fields_ = [("pip_point_evaluations", u64), ("pip_calls", u64)]


class QueryCounters(C.Structure):
    _fields_ = [("points", u64), ("boundary_points", u64),
                ("candidate_tests", u64), ("edge_tests", u64)]


# every symbol include/fastmap_b200.h declares (tests check the export table)
EXPORTS = (
    "fm_status_string", "fm_last_error", "fm_version", "fm_index_build",
    "fm_index_destroy", "fm_index_stats_get", "fm_query", "fm_query_host",
    "fm_index_export", "fm_index_device", "fm_query_mode", "fm_query_host_mode",
    "fm_index_save", "fm_index_load", "fm_hierarchy_load", "fm_hierarchy_destroy",
    "fm_hierarchy_sizes", "fm_hierarchy_leaves", "fm_index_build_hierarchy",
    "fm_read_points_f64", "fm_write_assign_csv", "fm_simple_build", "fm_simple_destroy",
    "fm_simple_assign", "fm_simple_assign_host", "fm_index_set_query_path",
    "fm_index_query_plan", "fm_query_host_counted", "fm_multi_build", "fm_multi_query_host",
    "fm_multi_size", "fm_multi_replica", "fm_multi_destroy",
)

MODE_EXACT, MODE_APPROX = 0, 1  # fm_mode (CoverMode, cell_index.hpp:246)
PATH_AUTO, PATH_STREAM, PATH_BINNED = 0, 1, 2  # fm_query_path

_lib = None
_synth = None


def _load(path: pathlib.Path) -> C.CDLL:
    if not path.exists():
        raise RuntimeError(
            f"native library {path} is missing: run `make` (or __graft_entry__.build()); "
            "the B200 projection has no fallback implementation")
    return C.CDLL(str(path), mode=os.RTLD_NOW | getattr(os, "RTLD_LOCAL", 0))


def lib() -> C.CDLL:
    """The product library, with argtypes set."""
    global _lib
    if _lib is None:
        L = _load(PRODUCT_SO)
        L.fm_status_string.restype = C.c_char_p
        L.fm_status_string.argtypes = [C.c_int]
        L.fm_last_error.restype = C.c_char_p
        L.fm_last_error.argtypes = []
        L.fm_version.restype = C.c_char_p
        L.fm_version.argtypes = []
        L.fm_index_build.restype = C.c_int
        L.fm_index_build.argtypes = [PD, PU64, u64, PU64, u64, C.POINTER(BuildParams),
                                     C.POINTER(C.c_void_p)]
        L.fm_index_destroy.restype = None
        L.fm_index_destroy.argtypes = [C.c_void_p]
        L.fm_index_stats_get.restype = C.c_int
        L.fm_index_stats_get.argtypes = [C.c_void_p, C.POINTER(IndexStats)]
        L.fm_query.restype = C.c_int
        L.fm_query.argtypes = [C.c_void_p, C.c_void_p, u64, C.c_void_p, C.c_void_p,
                               C.c_void_p, C.c_void_p]
        L.fm_query_host.restype = C.c_int
        L.fm_query_host.argtypes = [C.c_void_p, PD, u64, PI32, PI64]
        L.fm_query_host.restype = C.c_int
        L.fm_query_mode.argtypes = [C.c_void_p, C.c_int, C.c_void_p, u64, C.c_void_p, C.c_void_p,
                                    C.c_void_p, C.c_void_p]
        L.fm_query_mode.restype = C.c_int
        L.fm_query_host_mode.argtypes = [C.c_void_p, C.c_int, PD, u64, PI32, PI64]
        L.fm_query_host_mode.restype = C.c_int
        L.fm_index_save.restype = C.c_int
        L.fm_index_save.argtypes = [C.c_void_p, C.c_char_p]
        L.fm_index_load.restype = C.c_int
        L.fm_index_load.argtypes = [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]
        L.fm_hierarchy_load.restype = C.c_int
        L.fm_hierarchy_load.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.fm_hierarchy_destroy.restype = None
        L.fm_hierarchy_destroy.argtypes = [C.c_void_p]
        L.fm_hierarchy_sizes.restype = C.c_int
        L.fm_hierarchy_sizes.argtypes = [C.c_void_p] + [PU64] * 5
        L.fm_hierarchy_leaves.restype = C.c_int
        L.fm_hierarchy_leaves.argtypes = [C.c_void_p, PD, PU64, PU64, PU32, C.c_char_p]
        L.fm_index_build_hierarchy.restype = C.c_int
        L.fm_index_build_hierarchy.argtypes = [C.c_void_p, C.POINTER(BuildParams),
                                               C.POINTER(C.c_void_p)]
        L.fm_read_points_f64.restype = C.c_int
        L.fm_read_points_f64.argtypes = [C.c_char_p, PD, PU64]
        L.fm_write_assign_csv.restype = C.c_int
        L.fm_write_assign_csv.argtypes = [C.c_char_p, PD, u64, PI32, C.c_void_p]
        L.fm_simple_build.restype = C.c_int
        L.fm_simple_build.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]
        L.fm_simple_destroy.restype = None
        L.fm_simple_destroy.argtypes = [C.c_void_p]
        L.fm_simple_assign.restype = C.c_int
        L.fm_simple_assign.argtypes = [C.c_void_p, C.c_int, C.c_void_p, u64, C.c_void_p, C.c_void_p,
                                       C.c_void_p, C.POINTER(AssignCountersC), C.c_void_p]
        L.fm_simple_assign_host.restype = C.c_int
        L.fm_simple_assign_host.argtypes = [C.c_void_p, C.c_int, PD, u64, PI32, PI32, PI32,
                                            C.POINTER(AssignCountersC)]
        L.fm_index_export.restype = C.c_int
        L.fm_index_export.argtypes = [C.c_void_p, PU32, PU64, PU8, PU64, PD]
        L.fm_index_device.restype = C.c_int
        L.fm_index_device.argtypes = [C.c_void_p]
        L.fm_query_host_counted.restype = C.c_int
        L.fm_query_host_counted.argtypes = [C.c_void_p, C.c_int, PD, u64, PI32, PI64,
                                            C.POINTER(QueryCounters)]
        L.fm_index_set_query_path.restype = C.c_int
        L.fm_index_set_query_path.argtypes = [C.c_void_p, C.c_int, C.c_double]
        L.fm_index_query_plan.restype = C.c_int
        L.fm_index_query_plan.argtypes = [C.c_void_p, u64, C.POINTER(C.c_int), PI32, PI32]
        L.fm_multi_build.restype = C.c_int
        L.fm_multi_build.argtypes = [PD, PU64, u64, PU64, u64, C.POINTER(BuildParams),
                                     C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_void_p)]
        L.fm_multi_query_host.restype = C.c_int
        L.fm_multi_query_host.argtypes = [C.c_void_p, C.c_int, PD, u64, PI32, PI64]
        L.fm_multi_size.restype = C.c_int
        L.fm_multi_size.argtypes = [C.c_void_p]
        L.fm_multi_replica.restype = C.c_void_p
        L.fm_multi_replica.argtypes = [C.c_void_p, C.c_int]
        L.fm_multi_destroy.restype = None
        L.fm_multi_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def synth() -> C.CDLL:
    global _synth
    if _synth is None:
        L = _load(SYNTH_SO)
        L.synth_tiling.restype = C.c_int
        L.synth_tiling.argtypes = [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                   C.c_double, C.c_double, C.c_double, C.c_double,
                                   C.c_double, u64, C.c_int, PD, PU64, PU64]
        L.synth_nested.restype = C.c_int
        L.synth_nested.argtypes = [C.c_uint32] * 7 + [C.c_double] * 6 + [u64, C.c_int, PD, PU64,
                                                                        PU64, PU32]
        L.synth_points_uniform.restype = C.c_int
        L.synth_nested_fmcb.argtypes = [C.c_uint32] * 7 + [C.c_double] * 6 + [u64, C.c_int, C.c_char_p]
        L.synth_nested_fmcb.restype = C.c_int
        L.synth_points_uniform.argtypes = [PD, u64, u64, u64, C.c_int, PD]
        L.synth_points_clustered.restype = C.c_int
        L.synth_points_clustered.argtypes = [PD, PD, u64, u64, u64, C.c_uint32,
                                             C.c_double, C.c_double, C.c_double,
                                             C.c_int, PD]
        L.synth_points_near_edge.restype = C.c_int
        L.synth_points_near_edge.argtypes = [PD, PU64, PU64, u64, C.c_double, C.c_double,
                                             C.c_double, C.c_double, PD, u64, u64, u64,
                                             C.c_int, PD]
        L.synth_points_uniform_dev.restype = C.c_int
        L.synth_points_uniform_dev.argtypes = [PD, u64, u64, u64, C.c_void_p, C.c_void_p]
        L.synth_points_clustered_dev.restype = C.c_int
        L.synth_points_clustered_dev.argtypes = [PD, PD, u64, u64, u64, C.c_uint32, C.c_double,
                                                 C.c_double, C.c_double, C.c_void_p, C.c_void_p]
        L.synth_points_near_edge_dev.restype = C.c_int
        L.synth_points_near_edge_dev.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, u64,
                                                 C.c_double, C.c_double, C.c_double, C.c_double,
                                                 PD, u64, u64, u64, C.c_void_p, C.c_void_p]
        _synth = L
    return _synth


def ptr(a, ctype):
    """ctypes pointer to a contiguous numpy array's data."""
    return a.ctypes.data_as(C.POINTER(ctype))


class FastmapError(Exception):
    pass


def check(status: int, what: str = "") -> None:
    """Raise the Python analogue of the reference's exception type."""
    if status == FM_OK:
        return
    L = lib()
    msg = (L.fm_last_error() or b"").decode() or L.fm_status_string(status).decode()
    if what:
        msg = f"{what}: {msg}"
    if status == FM_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)          # std::invalid_argument
    if status == FM_ERR_DOMAIN:
        raise ArithmeticError(msg)     # std::domain_error
    if status == FM_ERR_OOM:
        raise MemoryError(msg)
    raise RuntimeError(msg)            # std::runtime_error, CUDA, no device
