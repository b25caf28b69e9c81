/*
 * fastmap_b200.h -- C-ABI of the B200-native point-to-block projection.
 *
 * This is the drop-in boundary for the reference's hot path (SURVEY.md
 * sec. 8b).  The reference is a header-only C++20 library with no FFI; its
 * path is four calls, each replaced here by a plain-pointer entry point:
 *
 *   reference (/root/reference/proj/include/fastmap/...)         here
 *   -------------------------------------------------------------  ---------------------
 *   CellCover build_cover(span<const LeafRegion>, const CoverParams&)
 *                                        cell_index.hpp:396-400   fm_index_build
 *   CellCover build_cover(const RegionHierarchy&, const CoverParams&)
 *                                        cell_index.hpp:402-405   fm_index_build
 *   TrieIndex build_trie(const CellCover&, int levels_per_node)
 *                                        cell_index.hpp:453-507   (folded into fm_index_build)
 *   AssignmentResult query_leaves(const TrieIndex&, span<const LeafRegion>,
 *                                 span<const Point>, CoverMode)
 *                                        cell_index.hpp:527-590   fm_query / fm_query_host
 *   vector<int32_t> exhaustive_assign(span<const LeafRegion>, span<const Point>)
 *                                        synthetic.hpp:193-205    fm_query (same answers)
 *   IndexStats index_stats(const TrieIndex&, const CellCover&)
 *                                        cell_index.hpp:616-631   fm_index_stats
 *
 * Semantics.  The output for point p is the leaf id (position in the
 * collect_leaves order, hierarchy.hpp:76-91) of the FIRST leaf, ascending,
 * whose reference point_in_polygon (geometry.hpp:214-225) is true, else -1;
 * points outside the lon/lat world box (cell_index.hpp:549-552) or with NaN
 * coordinates give -1.  This is exhaustive_assign's rule; it equals
 * query_leaves(..., exact) on every valid tiling and is bit-exact against
 * the reference fp64 predicate (no FMA contraction anywhere on the path).
 *
 * Polygon soup (one leaf = one polygon, possibly multi-ring, as
 * PolygonGeometry, geometry.hpp:64-87):
 *   vertex_lonlat[2*v], [2*v+1]        lon, lat of vertex v
 *   ring_offsets[r] .. [r+1]           vertices of ring r (open ring, >= 3
 *                                      vertices; the closing edge is implied,
 *                                      like PolygonGeometry::add_ring)
 *   poly_ring_offsets[p] .. [p+1]      rings of leaf p
 *
 * Errors map onto the reference's exception types (sec. 8b): the C++
 * adapter (include/fastmap_b200/fastmap_gpu.hpp) rethrows
 * FM_ERR_INVALID_ARGUMENT as std::invalid_argument, FM_ERR_RUNTIME as
 * std::runtime_error, FM_ERR_DOMAIN as std::domain_error; FM_ERR_CUDA and
 * FM_ERR_NO_DEVICE as std::runtime_error.  There is no CPU fallback: with
 * no usable CUDA device every compute call fails with FM_ERR_NO_DEVICE.
 *
 * Threading: a built index is immutable; fm_query may be called
 * concurrently on different streams.  One index lives on one device.
 */
#ifndef FASTMAP_B200_H_
#define FASTMAP_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum fm_status {
  FM_OK = 0,
  FM_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument in the reference */
  FM_ERR_RUNTIME = 2,          /* std::runtime_error */
  FM_ERR_DOMAIN = 3,           /* std::domain_error */
  FM_ERR_CUDA = 4,             /* CUDA runtime failure */
  FM_ERR_NO_DEVICE = 5,        /* no CUDA device: the product never falls back */
  FM_ERR_OOM = 6
} fm_status;

typedef struct fm_index fm_index;

/* Index build parameters (the analogue of CoverParams, cell_index.hpp:248-252).
 * Zero-initialise and set what you need. */
typedef struct fm_build_params {
  /* Grid resolution: cells per mean polygon bbox side.  0 = auto
   * (about 450M cells in total, 270M above 4M leaves, clamped to [4, 48]
   * per polygon side, and at least ~10M cells). */
  double cells_per_polygon;
  /* Explicit grid dimensions; both > 0 override cells_per_polygon. */
  int64_t nx, ny;
  /* Conservative classification margin in coordinate units; 0 = auto
   * (2^-40 * max(1, max |coordinate|)).  Must exceed fp64 rounding of the
   * predicate by a wide factor; see DESIGN.md sec. 4. */
  double margin;
  /* CUDA device ordinal the index lives on. */
  int device;
  /* 1 = build the cell index on the GPU (default path); 0 = host builder
   * (C++ threads).  Both produce bit-identical index arrays. */
  int build_on_gpu;
  /* Host build threads (0 = hardware concurrency). */
  int threads;
  /* > 0: also build the fast-approx cover (CoverMode::approx with this
   * epsilon, cell_index.hpp:248-252, :313-316): the grid is refined until
   * every cell's (margin-expanded) diagonal is <= epsilon and each boundary
   * cell gets a deemed leaf.  0 = exact-only index.  Values in
   * (0, level-30 cell diagonal) are rejected like validate_cover_params
   * (cell_index.hpp:382-394). */
  double approx_epsilon;
} fm_build_params;

/* CoverMode (cell_index.hpp:246). */
typedef enum fm_mode { FM_MODE_EXACT = 0, FM_MODE_APPROX = 1 } fm_mode;

typedef struct fm_index_stats {
  uint64_t n_polys, n_rings, n_vertices, n_edges;
  int64_t nx, ny;
  uint64_t cells_empty, cells_hit, cells_boundary;
  uint64_t grid_bytes, arena_bytes, geometry_bytes;
  uint64_t record_edges, record_cands, record_breaks; /* totals over records */
  uint64_t max_record_edges, max_record_cands;
  double gx0, gx1, gy0, gy1, cell_w, cell_h, margin;
  double build_seconds;
  int32_t built_on_gpu;   /* 1 when fm_index_build ran the GPU builder */
  int32_t reserved0;
  uint64_t cells_split;   /* 2x2 split nodes */
  uint64_t slots_phase1;  /* slots of cells that fit one slot */
  uint64_t slots_total;
  double approx_epsilon;      /* 0 for an exact-only index */
  uint64_t approx_grid_bytes; /* deemed-leaf grid of the approx cover */
  uint64_t query_grid_bytes;  /* query-side folded copy of the grid (blocks + sub-blocks) */
  int32_t query_block_log2;   /* its block side, log2 cells (0 = the flat grid itself) */
  int32_t approx_block_log2;  /* same for the approx cover */
  uint64_t slots_double;      /* 256-byte double leaf slots (polygon corners) */
  /* GPU builder wall time per phase, seconds: [0] plan + upload, [1] spans +
   * candidate CSR, [2] edge contributions, [3] classify + phase-1 slots,
   * [4] host phase 2 (cells that fit no phase-1 slot), [5] final arrays.
   * The renumbering / fold / approx cover after it are in build_seconds. */
  double build_phase_seconds[6];
} fm_index_stats;

/* Optional per-call work counters (diagnostics; device-side atomics). */
typedef struct fm_query_counters {
  uint64_t points;            /* points processed */
  uint64_t boundary_points;   /* points that landed in a boundary cell */
  uint64_t candidate_tests;   /* candidate leaves evaluated (reference: pip_point_evaluations) */
  uint64_t edge_tests;        /* fp64 crossing predicates evaluated */
} fm_query_counters;

const char* fm_status_string(fm_status s);
/* Message of the last failure on the calling thread ("" if none). */
const char* fm_last_error(void);
/* Version string of the library. */
const char* fm_version(void);

/* build_cover + build_trie (cell_index.hpp:396-405, :453-507).  Host
 * pointers.  Throws-equivalents: FM_ERR_INVALID_ARGUMENT for rings with < 3
 * vertices, non-finite vertices, bad offsets or params; FM_ERR_RUNTIME for a
 * boundary cell with more than 65535 candidates (cell_index.hpp:339-341). */
fm_status fm_index_build(const double* vertex_lonlat, const uint64_t* ring_offsets,
                         uint64_t n_rings, const uint64_t* poly_ring_offsets,
                         uint64_t n_polys, const fm_build_params* params,
                         fm_index** out_index);

void fm_index_destroy(fm_index* index);

fm_status fm_index_stats_get(const fm_index* index, fm_index_stats* out);

/* query_leaves(trie, leaves, points, CoverMode::exact) (cell_index.hpp:527-590)
 * on DEVICE pointers: d_lonlat = n interleaved (lon, lat) fp64 pairs (the
 * reference Point layout, geometry.hpp:17-22), d_out = n int32 leaf ids.
 * d_hist (nullable) = n_polys int64 counters incremented per assigned point.
 * d_counters (nullable) = device fm_query_counters accumulated into.
 * stream = cudaStream_t (NULL = legacy default stream).  Asynchronous. */
fm_status fm_query(const fm_index* index, const double* d_lonlat, uint64_t n,
                   int32_t* d_out, int64_t* d_hist, fm_query_counters* d_counters,
                   void* stream);

/* Same on HOST pointers: chunked and pipelined host->device copy, query and
 * device->host copy over internal streams; returns when h_out (and h_hist,
 * nullable, n_polys int64, accumulated into) are complete.  Pinned host
 * buffers give full PCIe overlap; pageable ones work but copy slower. */
fm_status fm_query_host(const fm_index* index, const double* h_lonlat, uint64_t n,
                        int32_t* h_out, int64_t* h_hist);

/* query_leaves(trie, leaves, points, mode) (cell_index.hpp:527-590) with an
 * explicit CoverMode.  FM_MODE_EXACT is fm_query.  FM_MODE_APPROX answers
 * boundary cells with their deemed leaf -- no crossing tests at all
 * (cell_index.hpp:558-560); it needs an index built with approx_epsilon > 0
 * (else FM_ERR_INVALID_ARGUMENT, cell_index.hpp:532-535).  A point whose
 * approx answer differs from the exact one lies within epsilon of the
 * answered leaf, and the answer is never -1 there. */
fm_status fm_query_mode(const fm_index* index, int mode, const double* d_lonlat, uint64_t n,
                        int32_t* d_out, int64_t* d_hist, fm_query_counters* d_counters,
                        void* stream);

/* fm_query_host with an explicit CoverMode. */
fm_status fm_query_host_mode(const fm_index* index, int mode, const double* h_lonlat,
                             uint64_t n, int32_t* h_out, int64_t* h_hist);

/* fm_query_host_mode that also accumulates the query's work counters into
 * the HOST struct `counters` (nullable): points, boundary points (the
 * points that needed crossing tests -- query_leaves' pending points,
 * cell_index.hpp:561-563), candidate leaves evaluated (its
 * pip_point_evaluations, :582-583) and fp64 edge predicates evaluated. */
fm_status fm_query_host_counted(const fm_index* index, int mode, const double* h_lonlat,
                                uint64_t n, int32_t* h_out, int64_t* h_hist,
                                fm_query_counters* counters);

/* Multi-GPU: run_chunked (parallel.hpp:30-82) one level up, for C++
 * callers owning several GPUs in one process.  fm_multi_build builds one
 * replica of the index (same arguments as fm_index_build; params->device is
 * ignored) on each of the n_devices distinct devices, concurrently.
 * fm_multi_query_host splits the host batch into contiguous, balanced
 * shards (the first n % N devices take one extra point), runs each shard
 * through the fm_query_host pipeline of its device from its own host
 * thread, and -- when h_hist (n_polys int64, accumulated into) is given --
 * sums the per-device histograms with one ncclAllReduce (NCCL is loaded at
 * run time; without it a histogram query fails with FM_ERR_RUNTIME).
 * h_out gets every point's id in input order, exactly as fm_query_host. */
typedef struct fm_multi fm_multi;
fm_status fm_multi_build(const double* vertex_lonlat, const uint64_t* ring_offsets,
                         uint64_t n_rings, const uint64_t* poly_ring_offsets, uint64_t n_polys,
                         const fm_build_params* params, const int* devices, int n_devices,
                         fm_multi** out);
fm_status fm_multi_query_host(fm_multi* multi, int mode, const double* h_lonlat, uint64_t n,
                              int32_t* h_out, int64_t* h_hist);
/* Number of replicas, and replica k (an ordinary fm_index owned by the multi). */
int fm_multi_size(const fm_multi* multi);
const fm_index* fm_multi_replica(const fm_multi* multi, int k);
void fm_multi_destroy(fm_multi* multi);

/* Query path of the exact mode.  Both paths answer every point with the
 * same locate / exact crossing code, so the ids are identical; they differ
 * only in memory order:
 *   FM_PATH_STREAM  points in input order: a streaming pass answers true-hit
 *                   and empty cells, a resolve pass the boundary points;
 *   FM_PATH_BINNED  points first partitioned by tile of the cell grid (the
 *                   analogue of query_leaves' pending sort, cell_index.hpp:
 *                   546-588), queried tile by tile so each tile's grid and
 *                   slots are fetched from HBM about once, then the ids are
 *                   gathered back into input order (24 B of scratch/point);
 *   FM_PATH_AUTO    (default) binned when the index is >= 1 GB with >= 25%
 *                   boundary cells and the batch has >= 4M points.
 * tile_bytes: index bytes per tile of the binned path (0 = 24 MB).  Not
 * synchronised with queries in flight: set it before querying. */
typedef enum fm_query_path { FM_PATH_AUTO = 0, FM_PATH_STREAM = 1, FM_PATH_BINNED = 2 } fm_query_path;
fm_status fm_index_set_query_path(fm_index* index, int path, double tile_bytes);
/* The path fm_query takes for a batch of n points (FM_PATH_STREAM or
 * FM_PATH_BINNED) and the binned path's tile side (log2 cells) and tile
 * count; any output may be NULL. */
fm_status fm_index_query_plan(const fm_index* index, uint64_t n, int* path, int32_t* tile_log2,
                              int32_t* n_tiles);

/* Copy of the index arrays to host memory (the FMCI-save analogue,
 * cell_index.hpp:641-664).  Two-call protocol: null buffers -> sizes.
 * arena = the 128-byte slot arena followed by the overflow arena;
 * geometry16 (nullable) receives gx0, gx1, gy0, gy1, cell_w, cell_h, inv_w,
 * inv_h, nx, ny, margin, n_polys, slot-arena bytes, 0, 0, 0. */
fm_status fm_index_export(const fm_index* index, uint32_t* grid, uint64_t* grid_len,
                          uint8_t* arena, uint64_t* arena_len, double* geometry16);

/* Device the index lives on. */
int fm_index_device(const fm_index* index);

/* ---- artifacts and IO ---------------------- */

/* Index persistence, the FMCI save/load analogue (cell_index.hpp:641-726):
 * a built index (grid, slot and overflow arenas, stats) to one file, and
 * back onto `device` (-1 = host-only) without rebuilding.  Errors are
 * FM_ERR_RUNTIME for unopenable, truncated or foreign files (bad magic or
 * version), like the reference's loaders. */
fm_status fm_index_save(const fm_index* index, const char* path);
fm_status fm_index_load(const char* path, int device, fm_index** out_index);

/* An FMCB region hierarchy (load_hierarchy, hierarchy.hpp:204-223) flattened
 * to its leaves in collect_leaves order (hierarchy.hpp:76-91): the polygon
 * soup fm_index_build takes, each leaf's (state, county, block) indices and
 * its 12-character FIPS code.  FM_ERR_RUNTIME for bad magic / version,
 * truncation, corrupt ring tables or count mismatches; FM_ERR_INVALID_ARGUMENT
 * for rings with < 3 vertices (geometry.hpp:75-77). */
typedef struct fm_hierarchy fm_hierarchy;
fm_status fm_hierarchy_load(const char* path, fm_hierarchy** out);
void fm_hierarchy_destroy(fm_hierarchy* h);
fm_status fm_hierarchy_sizes(const fm_hierarchy* h, uint64_t* n_states, uint64_t* n_counties,
                             uint64_t* n_leaves, uint64_t* n_rings, uint64_t* n_vertices);
/* Copies into caller buffers sized by fm_hierarchy_sizes (any may be NULL):
 * vertex_lonlat 2*n_vertices, ring_offsets n_rings+1, poly_ring_offsets
 * n_leaves+1, scb 3*n_leaves, fips12 12*n_leaves bytes (not terminated). */
fm_status fm_hierarchy_leaves(const fm_hierarchy* h, double* vertex_lonlat, uint64_t* ring_offsets,
                              uint64_t* poly_ring_offsets, uint32_t* scb, char* fips12);
/* fm_index_build over the hierarchy's leaves. */
fm_status fm_index_build_hierarchy(const fm_hierarchy* h, const fm_build_params* params,
                                   fm_index** out_index);

/* Raw little-endian f64 (lon, lat) pairs (read_points_f64, io.hpp:154-167).
 * Two-call protocol: lonlat = NULL -> *n = point count; else *n is the
 * buffer capacity in points and receives the count read. */
fm_status fm_read_points_f64(const char* path, double* lonlat, uint64_t* n);

/* ---- the simple engine ---------------------- */

/* The paper's hierarchical descent, assign(h, points, mode)
 * (simple_mapper.hpp:119-166), on the GPU: per level, the parent's children
 * whose file bbox strictly contains the point; strict mode takes the first
 * whose polygon holds it; relaxed mode takes a single candidate untested and
 * otherwise the first holding polygon, else the highest-indexed candidate.
 * Outputs are local (state, county-in-state, block-in-county) indices, -1
 * where unresolved. */
typedef enum fm_assign_mode { FM_ASSIGN_RELAXED = 0, FM_ASSIGN_STRICT = 1 } fm_assign_mode;  /* simple_mapper.hpp:24 */
typedef struct fm_assign_counters {  /* AssignCounters, simple_mapper.hpp:26-35 */
  uint64_t pip_point_evaluations;    /* (point, region) polygon tests */
  uint64_t pip_calls;                /* regions that received a polygon test */
} fm_assign_counters;
typedef struct fm_simple fm_simple;
fm_status fm_simple_build(const fm_hierarchy* h, int device, fm_simple** out);
void fm_simple_destroy(fm_simple* s);
/* Device pointers, asynchronous on `stream` unless `counters` (host struct,
 * accumulated into) is given, which makes the call synchronous. */
fm_status fm_simple_assign(const fm_simple* s, int mode, const double* d_lonlat, uint64_t n,
                           int32_t* d_state, int32_t* d_county, int32_t* d_block,
                           fm_assign_counters* counters, void* stream);
/* Host pointers (chunked copies); one batch for the counters. */
fm_status fm_simple_assign_host(const fm_simple* s, int mode, const double* lonlat, uint64_t n,
                                int32_t* state, int32_t* county, int32_t* block,
                                fm_assign_counters* counters);

/* The assignment CSV of the reference CLI (tools/fastmap.cpp:288-301):
 * header "idx,lon,lat,fips", one row per finite input point (non-finite rows
 * are skipped and keep their input index), coordinates as %.17g
 * (io.hpp:115-119), the leaf's FIPS code or an empty field for -1. */
fm_status fm_write_assign_csv(const char* path, const double* lonlat, uint64_t n, const int32_t* ids,
                              const fm_hierarchy* h);

#ifdef __cplusplus
}
#endif

#endif /* FASTMAP_B200_H_ */
