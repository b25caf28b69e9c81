// fastmap_gpu.hpp -- C++ drop-in adapter: the reference's build/query
// interface (proj/include/fastmap/cell_index.hpp) backed by the B200 C-ABI
// (include/fastmap_b200.h).
//
// Include it next to the reference headers (it uses the reference's own
// Point, LeafRegion, RegionHierarchy, CoverParams, CoverMode and
// AssignmentResult types) and link libfastmap_b200.so.  A call site that
// reads
//
//     const auto cover = build_cover(leaves, params);          // cell_index.hpp:396
//     const auto trie  = build_trie(cover, 4);                  // cell_index.hpp:453
//     auto res = query_leaves(trie, leaves, pts, CoverMode::exact);  // :527
//
// becomes
//
//     const auto index = fastmap::gpu::build_index(leaves, params);
//     auto res = fastmap::gpu::query_leaves(index, leaves, pts, CoverMode::exact);
//
// with the same AssignmentResult (state / county / block per point, -1 when
// unassigned) and the same exception types:
//   std::invalid_argument  bad parameters, fanout, approx query on an exact-only
//                          index, leaf-table
//                          mismatch, rings with < 3 vertices
//   std::runtime_error     reference limits, CUDA failures, no CUDA device
//                          (there is no CPU fallback)
// Answers follow exhaustive_assign semantics (synthetic.hpp:193-205): the
// first leaf, ascending, whose point_in_polygon is true; identical to
// query_leaves(exact) on every valid tiling.
#pragma once

#include <cstdint>
#include <cstdlib>
#include <filesystem>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "fastmap/cell_index.hpp"
#include "fastmap/geometry.hpp"
#include "fastmap/hierarchy.hpp"
#include "fastmap/simple_mapper.hpp"
#include "fastmap_b200.h"

#include <unistd.h>

namespace fastmap::gpu {

namespace detail {

[[noreturn]] inline void throw_status(fm_status s, const char* what) {
  std::string msg = std::string(what) + ": " + fm_last_error();
  switch (s) {
    case FM_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case FM_ERR_DOMAIN: throw std::domain_error(msg);
    default: throw std::runtime_error(msg);
  }
}

inline void check(fm_status s, const char* what) {
  if (s != FM_OK) throw_status(s, what);
}

struct IndexDeleter {
  void operator()(fm_index* p) const { fm_index_destroy(p); }
};

}  // namespace detail

/// Knobs of the GPU index beyond CoverParams (which is validated exactly as
/// validate_cover_params does, cell_index.hpp:382-394).
struct IndexParams {
  double cells_per_polygon = 0.0;  // 0 = auto
  int device = 0;                  // CUDA ordinal; -1 = host-only (export, no queries)
  int threads = 0;                 // host build threads (0 = all)
};

/// RAII owner of an fm_index (the CellCover + TrieIndex analogue).
class CellIndex {
 public:
  CellIndex() = default;
  explicit CellIndex(fm_index* p, std::size_t n_leaves) : h_(p), n_leaves_(n_leaves) {}
  fm_index* get() const { return h_.get(); }
  std::size_t n_leaves() const { return n_leaves_; }
  fm_index_stats stats() const {
    fm_index_stats s{};
    detail::check(fm_index_stats_get(h_.get(), &s), "fm_index_stats_get");
    return s;
  }

 private:
  std::unique_ptr<fm_index, detail::IndexDeleter> h_;
  std::size_t n_leaves_ = 0;
};

/// build_cover + build_trie over a leaf table (cell_index.hpp:396-400, :453).
inline CellIndex build_index(std::span<const LeafRegion> leaves,
                             const CoverParams& params = {},
                             const IndexParams& ip = {}) {
  validate_cover_params(params);  // the reference's own validation
  std::vector<double> vxy;
  std::vector<std::uint64_t> ring_off{0}, poly_ring{0};
  for (const LeafRegion& leaf : leaves) {
    if (leaf.geometry != nullptr) {
      const PolygonGeometry& g = *leaf.geometry;
      for (std::size_t r = 0; r < g.ring_starts.size(); ++r) {
        const std::uint32_t b = g.ring_starts[r];
        const std::uint32_t e = r + 1 < g.ring_starts.size()
                                    ? g.ring_starts[r + 1]
                                    : static_cast<std::uint32_t>(g.nodes.size());
        for (std::uint32_t v = b; v < e; ++v) {
          vxy.push_back(g.nodes[v].lon);
          vxy.push_back(g.nodes[v].lat);
        }
        ring_off.push_back(vxy.size() / 2);
      }
    }
    poly_ring.push_back(ring_off.size() - 1);
  }
  fm_build_params bp{};
  bp.cells_per_polygon = ip.cells_per_polygon;
  bp.device = ip.device;
  bp.build_on_gpu = ip.device >= 0 ? 1 : 0;
  bp.threads = ip.threads;
  bp.approx_epsilon = params.mode == CoverMode::approx ? params.epsilon : 0.0;
  fm_index* h = nullptr;
  detail::check(fm_index_build(vxy.data(), ring_off.data(), ring_off.size() - 1,
                               poly_ring.data(), poly_ring.size() - 1, &bp, &h),
                "fm_index_build");
  return CellIndex(h, leaves.size());
}

inline CellIndex build_index(const RegionHierarchy& h, const CoverParams& params = {},
                             const IndexParams& ip = {}) {
  const auto leaves = collect_leaves(h);  // hierarchy.hpp:76-91
  return build_index(leaves, params, ip);
}

/// Leaf id per point (collect_leaves position, -1 = none), host buffers.
inline std::vector<std::int32_t> project(const CellIndex& index, std::span<const Point> points,
                                         CoverMode mode = CoverMode::exact) {
  std::vector<std::int32_t> out(points.size());
  detail::check(fm_query_host_mode(index.get(),
                                   mode == CoverMode::approx ? FM_MODE_APPROX : FM_MODE_EXACT,
                                   reinterpret_cast<const double*>(points.data()), points.size(),
                                   out.data(), nullptr),
                "fm_query_host");
  return out;
}

/// Device-pointer variant (asynchronous on `stream`, a cudaStream_t).
inline void project_device(const CellIndex& index, const Point* d_points, std::size_t n,
                           std::int32_t* d_out, void* stream = nullptr,
                           std::int64_t* d_hist = nullptr) {
  detail::check(fm_query(index.get(), reinterpret_cast<const double*>(d_points), n, d_out,
                         d_hist, nullptr, stream),
                "fm_query");
}

/// query_leaves (cell_index.hpp:527-590): per-point (state, county, block)
/// set exactly as set_leaf does (cell_index.hpp:515-519).
inline AssignmentResult query_leaves(const CellIndex& index, std::span<const LeafRegion> leaves,
                                     std::span<const Point> points, CoverMode mode) {
  if (mode == CoverMode::approx && index.stats().approx_epsilon <= 0.0) {  // :532-535
    throw std::invalid_argument("approximate queries require an approximate-mode cover");
  }
  if (index.n_leaves() != leaves.size()) {
    throw std::invalid_argument("cover was built for a different hierarchy");
  }
  std::vector<std::int32_t> ids(points.size());
  fm_query_counters qc{};
  detail::check(fm_query_host_counted(index.get(),
                                      mode == CoverMode::approx ? FM_MODE_APPROX : FM_MODE_EXACT,
                                      reinterpret_cast<const double*>(points.data()), points.size(),
                                      ids.data(), nullptr, &qc),
                "fm_query_host_counted");
  AssignmentResult res;
  // the GPU index's own work counts (cell_index.hpp:582-583 counts the
  // reference cover's): one exact evaluation per point in a boundary cell
  // (pip_calls) and one (point, candidate leaf) parity per candidate tested
  // (pip_point_evaluations); true-hit and empty cells cost neither
  res.counters.pip_calls = qc.boundary_points;
  res.counters.pip_point_evaluations = qc.candidate_tests;
  res.state.assign(points.size(), -1);
  res.county.assign(points.size(), -1);
  res.block.assign(points.size(), -1);
  for (std::size_t i = 0; i < ids.size(); ++i) {
    if (ids[i] < 0) continue;
    const LeafRegion& leaf = leaves[static_cast<std::size_t>(ids[i])];
    res.state[i] = static_cast<std::int32_t>(leaf.state);
    res.county[i] = static_cast<std::int32_t>(leaf.county);
    res.block[i] = static_cast<std::int32_t>(leaf.block);
  }
  return res;
}

inline AssignmentResult query(const CellIndex& index, const RegionHierarchy& h,
                              std::span<const Point> points, CoverMode mode) {
  const auto leaves = collect_leaves(h);  // cell_index.hpp:592-596
  return query_leaves(index, leaves, points, mode);
}

/// index_stats(trie, cover) (cell_index.hpp:607-631) for the GPU index:
/// the reference's IndexStats fields mapped onto the cell grid --
/// interior_cells = true-hit cells, boundary_cells = cells with a boundary
/// slot, entry_bytes = the slot and overflow arenas (the cover entries'
/// role), node_bytes = the query grid (the trie's role; trie_nodes = 0, the
/// grid is direct-mapped), total_bytes = their sum.
inline IndexStats index_stats(const CellIndex& index) {
  const fm_index_stats s = index.stats();
  IndexStats r;
  r.interior_cells = static_cast<std::size_t>(s.cells_hit);
  r.boundary_cells = static_cast<std::size_t>(s.cells_boundary);
  r.trie_nodes = 0;
  r.entry_bytes = static_cast<std::size_t>(s.arena_bytes);
  r.node_bytes = static_cast<std::size_t>(s.query_grid_bytes ? s.query_grid_bytes : s.grid_bytes);
  r.total_bytes = r.entry_bytes + r.node_bytes;
  return r;
}

/// Index persistence (the FMCI save/load analogue, cell_index.hpp:641-726).
inline void save_index(const CellIndex& index, const std::string& path) {
  detail::check(fm_index_save(index.get(), path.c_str()), "fm_index_save");
}

inline CellIndex load_index(const std::string& path, int device = 0) {
  fm_index* h = nullptr;
  detail::check(fm_index_load(path.c_str(), device, &h), "fm_index_load");
  fm_index_stats s{};
  detail::check(fm_index_stats_get(h, &s), "fm_index_stats_get");
  return CellIndex(h, static_cast<std::size_t>(s.n_polys));
}

/// exhaustive_assign semantics (synthetic.hpp:193-205) on the GPU.
inline std::vector<std::int32_t> exhaustive_assign(std::span<const LeafRegion> leaves,
                                                   std::span<const Point> points,
                                                   int device = 0) {
  const auto index = build_index(leaves, CoverParams{}, IndexParams{0.0, device, 0});
  return project(index, points);
}

namespace detail {
struct HierarchyDeleter {
  void operator()(fm_hierarchy* p) const { fm_hierarchy_destroy(p); }
};
struct SimpleDeleter {
  void operator()(fm_simple* p) const { fm_simple_destroy(p); }
};
}  // namespace detail

/// The simple engine (the paper's hierarchical descent, simple_mapper.hpp:
/// 62-166) on the GPU.  The hierarchy is handed to the library as FMCB
/// bytes written by the reference's own save_hierarchy (hierarchy.hpp:
/// 187-198), through a temporary file.
class SimpleEngine {
 public:
  explicit SimpleEngine(const RegionHierarchy& h, int device = 0) {
    namespace fs = std::filesystem;
    // a fresh file of our own (mkstemp: O_EXCL, never follows a planted
    // link), removed on every exit path
    std::string tmpl = (fs::temp_directory_path() / "fastmap_gpu_XXXXXX").string();
    const int fd = ::mkstemp(tmpl.data());
    if (fd < 0) throw std::runtime_error("cannot create a temporary hierarchy file");
    ::close(fd);
    struct Remove {
      std::string p;
      ~Remove() {
        std::error_code ec;
        std::filesystem::remove(p, ec);
      }
    } guard{tmpl};
    save_hierarchy(h, tmpl);
    fm_hierarchy* hh = nullptr;
    detail::check(fm_hierarchy_load(tmpl.c_str(), &hh), "fm_hierarchy_load");
    h_.reset(hh);
    fm_simple* e = nullptr;
    detail::check(fm_simple_build(h_.get(), device, &e), "fm_simple_build");
    e_.reset(e);
  }
  fm_simple* get() const { return e_.get(); }

 private:
  std::unique_ptr<fm_hierarchy, detail::HierarchyDeleter> h_;
  std::unique_ptr<fm_simple, detail::SimpleDeleter> e_;
};

/// assign(h, points, mode) (simple_mapper.hpp:119-166): state / county /
/// block per point (local indices, -1 unresolved) and the reference's
/// AssignCounters, bit-identical to the reference's.
inline AssignmentResult assign(const SimpleEngine& engine, std::span<const Point> points,
                               AssignMode mode = AssignMode::relaxed) {
  static_assert(sizeof(Point) == 16, "Point is two doubles");
  AssignmentResult r;
  r.state.resize(points.size());
  r.county.resize(points.size());
  r.block.resize(points.size());
  fm_assign_counters c{};
  detail::check(fm_simple_assign_host(engine.get(),
                                      mode == AssignMode::strict ? FM_ASSIGN_STRICT : FM_ASSIGN_RELAXED,
                                      reinterpret_cast<const double*>(points.data()), points.size(),
                                      r.state.data(), r.county.data(), r.block.data(), &c),
                "fm_simple_assign_host");
  r.counters.pip_point_evaluations = c.pip_point_evaluations;
  r.counters.pip_calls = c.pip_calls;
  return r;
}

inline AssignmentResult assign(const RegionHierarchy& h, std::span<const Point> points,
                               AssignMode mode = AssignMode::relaxed, int device = 0) {
  return assign(SimpleEngine(h, device), points, mode);
}

}  // namespace fastmap::gpu
