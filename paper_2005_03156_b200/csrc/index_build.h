// index_build.h -- internal API of the cell-index builders (host and GPU).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "index_format.h"

namespace fm {

struct Soup {
  const double* vxy = nullptr;
  const std::uint64_t* ring_off = nullptr;
  std::uint64_t n_rings = 0;
  const std::uint64_t* poly_ring = nullptr;
  std::uint64_t n_polys = 0;
};

struct BuildOptions {
  double cells_per_polygon = 0.0;
  std::int64_t nx = 0, ny = 0;
  double margin = 0.0;
  int threads = 0;
  double approx_epsilon = 0.0;  // > 0: cell diagonal bound of a fast-approx cover
};

struct BuildStats {
  std::uint64_t n_edges = 0;
  std::uint64_t cells_empty = 0, cells_hit = 0, cells_boundary = 0;
  std::uint64_t record_edges = 0, record_cands = 0, record_breaks = 0;
  std::uint64_t max_record_edges = 0, max_record_cands = 0;
  std::uint64_t records_compact = 0, records_wide = 0;
  std::uint64_t records = 0;      // leaf slots + overflow records
  std::uint64_t records_overflow = 0;
  std::uint64_t cells_split = 0;  // split records (2x2 sub-cell nodes)
  std::uint64_t slots_double = 0; // double leaf slots (kind 4, 256 bytes)
  // GPU builder wall time per phase (s): 0 plan + upload, 1 spans + candidate
  // CSR, 2 contributions, 3 classify + phase-1 slots, 4 host phase 2,
  // 5 final arrays
  double phase_s[6] = {0, 0, 0, 0, 0, 0};
  // fast-approx epsilon finer than a uniform grid of <= 2^31 cells can
  // resolve: the grid is planned as for an exact index and approximate
  // queries are answered exactly (error 0 <= epsilon)
  bool approx_served_exact = false;
};

struct HostIndex {
  GridGeom g{};
  std::vector<std::uint32_t> grid;
  std::vector<std::uint8_t> slots;     // 128-byte boundary slots
  std::uint64_t n_slots = 0;
  std::uint64_t n_phase1_slots = 0;    // slots of cells that fit one slot (row-major first)
  std::vector<std::uint8_t> overflow;  // variable-size records past the split depth, + 512 B tail
  BuildStats stats;
};

// Exceptions mirror the reference's.
struct InvalidArgument : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};
struct RuntimeError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Validates the soup (rings >= 3 vertices like PolygonGeometry::add_ring,
// geometry.hpp:74-77; finite vertices; monotone offsets) and fixes the grid.
GridGeom plan_grid(const Soup& s, const BuildOptions& o, BuildStats* st);

// Host builder: C++ threads over grid rows.  Slot order (shared with the
// GPU builder, so both emit identical arrays): phase 1 -- every cell whose
// content fits one slot, row-major; phase 2 -- the split / overflow subtree
// of every other boundary cell, row-major, each subtree in post-order.
HostIndex build_index_host(const Soup& s, const BuildOptions& o);

// Phase 2 for cells the GPU builder deferred (linear ids, row-major, with
// their candidate leaves as a CSR); appends after `slot_base` slots and
// writes their grid entries.
void finish_deferred_cells(const Soup& s, const GridGeom& g, const BuildOptions& o,
                           const std::vector<std::int64_t>& cells,
                           const std::vector<std::uint64_t>& cand_off,
                           const std::vector<std::uint32_t>& cand_ids, std::uint64_t slot_base,
                           std::vector<std::uint32_t>& grid, std::vector<std::uint8_t>& slots_out,
                           std::vector<std::uint8_t>& ovf_out, BuildStats& stats);

// GPU builder (index_gpu.cu): same arrays as build_index_host, built on
// `device`; returns the device arrays (ownership to the caller) and fills
// out.g / out.stats / out.n_slots (no host copies of the arrays).
void build_index_gpu(const Soup& s, const BuildOptions& o, int device, HostIndex& out,
                     std::uint32_t** dev_grid, std::uint8_t** dev_slots, std::uint64_t* slots_len,
                     std::uint8_t** dev_overflow, std::uint64_t* overflow_len);

}  // namespace fm
