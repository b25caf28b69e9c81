// hierarchy.h -- the in-memory FMCB hierarchy behind the opaque fm_hierarchy
// (io.cpp reads it; simple.cu builds the simple-engine structures from it).
// Regions are numbered per level in depth-first file order, which is the
// reference's order: states, then counties state by state, then blocks in
// collect_leaves order (hierarchy.hpp:76-91).
#pragma once

#include <cstdint>
#include <vector>

namespace fm {

struct HierLevel {
  std::vector<double> vxy;                 // vertices of every ring, region order
  std::vector<std::uint64_t> ring_off{0};  // n_rings + 1
  std::vector<std::uint64_t> poly_ring{0}; // n_regions + 1
  std::vector<double> bbox;                // 4 per region, as stored in the file (x0, x1, y0, y1)
  std::vector<std::uint32_t> child_lo, child_hi;  // children in the next level (levels 0, 1)
  std::uint64_t n_regions() const { return poly_ring.size() - 1; }
};

}  // namespace fm

struct fm_hierarchy {
  std::uint64_t n_states = 0, n_counties = 0, n_leaves = 0;
  fm::HierLevel level[3];          // states, counties, blocks
  std::vector<std::uint32_t> scb;  // n_leaves x (state, county, block)
  std::vector<char> fips;          // n_leaves x 12
};
