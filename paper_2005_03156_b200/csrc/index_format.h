// index_format.h -- HBM layout of the cell index (shared by the host
// builder, the GPU builder and the query kernel).  DESIGN.md sec. 4 states
// the exactness argument this layout encodes.
//
// Grid.  A uniform nx x ny grid over the padded union bbox of all leaves.
// Cell (ix, iy) covers [gx0 + ix*w, gx0 + (ix+1)*w] x [gy0 + iy*h, ...].
// One u32 entry per cell, row-major:
//   0xFFFFFFFF            empty: no leaf contains any point of the cell
//   < 0x80000000          true hit: every point of the cell maps to this leaf
//   0x80000000 | k        boundary: record at arena byte offset 16*k
//
// Boundary record (16-byte aligned, little endian):
//   u16 n_edges, u16 n_cands, u16 n_words, u16 n_breaks   (header, 16 B)
//   u32 reserved[2]
//   n_edges x {f64 lo.lon, lo.lat, hi.lon, hi.lat}   oriented edges,
//       lo.lat < hi.lat, exactly the (lo, hi) the reference forms in
//       point_in_polygon (geometry.hpp:217-219); deduplicated across leaves
//   n_cands x {i32 leaf, u32 info}   ascending leaf id; info bit 0 = c0
//       (constant parity of the leaf's edges that lie wholly right of the
//       cell), bits 1..15 = number of latitude breakpoints of this leaf
//   n_cands x n_words x u32          per-leaf edge membership masks
//       (bit k set iff edge k occurs an odd number of times in the leaf)
//   pad to 8 B
//   n_breaks x f64                   breakpoints, per leaf in leaf order
//   pad to 16 B
// Point p in the cell maps to the first candidate whose parity
//   c0 ^ popc(cross_mask & mask) ^ #{b : p.lat > b}
// is odd, where bit k of cross_mask is the reference predicate of edge k at
// p.  A candidate with no edges and no breakpoints and c0 = 1 is a
// terminal: it always wins, and nothing after it is stored.
#pragma once

#include <cstdint>

#ifdef __CUDACC__
#define FM_HD __host__ __device__ __forceinline__
#else
#define FM_HD inline
#endif

namespace fm {

constexpr std::uint32_t kEmpty = 0xFFFFFFFFu;
constexpr std::uint32_t kRecordBit = 0x80000000u;
constexpr std::uint32_t kMaxLeaves = 0x7FFFFFFEu;
constexpr std::uint64_t kRecordAlign = 16;
constexpr std::uint32_t kMaxCands = 0xFFFFu;  // cell_index.hpp:339-341 limit
constexpr std::uint32_t kMaxRecordEdges = 0xFFFFu;
constexpr std::uint32_t kMaxBreaksPerCand = 0x7FFFu;

struct RecordHeader {
  std::uint16_t n_edges;
  std::uint16_t n_cands;
  std::uint16_t n_words;
  std::uint16_t n_breaks;
  std::uint32_t reserved0;
  std::uint32_t reserved1;
};
static_assert(sizeof(RecordHeader) == 16, "record header is 16 bytes");

FM_HD std::uint64_t record_bytes(std::uint32_t n_edges, std::uint32_t n_cands,
                                 std::uint32_t n_words, std::uint32_t n_breaks) {
  std::uint64_t b = 16 + 32ull * n_edges + 8ull * n_cands + 4ull * n_cands * n_words;
  b = (b + 7) & ~std::uint64_t{7};
  b += 8ull * n_breaks;
  return (b + 15) & ~std::uint64_t{15};
}
FM_HD std::uint64_t record_cands_offset(std::uint32_t n_edges) {
  return 16 + 32ull * n_edges;
}
FM_HD std::uint64_t record_masks_offset(std::uint32_t n_edges, std::uint32_t n_cands) {
  return 16 + 32ull * n_edges + 8ull * n_cands;
}
FM_HD std::uint64_t record_breaks_offset(std::uint32_t n_edges, std::uint32_t n_cands,
                                         std::uint32_t n_words) {
  std::uint64_t b = 16 + 32ull * n_edges + 8ull * n_cands + 4ull * n_cands * n_words;
  return (b + 7) & ~std::uint64_t{7};
}

// Grid geometry.  Cell rectangles are always formed by these two functions
// (builder) and points are always located by cell_of (kernel); the margin
// absorbs their rounding disagreement.
struct GridGeom {
  double gx0, gx1, gy0, gy1;  // padded domain
  double w, h;                // cell size
  double inv_w, inv_h;
  std::int64_t nx, ny;
  double margin;
};

FM_HD double cell_x0(const GridGeom& g, std::int64_t ix) {
  return g.gx0 + static_cast<double>(ix) * g.w;
}
FM_HD double cell_y0(const GridGeom& g, std::int64_t iy) {
  return g.gy0 + static_cast<double>(iy) * g.h;
}

}  // namespace fm
