// index_format.h -- HBM layout of the cell index (shared by the host
// builder, the GPU builder and the query kernel).  DESIGN.md sec. 4 states
// the exactness argument this layout encodes.
//
// Grid.  A uniform nx x ny grid over the padded union bbox of all leaves.
// Cell (ix, iy) covers [gx0 + ix*w, gx0 + (ix+1)*w] x [gy0 + iy*h, ...].
// One u32 entry per cell, row-major:
//   0xFFFFFFFF            empty: no leaf contains any point of the cell
//   < 0x80000000          true hit: every point of the cell maps to this leaf
//   0x80000000 | k        boundary: slot k of the slot arena (128 bytes each)
//
// A boundary cell's slot lists its candidate leaves in ascending id order
// and the exact (fp64) polygon edges near the cell.  Point p maps to the
// first candidate whose parity
//     c0  ^  popc(cross_mask & edge_mask)  ^  popc(break_mask & {b : p.lat > b})
// is odd, where bit i of cross_mask is the reference predicate
// (geometry.hpp:214-225) of edge i at p.  c0 is the constant parity of the
// leaf's edges lying wholly right of the cell; the breakpoints are the
// latitudes where that constant changes inside the cell's slab.  A
// candidate with no edges, no breakpoints and c0 = 1 is terminal.
//
// Slot kinds (128 bytes, 128-byte aligned, little endian):
//  kind 1, leaf (<= 4 candidates, <= 2 breakpoints, <= 5 chain vertices):
//   +0   u8 kind=1, u8 n_verts, u8 n_cands, u8 n_breaks
//   +4   u32 chain_mask          bit i set: vertex i starts a new chain
//   +8   i32 leaf[4]
//   +24  u8 edge_mask[4]
//   +28  u8 info[4]              bit 7 = c0, bits 0..1 = break mask
//   +32  f64 break[2]
//   +48  {f64 lon, f64 lat} vert[5]
//   Edge i joins vertex i and i+1 unless bit i+1 of chain_mask is set; it
//   is oriented exactly like the reference (lo = lower latitude,
//   geometry.hpp:219), which reproduces its (lo, hi) bit for bit.
//  kind 3, split: a cell whose content does not fit one slot is split 2x2
//   (recursively, up to kMaxSplitDepth levels):
//   +8   f64 x0, f64 y0          lower-left corner of the split cell
//   +24  f64 inv_hw, f64 inv_hh  1 / child width, 1 / child height
//   +40  u32 child[4]            grid-format entries, index 2*j + i
//   Child (i, j) covers [x0 + i*hw, x0 + (i+1)*hw] x [y0 + j*hh, ...]; a
//   point goes to i = clamp(int((lon - x0) * inv_hw), 0, 1) (same for j).
//  kind 2, overflow (past the split depth): +8 u64 byte offset of a
//   variable-size record in the overflow arena, one of
//   compact (kind 1, fits when n_verts <= 32, n_cands <= 15, n_breaks <= 7):
//     +0   u8 kind=1, u8 n_verts, u8 n_cands, u8 n_breaks
//     +4   u32 chain_mask
//     +8   n_cands x {i32 leaf, u32 edge_mask}
//          n_cands x u8 info     bit 7 = c0, bits 0..6 = break mask
//          pad to 8;  n_breaks x f64;  pad to 16;  n_verts x {f64, f64}
//   wide (kind 2, anything else):
//     +0   u8 kind=2, u8 0, u16 n_words, u16 n_edges, u16 n_cands,
//          u16 n_breaks, u16 0, u32 0
//     +16  n_edges x {f64 lo.lon, lo.lat, hi.lon, hi.lat}  (lo.lat < hi.lat)
//          n_cands x {i32 leaf, u32 info}  info bit 0 = c0, bits 1..15 = #breaks
//          n_cands x n_words x u32        edge masks
//          pad to 8;  sum(#breaks) x f64 (per candidate, in order);  pad to 16
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

// slot kinds
constexpr std::uint8_t kSlotLeaf = 1;
constexpr std::uint8_t kSlotOverflow = 2;
constexpr std::uint8_t kSlotSplit = 3;
constexpr std::uint64_t kSlotBytes = 128;
constexpr std::uint32_t kSlotMaxCands = 4;
constexpr std::uint32_t kSlotMaxBreaks = 2;
constexpr std::uint32_t kSlotMaxVerts = 5;
constexpr int kMaxSplitDepth = 6;
// overflow record kinds
constexpr std::uint8_t kKindCompact = 1;
constexpr std::uint8_t kKindWide = 2;
constexpr std::uint32_t kCompactMaxVerts = 32;
constexpr std::uint32_t kCompactMaxCands = 15;
constexpr std::uint32_t kCompactMaxBreaks = 7;

FM_HD std::uint64_t align_up(std::uint64_t v, std::uint64_t a) { return (v + a - 1) & ~(a - 1); }

// ---- compact record offsets ----
FM_HD std::uint64_t compact_info_offset(std::uint32_t nc) { return 8 + 8ull * nc; }
FM_HD std::uint64_t compact_breaks_offset(std::uint32_t nc) {
  return align_up(8 + 8ull * nc + nc, 8);
}
FM_HD std::uint64_t compact_verts_offset(std::uint32_t nc, std::uint32_t nb) {
  return align_up(compact_breaks_offset(nc) + 8ull * nb, 16);
}
FM_HD std::uint64_t compact_bytes(std::uint32_t nv, std::uint32_t nc, std::uint32_t nb) {
  return compact_verts_offset(nc, nb) + 16ull * nv;
}

// ---- wide record offsets ----
FM_HD std::uint64_t wide_cands_offset(std::uint32_t ne) { return 16 + 32ull * ne; }
FM_HD std::uint64_t wide_masks_offset(std::uint32_t ne, std::uint32_t nc) {
  return 16 + 32ull * ne + 8ull * nc;
}
FM_HD std::uint64_t wide_breaks_offset(std::uint32_t ne, std::uint32_t nc, std::uint32_t nw) {
  return align_up(wide_masks_offset(ne, nc) + 4ull * nc * nw, 8);
}
FM_HD std::uint64_t wide_bytes(std::uint32_t ne, std::uint32_t nc, std::uint32_t nw,
                               std::uint32_t nb) {
  return align_up(wide_breaks_offset(ne, nc, nw) + 8ull * nb, 16);
}

// Grid geometry.  Cell rectangles are always formed by cell_x0/cell_y0
// (builder) and points are always located by the kernel's
// (p - g0) * inv truncation; the margin absorbs their rounding
// disagreement.
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
