// index_format.h -- HBM layout of the cell index (shared by the host
// builder, the GPU builder and the query kernel).  DESIGN.md sec. 4 states
// the exactness argument this layout encodes.
//
// Grid.  A uniform nx x ny grid over the padded union bbox of all leaves.
// Cell (ix, iy) covers [gx0 + ix*w, gx0 + (ix+1)*w] x [gy0 + iy*h, ...].
// One u32 entry per cell, row-major:
//   0xFFFFFFFF            empty: no leaf contains any point of the cell
//   < 0x80000000          true hit: every point of the cell maps to this leaf
//   0x80000000 | h<<30 | d<<29 | k  boundary: slot k (< 2^29 - 1) of the
//                         slot arena (128 bytes each); h = 1 when the slot's
//                         content lies in its first 64 bytes, so the query
//                         fetches only those (two sectors instead of four);
//                         d = 1 when slot k is a double slot (kind 4, slots
//                         k and k+1), so the query can batch those apart
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
//  kind 1, leaf (<= 4 candidates, <= 2 breakpoints, <= 5 chain vertices),
//  laid out so the common cells -- <= 2 candidates and either <= 2
//  vertices with <= 1 breakpoint or 3 vertices with none -- live in the
//  first 64 bytes:
//   +0   u8 kind=1, u8 n_verts, u8 n_cands, u8 n_breaks
//   +4   u8 edge_mask[0..1], u8 info[0..1]   info: bit 7 = c0, bits 0..1 = break mask
//   +8   i32 leaf[0..1]
//   +16  {f64 lon, f64 lat} vert[0..1]
//   +48  n_verts >= 3: vert[2];  else f64 break[0], 8 zero bytes
//   +64  u32 chain_mask          bit i set: vertex i starts a new chain
//                                (<= 3 vertices are always one chain)
//   +68  u8 edge_mask[2..3], u8 info[2..3]
//   +72  i32 leaf[2..3]
//   +80  n_verts >= 3: f64 break[0..1];  else f64 break[1], 8 zero bytes
//   +96  {f64 lon, f64 lat} vert[3..4]
//   Edge i joins vertex i and i+1 unless bit i+1 of chain_mask is set; it
//   is oriented exactly like the reference (lo = lower latitude,
//   geometry.hpp:219), which reproduces its (lo, hi) bit for bit.
//  kind 4, double leaf (256 bytes: slots k and k+1; the entry names k and
//   is never half) -- a cell that fits no leaf slot but <= 8 candidates,
//   <= 4 breakpoints and <= 10 chain vertices (typically a polygon corner:
//   3-4 leaves and their chains meeting at one vertex):
//   +0   u8 kind=4, u8 n_verts, u8 n_cands, u8 n_breaks
//   +4   u32 chain_mask
//   +8   i32 leaf[0..7]
//   +40  u16 edge_mask[0..7]
//   +56  u8 info[0..7]            bit 7 = c0, bits 0..3 = break mask
//   +64  f64 break[0..3]
//   +96  {f64 lon, f64 lat} vert[0..9]
//   The query stages the first 128 bytes like any slot and loads the
//   second (vert[2..9]) from global memory.
//  kind 3, split: a cell whose content does not fit one slot is split 2x2
//   (recursively, up to kMaxSplitDepth levels):
//   +8   f64 x0, f64 y0          lower-left corner of the split cell
//   +24  f64 inv_hw, f64 inv_hh  1 / child width, 1 / child height
//   +40  u32 child[4]            grid-format entries, index 2*j + i
//   Child (i, j) covers [x0 + i*hw, x0 + (i+1)*hw] x [y0 + j*hh, ...]; a
//   point goes to i = clamp(int((lon - x0) * inv_hw), 0, 1) (same for j).
//  kind 2, overflow (a cell whose compact record is <= kSmallRecordBytes,
//   or past the split depth): +8 u64 byte offset of a
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
constexpr std::uint32_t kHalfBit = 0x40000000u;     // slot content fits 64 bytes
// query-side block entries (fold, KParams): kRecordBit | kHalfBit | unit k
// names an exact compact sub-block at 16-byte unit k of the palette arena;
// with kSmallBit it is a one-unit "small" sub-block
constexpr std::uint32_t kSmallBit = 0x20000000u;
constexpr std::uint32_t kUnitMask = 0x1FFFFFFFu;
// cell / child entries: kRecordBit | kDoubleBit | k names double slot k
// (kind 4; never together with kHalfBit)
constexpr std::uint32_t kDoubleBit = 0x20000000u;
constexpr std::uint32_t kSlotIndexMask = 0x1FFFFFFFu;
constexpr std::uint64_t kMaxSlots = 0x1FFFFFFFull;  // k + flags never equals kEmpty
constexpr std::uint32_t kMaxLeaves = 0x7FFFFFFEu;
constexpr std::uint64_t kRecordAlign = 16;
constexpr std::uint32_t kMaxCands = 0xFFFFu;  // cell_index.hpp:339-341 limit
constexpr std::uint32_t kMaxRecordEdges = 0xFFFFu;
constexpr std::uint32_t kMaxBreaksPerCand = 0x7FFFu;

// slot kinds
constexpr std::uint8_t kSlotLeaf = 1;
constexpr std::uint8_t kSlotOverflow = 2;
constexpr std::uint8_t kSlotSplit = 3;
constexpr std::uint8_t kSlotDouble = 4;
constexpr std::uint32_t kDblMaxCands = 8;
constexpr std::uint32_t kDblMaxBreaks = 4;
constexpr std::uint32_t kDblMaxVerts = 10;
constexpr std::uint64_t kSlotBytes = 128;
constexpr std::uint32_t kSlotMaxCands = 4;
constexpr std::uint32_t kSlotMaxBreaks = 2;
constexpr std::uint32_t kSlotMaxVerts = 5;
constexpr int kMaxSplitDepth = 6;
// A boundary cell that does not fit one slot but whose compact record is at
// most this many bytes gets that record (overflow slot) instead of a split.
constexpr std::uint64_t kSmallRecordBytes = 256;

// Grid/child entry of slot k: split and overflow slots use only their first
// 64 bytes; so does a leaf slot with <= 2 candidates and either <= 2
// vertices and <= 1 breakpoint or 3 vertices and none (the layout above);
// a double slot never does.
FM_HD bool leaf_slot_half(std::uint32_t nv, std::uint32_t nc, std::uint32_t nb) {
  return nc <= 2 && ((nv <= 2 && nb <= 1) || (nv == 3 && nb == 0));
}
FM_HD std::uint32_t slot_entry(std::uint64_t k, std::uint32_t kind, std::uint32_t nv,
                               std::uint32_t nc, std::uint32_t nb) {
  const bool half = kind == kSlotSplit || kind == kSlotOverflow ||
                    (kind == kSlotLeaf && leaf_slot_half(nv, nc, nb));
  return kRecordBit | (half ? kHalfBit : 0u) | (kind == kSlotDouble ? kDoubleBit : 0u) |
         static_cast<std::uint32_t>(k);
}
// same, from the slot's first 4 bytes (u8 kind, nv, nc, nb)
FM_HD std::uint32_t slot_entry_hdr(std::uint64_t k, std::uint32_t h) {
  return slot_entry(k, h & 0xFFu, (h >> 8) & 0xFFu, (h >> 16) & 0xFFu, h >> 24);
}
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
