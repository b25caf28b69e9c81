// query.cuh -- device side of the projection: point location and the exact
// fp64 crossing-number evaluation of boundary records (index_format.h).
//
// Parity with the reference rests on ray_crosses below evaluating
//   (hi.lon - lo.lon) * (p.lat - lo.lat) - (hi.lat - lo.lat) * (p.lon - lo.lon) > 0
// (geometry.hpp:170-174) as rounded subtractions and rounded products --
// never a fused multiply-add.  __dsub_rn/__dmul_rn are never contracted by
// nvcc, the library is also compiled with --fmad=false, and
// tests/test_sass.py checks the shipped SASS for DFMA.
#pragma once

#include <cstdint>

#include "index_format.h"

namespace fm {

struct KParams {
  const std::uint32_t* __restrict__ grid;     // flat grid (index_format.h)
  const std::uint8_t* __restrict__ slots;     // 128-byte boundary slots
  const std::uint8_t* __restrict__ overflow;  // variable-size records
  // The query-side copy of the grid, folded into blocks of 2^ls x 2^ls
  // cells: a block entry is the common entry of a uniform block, or
  // kRecordBit | k for sub-block k (2^(2 ls) entries, row-major) -- so the
  // first level stays L2-resident.
  const std::uint32_t* __restrict__ blocks;
  const std::uint32_t* __restrict__ sub;
  const std::uint32_t* __restrict__ pal;      // palette sub-blocks (kRecordBit | kHalfBit | k)
  double gx0, gy0, inv_w, inv_h;
  double ax0, ax1, ay0, ay1;  // acceptance box = padded domain intersect world box
  int nx, ny;
  int bnx, ls;                // blocks per row, log2 block side
  int compact;                // `pal` format: 0 approx palettes, 1 exact compact sub-blocks
};

__device__ __forceinline__ const std::uint8_t* slot_ptr(const KParams& P, std::uint32_t e) {
  return P.slots + static_cast<std::size_t>(e & kSlotIndexMask) * kSlotBytes;
}

__device__ __forceinline__ bool ray_crosses(double px, double py, double lx,
                                            double ly, double hx, double hy) {
  const double a = __dmul_rn(__dsub_rn(hx, lx), __dsub_rn(py, ly));
  const double b = __dmul_rn(__dsub_rn(hy, ly), __dsub_rn(px, lx));
  return __dsub_rn(a, b) > 0.0;
}

// Crossing bit of the edge (a, b) at p, oriented like geometry.hpp:217-220.
__device__ __forceinline__ std::uint32_t edge_bit(double px, double py, double ax,
                                                  double ay, double bx, double by) {
  const bool up = ay < by;
  const double lx = up ? ax : bx, ly = up ? ay : by;
  const double hx = up ? bx : ax, hy = up ? by : ay;
  return (ly < py && py <= hy && ray_crosses(px, py, lx, ly, hx, hy)) ? 1u : 0u;
}

// Grid entries of kN points (kEmpty outside the acceptance box, which also
// rejects NaN: every comparison with NaN is false), phased so every point's
// loads are in flight together: block entries first, then the second level
// as predicated loads rather than divergent branches, then the decode.
// kExact: exact grid (compact sub-blocks: two 16-byte loads;
// full: one 4-byte load); else an approx cover (palettes: one 16-byte load,
// or two for 8x8 blocks; full: one 4-byte load).
// kLs >= 0: the fold's block size as a compile-time constant (the query
// kernels are instantiated per block size); -1: read it from ls.
template <int kN, bool kExact, int kLs = -1>
__device__ __forceinline__ void locate_n(const KParams& P, const double2 (&p)[kN],
                                         std::uint32_t (&e)[kN]) {
  std::uint32_t be[kN];
  int cc[kN];
  const int ls = kLs >= 0 ? kLs : P.ls;
  const int m = (1 << ls) - 1;
#pragma unroll
  for (int u = 0; u < kN; ++u) {
    const double px = p[u].x, py = p[u].y;
    const bool in = px >= P.ax0 && px <= P.ax1 && py >= P.ay0 && py <= P.ay1;
    int ix = in ? static_cast<int>(__dmul_rn(__dsub_rn(px, P.gx0), P.inv_w)) : 0;
    int iy = in ? static_cast<int>(__dmul_rn(__dsub_rn(py, P.gy0), P.inv_h)) : 0;
    ix = min(max(ix, 0), P.nx - 1);
    iy = min(max(iy, 0), P.ny - 1);
    cc[u] = ((iy & m) << ls) + (ix & m);
    be[u] = in ? __ldg(P.blocks + static_cast<std::size_t>(iy >> ls) * static_cast<std::size_t>(P.bnx) +
                       (ix >> ls))
               : kEmpty;
  }
  const uint4* pal4 = reinterpret_cast<const uint4*>(P.pal);
  if (kExact) {
    // compact sub-blocks in 16-byte units: small (one unit: value[2], slot
    // base, 2-bit codes -- 0/1 value, 2 slot base + rank, 3 empty) or
    // compact (two units: value[3], slot base, 4-bit codes, half mask)
#pragma unroll
    for (int u = 0; u < kN; ++u) {
      const std::uint32_t x = be[u];
      const bool rec = ls != 0 && x != kEmpty && x >= kRecordBit;
      const bool cmp = rec && (x & kHalfBit);
      const bool small = x & kSmallBit;
      const std::size_t k = x & kUnitMask;
      uint4 a = make_uint4(0u, 0u, 0u, 0u), b = a;
      std::uint32_t f = x;
      if (cmp) a = __ldg(pal4 + k);
      if (cmp && !small) b = __ldg(pal4 + k + 1);
      if (rec && !cmp) f = __ldg(P.sub + ((x & kSlotIndexMask) << (2 * ls)) + cc[u]);
      const int c = cc[u];
      std::uint32_t ce;
      if (small) {
        const std::uint32_t code = (a.w >> (2 * c)) & 3u;
        const std::uint32_t eq2 = (a.w >> 1) & ~a.w & 0x55555555u;
        const std::uint32_t rank = __popc(eq2 & ((1u << (2 * c)) - 1u));
        ce = code == 0u ? a.x : (code == 1u ? a.y : (code == 2u ? (kRecordBit | (a.z + rank)) : kEmpty));
      } else {  // value[3], slot base, 4-bit codes[16], half mask
        const std::uint32_t code = ((c < 8 ? b.x : b.y) >> (4 * (c & 7))) & 15u;
        const std::uint32_t off = (code - 4u) & 31u;
        ce = code < 3u ? (code == 0 ? a.x : (code == 1 ? a.y : a.z))
                       : (kRecordBit | (((b.z >> off) & 1u) ? kHalfBit : 0u) | (a.w + off));
      }
      e[u] = cmp ? ce : f;
    }
    return;
  }
  const bool two = ls == 3;  // 32-byte approx palettes
#pragma unroll
  for (int u = 0; u < kN; ++u) {
    const std::uint32_t x = be[u];
    const bool rec = ls != 0 && x != kEmpty && x >= kRecordBit;
    const bool cmp = rec && (x & kHalfBit);
    const std::size_t k = x & kSlotIndexMask;
    uint4 a = make_uint4(0u, 0u, 0u, 0u), b = a;
    std::uint32_t f = x;
    if (cmp) a = __ldg(pal4 + (two ? 2 * k : k));
    if (cmp && two) b = __ldg(pal4 + 2 * k + 1);
    if (rec && !cmp) f = __ldg(P.sub + (k << (2 * ls)) + cc[u]);
    const int c = cc[u];
    // value[3], 2-bit codes
    const std::uint32_t wsel = (c >> 4) == 0 ? b.x : ((c >> 4) == 1 ? b.y : ((c >> 4) == 2 ? b.z : b.w));
    const std::uint32_t word = two ? wsel : a.w;
    const std::uint32_t code = (word >> (2 * (c & 15))) & 3u;
    const std::uint32_t ce = code == 0 ? a.x : (code == 1 ? a.y : a.z);
    e[u] = cmp ? ce : f;
  }
}

struct WorkCount {
  unsigned long long boundary = 0, cands = 0, edges = 0;
};

// Wide records (rare): evaluated straight from global memory.
template <bool kCount>
__device__ __noinline__ int resolve_wide(const std::uint8_t* __restrict__ rec, double px,
                                         double py, WorkCount& wc) {
  const uint4 h = __ldg(reinterpret_cast<const uint4*>(rec));
  const std::uint32_t n_words = h.x >> 16, n_edges = h.y & 0xFFFFu, n_cands = h.y >> 16;
  const double2* E = reinterpret_cast<const double2*>(rec + 16);
  const int2* C = reinterpret_cast<const int2*>(rec + wide_cands_offset(n_edges));
  const std::uint32_t* Mk =
      reinterpret_cast<const std::uint32_t*>(rec + wide_masks_offset(n_edges, n_cands));
  const double* B =
      reinterpret_cast<const double*>(rec + wide_breaks_offset(n_edges, n_cands, n_words));
  std::uint32_t boff = 0;
  for (std::uint32_t c = 0; c < n_cands; ++c) {
    const int2 cd = __ldg(C + c);
    const std::uint32_t info = static_cast<std::uint32_t>(cd.y);
    const std::uint32_t nb = info >> 1;
    std::uint32_t par = info & 1u;
    for (std::uint32_t w = 0; w < n_words; ++w) {
      std::uint32_t bits = __ldg(Mk + static_cast<std::size_t>(c) * n_words + w);
      while (bits) {
        const std::uint32_t k = w * 32 + (__ffs(bits) - 1);
        bits &= bits - 1;
        const double2 lo = __ldg(E + 2 * k);
        const double2 hi = __ldg(E + 2 * k + 1);
        if (lo.y < py && py <= hi.y) {
          if (kCount) wc.edges++;
          if (ray_crosses(px, py, lo.x, lo.y, hi.x, hi.y)) par ^= 1u;
        }
      }
    }
    for (std::uint32_t b = 0; b < nb; ++b) par ^= (py > __ldg(B + boff + b)) ? 1u : 0u;
    boff += nb;
    if (kCount) wc.cands++;
    if (par & 1u) return cd.x;
  }
  return -1;
}

// Compact record.  `Rd` reads the record: from a shared-memory window
// (WinReader, fast path) or from global memory (GlobalReader).
struct GlobalReader {
  const std::uint8_t* __restrict__ rec;
  __device__ __forceinline__ double f64(std::uint32_t off) const {
    return __ldg(reinterpret_cast<const double*>(rec + off));
  }
  __device__ __forceinline__ std::uint32_t u32(std::uint32_t off) const {
    return __ldg(reinterpret_cast<const std::uint32_t*>(rec + off));
  }
};

// Record bytes staged in shared memory.
struct SmemReader {
  const std::uint8_t* win;
  __device__ __forceinline__ double f64(std::uint32_t off) const {
    return *reinterpret_cast<const double*>(win + off);
  }
  __device__ __forceinline__ std::uint32_t u32(std::uint32_t off) const {
    return *reinterpret_cast<const std::uint32_t*>(win + off);
  }
};

template <bool kCount, typename Rd>
__device__ __forceinline__ int resolve_compact(const Rd& R, std::uint32_t h, double px,
                                               double py, WorkCount& wc) {
  const std::uint32_t nv = (h >> 8) & 0xFFu, nc = (h >> 16) & 0xFFu, nb = h >> 24;
  const std::uint32_t chain = R.u32(4);
  const std::uint32_t voff = static_cast<std::uint32_t>(compact_verts_offset(nc, nb));
  // crossing mask over the vertex chains
  std::uint32_t m = 0;
  double ax = R.f64(voff), ay = R.f64(voff + 8);
  for (std::uint32_t i = 0; i + 1 < nv; ++i) {
    const double bx = R.f64(voff + 16 * (i + 1)), by = R.f64(voff + 16 * (i + 1) + 8);
    if (!((chain >> (i + 1)) & 1u)) {
      if (kCount) wc.edges++;
      m |= edge_bit(px, py, ax, ay, bx, by) << i;
    }
    ax = bx;
    ay = by;
  }
  std::uint32_t bm = 0;
  const std::uint32_t boff = static_cast<std::uint32_t>(compact_breaks_offset(nc));
  for (std::uint32_t j = 0; j < nb; ++j) bm |= (py > R.f64(boff + 8 * j)) ? (1u << j) : 0u;
  const std::uint32_t ioff = static_cast<std::uint32_t>(compact_info_offset(nc));
  for (std::uint32_t c = 0; c < nc; ++c) {
    const std::uint32_t mask = R.u32(12 + 8 * c);
    const std::uint32_t info = (R.u32((ioff + c) & ~3u) >> (8 * ((ioff + c) & 3u))) & 0xFFu;
    const std::uint32_t par = (info >> 7) ^ __popc(m & mask) ^ __popc(bm & info & 0x7Fu);
    if (kCount) wc.cands++;
    if (par & 1u) return static_cast<int>(R.u32(8 + 8 * c));
  }
  return -1;
}

__device__ __forceinline__ double as_f64(std::uint32_t lo, std::uint32_t hi) {
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(lo));
}

// Leaf slot (index_format.h, kind 1) held in registers as eight 16-byte
// chunks; every offset is static, every branch is a predicate.  For a
// half slot (kHalfBit) chunks 4..7 may hold stale bytes: every value read
// from them is masked by n_verts / n_cands / n_breaks.
template <bool kCount>
__device__ __forceinline__ int eval_leaf_slot(const uint4 (&c)[8], double px, double py,
                                              WorkCount& wc) {
  const std::uint32_t h = c[0].x;
  const std::uint32_t nv = (h >> 8) & 0xFFu, nc = (h >> 16) & 0xFFu, nb = h >> 24;
  const std::uint32_t chain = nv <= 3u ? 1u : c[4].x;  // <= 3 vertices: one chain
  double vx[kSlotMaxVerts], vy[kSlotMaxVerts];
#pragma unroll
  for (int k = 0; k < static_cast<int>(kSlotMaxVerts); ++k) {
    const uint4 v = c[k < 3 ? 1 + k : 3 + k];
    vx[k] = as_f64(v.x, v.y);
    vy[k] = as_f64(v.z, v.w);
  }
  std::uint32_t m = 0;
#pragma unroll
  for (int k = 0; k + 1 < static_cast<int>(kSlotMaxVerts); ++k) {
    if (static_cast<std::uint32_t>(k + 1) < nv && !((chain >> (k + 1)) & 1u)) {
      if (kCount) wc.edges++;
      m |= edge_bit(px, py, vx[k], vy[k], vx[k + 1], vy[k + 1]) << k;
    }
  }
  const bool v3 = nv >= 3u;
  const double b0 = v3 ? as_f64(c[5].x, c[5].y) : as_f64(c[3].x, c[3].y);
  const double b1 = v3 ? as_f64(c[5].z, c[5].w) : as_f64(c[5].x, c[5].y);
  const std::uint32_t bm = ((nb > 0u && py > b0) ? 1u : 0u) | ((nb > 1u && py > b1) ? 2u : 0u);
  const std::uint32_t ids[4] = {c[0].z, c[0].w, c[4].z, c[4].w};
  const std::uint32_t lo = c[0].y, hi = c[4].y;  // {mask, mask, info, info} per pair
  const std::uint32_t masks = (lo & 0xFFFFu) | (hi << 16);
  const std::uint32_t infos = (lo >> 16) | (hi & 0xFFFF0000u);
  int id = -1;
#pragma unroll
  for (int q = 3; q >= 0; --q) {  // descending, so the smallest odd candidate wins
    const std::uint32_t mk = (masks >> (8 * q)) & 0xFFu, inf = (infos >> (8 * q)) & 0xFFu;
    const std::uint32_t par = (inf >> 7) ^ __popc(m & mk) ^ __popc(bm & inf & 3u);
    if (static_cast<std::uint32_t>(q) < nc && (par & 1u)) id = static_cast<int>(ids[q]);
  }
  if (kCount) wc.cands += nc;
  return id;
}

// Double leaf slot (index_format.h, kind 4): a[] = its first 128 bytes (as
// staged), b[] = the second (vert[2..9]).  Static offsets, predicated like
// eval_leaf_slot.
template <bool kCount>
__device__ __forceinline__ int eval_double_slot(const uint4 (&a)[8], const uint4 (&b)[8], double px,
                                                double py, WorkCount& wc) {
  const std::uint32_t h = a[0].x;
  const std::uint32_t nv = (h >> 8) & 0xFFu, nc = (h >> 16) & 0xFFu, nb = h >> 24;
  const std::uint32_t chain = a[0].y;
  double vx[kDblMaxVerts], vy[kDblMaxVerts];
#pragma unroll
  for (int k = 0; k < static_cast<int>(kDblMaxVerts); ++k) {
    const uint4 v = k < 2 ? a[6 + k] : b[k - 2];
    vx[k] = as_f64(v.x, v.y);
    vy[k] = as_f64(v.z, v.w);
  }
  std::uint32_t m = 0;
#pragma unroll
  for (int k = 0; k + 1 < static_cast<int>(kDblMaxVerts); ++k) {
    if (static_cast<std::uint32_t>(k + 1) < nv && !((chain >> (k + 1)) & 1u)) {
      if (kCount) wc.edges++;
      m |= edge_bit(px, py, vx[k], vy[k], vx[k + 1], vy[k + 1]) << k;
    }
  }
  const double br[4] = {as_f64(a[4].x, a[4].y), as_f64(a[4].z, a[4].w), as_f64(a[5].x, a[5].y),
                        as_f64(a[5].z, a[5].w)};
  std::uint32_t bm = 0;
#pragma unroll
  for (int j = 0; j < 4; ++j) bm |= (static_cast<std::uint32_t>(j) < nb && py > br[j]) ? (1u << j) : 0u;
  const std::uint32_t ids[8] = {a[0].z, a[0].w, a[1].x, a[1].y, a[1].z, a[1].w, a[2].x, a[2].y};
  const std::uint32_t mk2[4] = {a[2].z, a[2].w, a[3].x, a[3].y};  // u16 edge masks, two per word
  int id = -1;
#pragma unroll
  for (int q = 7; q >= 0; --q) {  // descending, so the smallest odd candidate wins
    const std::uint32_t mk = (mk2[q >> 1] >> (16 * (q & 1))) & 0xFFFFu;
    const std::uint32_t inf = ((q < 4 ? a[3].z : a[3].w) >> (8 * (q & 3))) & 0xFFu;
    const std::uint32_t par = (inf >> 7) ^ __popc(m & mk) ^ __popc(bm & inf & 15u);
    if (static_cast<std::uint32_t>(q) < nc && (par & 1u)) id = static_cast<int>(ids[q]);
  }
  if (kCount) wc.cands += nc;
  return id;
}

// The second half of double slot `e` from global memory.
__device__ __forceinline__ void load_double_tail(const KParams& P, std::uint32_t e, uint4 (&b)[8]) {
  const uint4* g = reinterpret_cast<const uint4*>(slot_ptr(P, e) + kSlotBytes);
#pragma unroll
  for (int k = 0; k < 8; ++k) b[k] = __ldg(g + k);
}

// An overflow record (compact or wide) at byte offset `off` of the overflow
// arena, evaluated from global memory.
template <bool kCount>
__device__ __noinline__ int resolve_overflow(const KParams& P, std::uint64_t off, double px, double py,
                                             WorkCount& wc) {
  const std::uint8_t* rec = P.overflow + off;
  const std::uint32_t h = __ldg(reinterpret_cast<const std::uint32_t*>(rec));
  if ((h & 0xFFu) == kKindCompact) return resolve_compact<kCount>(GlobalReader{rec}, h, px, py, wc);
  return resolve_wide<kCount>(rec, px, py, wc);
}

// A boundary slot fetched straight from global memory (split descents and
// overflow records; rare).  Counts like the staged evaluation: a point is a
// boundary point once it reaches a leaf, double or overflow record.
template <bool kCount>
__device__ __noinline__ int resolve_slot_global(const KParams& P, std::uint32_t e, double px,
                                                double py, WorkCount& wc) {
  for (int depth = 0; depth <= kMaxSplitDepth + 1; ++depth) {
    const uint4* g = reinterpret_cast<const uint4*>(slot_ptr(P, e));
    uint4 c[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) c[k] = __ldg(g + k);
    const std::uint32_t kind = c[0].x & 0xFFu;
    if (kCount && kind != kSlotSplit) wc.boundary++;
    if (kind == kSlotLeaf) return eval_leaf_slot<kCount>(c, px, py, wc);
    if (kind == kSlotDouble) {
      uint4 b[8];
      load_double_tail(P, e, b);
      return eval_double_slot<kCount>(c, b, px, py, wc);
    }
    if (kind == kSlotOverflow) {
      return resolve_overflow<kCount>(P, (static_cast<std::uint64_t>(c[0].w) << 32) | c[0].z, px, py, wc);
    }
    // split
    const double x0 = as_f64(c[0].z, c[0].w), y0 = as_f64(c[1].x, c[1].y);
    const double ihw = as_f64(c[1].z, c[1].w), ihh = as_f64(c[2].x, c[2].y);
    int ci = static_cast<int>(__dmul_rn(__dsub_rn(px, x0), ihw));
    int cj = static_cast<int>(__dmul_rn(__dsub_rn(py, y0), ihh));
    ci = min(max(ci, 0), 1);
    cj = min(max(cj, 0), 1);
    const std::uint32_t ch[4] = {c[2].z, c[2].w, c[3].x, c[3].y};
    e = ch[2 * cj + ci];
    if (e == kEmpty) return -1;
    if (e < kRecordBit) return static_cast<int>(e);
  }
  return -1;  // unreachable for a well-formed index
}

// Smallest leaf id that a boundary entry's records list (its first
// candidate; split cells: the minimum over the subtree), kEmpty if none.
// Every listed candidate has boundary, breakpoints or a terminal inside the
// margin-expanded cell, so any point of the cell lies within the expanded
// cell diagonal of it -- the fast-approx fallback.
static __device__ __noinline__ std::uint32_t min_leaf_of_entry(const KParams& P, std::uint32_t e) {
  std::uint32_t best = kEmpty, stack[4 * (kMaxSplitDepth + 2)];
  int sp = 0;
  stack[sp++] = e;
  while (sp > 0) {
    const std::uint32_t x = stack[--sp];
    if (x == kEmpty) continue;
    if (x < kRecordBit) {
      best = min(best, x);
      continue;
    }
    const std::uint8_t* s = slot_ptr(P, x);
    const std::uint32_t h = __ldg(reinterpret_cast<const std::uint32_t*>(s));
    const std::uint32_t kind = h & 0xFFu;
    if (kind == kSlotLeaf || kind == kSlotDouble) {  // first candidate at +8 in both
      if ((h >> 16) & 0xFFu) best = min(best, __ldg(reinterpret_cast<const std::uint32_t*>(s + 8)));
    } else if (kind == kSlotSplit) {
      for (int k = 0; k < 4 && sp < static_cast<int>(sizeof(stack) / 4); ++k) {
        stack[sp++] = __ldg(reinterpret_cast<const std::uint32_t*>(s + 40) + k);
      }
    } else {  // overflow record
      const std::uint64_t off = __ldg(reinterpret_cast<const unsigned long long*>(s + 8));
      const std::uint8_t* rec = P.overflow + off;
      const uint2 rh = __ldg(reinterpret_cast<const uint2*>(rec));
      if ((rh.x & 0xFFu) == kKindCompact) {
        if ((rh.x >> 16) & 0xFFu) best = min(best, __ldg(reinterpret_cast<const std::uint32_t*>(rec + 8)));
      } else if (rh.y >> 16) {  // wide: n_edges = rh.y & 0xFFFF, n_cands = rh.y >> 16
        best = min(best, __ldg(reinterpret_cast<const std::uint32_t*>(rec + wide_cands_offset(rh.y & 0xFFFFu))));
      }
    }
  }
  return best;
}

}  // namespace fm
