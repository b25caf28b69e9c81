// record_encode.h -- host encoder of boundary records (format: index_format.h).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <vector>

#include "index_build.h"
#include "index_format.h"

namespace fm {

struct Edge4 {
  double lx, ly, hx, hy;  // lo.lat < hi.lat
};
inline bool same_edge(const Edge4& a, const Edge4& b) {
  return std::memcmp(&a, &b, sizeof(Edge4)) == 0;
}

struct CandIn {
  std::uint32_t id;
  std::uint32_t c0;
  std::vector<std::uint32_t> edges;  // indices into the record's edge list (odd multiplicity)
  std::vector<double> breaks;        // ascending, distinct
};

struct EncodeStats {
  std::uint64_t compact = 0, wide = 0;
};

namespace detail {

inline bool same_pt(double ax, double ay, double bx, double by) {
  return std::memcmp(&ax, &bx, 8) == 0 && std::memcmp(&ay, &by, 8) == 0;
}

// Orders the edges into vertex chains (edges sharing bit-identical
// endpoints are consecutive).  Returns the vertex list, the chain-start
// mask and, per input edge, the index of its first vertex.
inline bool chain_edges(const std::vector<Edge4>& E, std::vector<double>& vx,
                        std::vector<double>& vy, std::uint32_t& chain_mask,
                        std::vector<std::uint32_t>& bit_of, std::uint32_t max_verts) {
  const std::size_t n = E.size();
  std::vector<char> used(n, 0);
  std::vector<std::uint32_t> order;  // edge ids along the final vertex list
  vx.clear();
  vy.clear();
  chain_mask = 0;
  bit_of.assign(n, 0);
  for (std::size_t s = 0; s < n; ++s) {
    if (used[s]) continue;
    used[s] = 1;
    // chain as a deque of (vertex, edge-to-next) built from edge s
    std::vector<double> cx{E[s].lx, E[s].hx}, cy{E[s].ly, E[s].hy};
    std::vector<std::int64_t> ce{static_cast<std::int64_t>(s)};
    for (bool grew = true; grew;) {
      grew = false;
      for (std::size_t k = 0; k < n; ++k) {
        if (used[k]) continue;
        const Edge4& e = E[k];
        const double tx = cx.back(), ty = cy.back();
        const double hx0 = cx.front(), hy0 = cy.front();
        if (same_pt(e.lx, e.ly, tx, ty)) {
          cx.push_back(e.hx); cy.push_back(e.hy); ce.push_back(static_cast<std::int64_t>(k));
        } else if (same_pt(e.hx, e.hy, tx, ty)) {
          cx.push_back(e.lx); cy.push_back(e.ly); ce.push_back(static_cast<std::int64_t>(k));
        } else if (same_pt(e.hx, e.hy, hx0, hy0)) {
          cx.insert(cx.begin(), e.lx); cy.insert(cy.begin(), e.ly);
          ce.insert(ce.begin(), static_cast<std::int64_t>(k));
        } else if (same_pt(e.lx, e.ly, hx0, hy0)) {
          cx.insert(cx.begin(), e.hx); cy.insert(cy.begin(), e.hy);
          ce.insert(ce.begin(), static_cast<std::int64_t>(k));
        } else {
          continue;
        }
        used[k] = 1;
        grew = true;
      }
    }
    const std::uint32_t base = static_cast<std::uint32_t>(vx.size());
    if (base + cx.size() > max_verts) return false;
    chain_mask |= 1u << base;
    for (std::size_t q = 0; q < ce.size(); ++q) bit_of[static_cast<std::size_t>(ce[q])] = base + static_cast<std::uint32_t>(q);
    vx.insert(vx.end(), cx.begin(), cx.end());
    vy.insert(vy.end(), cy.begin(), cy.end());
  }
  return true;
}

}  // namespace detail

// Appends one record to `arena` (which stays 16-byte granular) and returns
// its byte offset.  Throws RuntimeError on the reference's limits.
inline std::uint64_t encode_record(const std::vector<Edge4>& E, const std::vector<CandIn>& C,
                                   std::vector<std::uint8_t>& arena, EncodeStats* es) {
  if (C.size() > kMaxCands) throw RuntimeError("boundary cell with more than 65535 candidates");
  if (E.size() > kMaxRecordEdges) throw RuntimeError("boundary cell with more than 65535 edges");
  // distinct breakpoints across candidates
  std::vector<double> ub;
  for (const auto& c : C) {
    if (c.breaks.size() > kMaxBreaksPerCand) {
      throw RuntimeError("boundary cell leaf with more than 32767 latitude breakpoints");
    }
    for (double b : c.breaks) {
      if (std::find(ub.begin(), ub.end(), b) == ub.end()) ub.push_back(b);
    }
  }
  std::sort(ub.begin(), ub.end());
  std::vector<double> vx, vy;
  std::uint32_t chain_mask = 0;
  std::vector<std::uint32_t> bit_of;
  const bool compact = C.size() <= kCompactMaxCands && ub.size() <= kCompactMaxBreaks &&
                       detail::chain_edges(E, vx, vy, chain_mask, bit_of, kCompactMaxVerts);
  const std::uint64_t off = arena.size();
  if (compact) {
    const std::uint32_t nv = static_cast<std::uint32_t>(vx.size());
    const std::uint32_t nc = static_cast<std::uint32_t>(C.size());
    const std::uint32_t nb = static_cast<std::uint32_t>(ub.size());
    arena.resize(off + compact_bytes(nv, nc, nb), 0);
    std::uint8_t* r = arena.data() + off;
    r[0] = kKindCompact;
    r[1] = static_cast<std::uint8_t>(nv);
    r[2] = static_cast<std::uint8_t>(nc);
    r[3] = static_cast<std::uint8_t>(nb);
    std::memcpy(r + 4, &chain_mask, 4);
    for (std::uint32_t c = 0; c < nc; ++c) {
      const std::int32_t id = static_cast<std::int32_t>(C[c].id);
      std::uint32_t mask = 0;
      for (std::uint32_t e : C[c].edges) mask |= 1u << bit_of[e];
      std::uint8_t info = static_cast<std::uint8_t>((C[c].c0 & 1u) << 7);
      for (double b : C[c].breaks) {
        info |= static_cast<std::uint8_t>(
            1u << (std::lower_bound(ub.begin(), ub.end(), b) - ub.begin()));
      }
      std::memcpy(r + 8 + 8 * c, &id, 4);
      std::memcpy(r + 12 + 8 * c, &mask, 4);
      r[compact_info_offset(nc) + c] = info;
    }
    std::memcpy(r + compact_breaks_offset(nc), ub.data(), 8 * nb);
    std::uint8_t* v = r + compact_verts_offset(nc, nb);
    for (std::uint32_t k = 0; k < nv; ++k) {
      std::memcpy(v + 16 * k, &vx[k], 8);
      std::memcpy(v + 16 * k + 8, &vy[k], 8);
    }
    if (es) es->compact++;
    return off;
  }
  const std::uint32_t ne = static_cast<std::uint32_t>(E.size());
  const std::uint32_t nc = static_cast<std::uint32_t>(C.size());
  const std::uint32_t nw = (ne + 31) / 32;
  std::uint32_t nbt = 0;
  for (const auto& c : C) nbt += static_cast<std::uint32_t>(c.breaks.size());
  if (nbt > 0xFFFFu) throw RuntimeError("boundary cell with more than 65535 breakpoints");
  arena.resize(off + wide_bytes(ne, nc, nw, nbt), 0);
  std::uint8_t* r = arena.data() + off;
  r[0] = kKindWide;
  const std::uint16_t h16[4] = {static_cast<std::uint16_t>(nw), static_cast<std::uint16_t>(ne),
                                static_cast<std::uint16_t>(nc), static_cast<std::uint16_t>(nbt)};
  std::memcpy(r + 2, h16, 8);
  std::memcpy(r + 16, E.data(), 32ull * ne);
  std::uint8_t* cp = r + wide_cands_offset(ne);
  std::uint32_t* mp = reinterpret_cast<std::uint32_t*>(r + wide_masks_offset(ne, nc));
  double* bp = reinterpret_cast<double*>(r + wide_breaks_offset(ne, nc, nw));
  std::uint32_t bw = 0;
  for (std::uint32_t c = 0; c < nc; ++c) {
    const std::int32_t id = static_cast<std::int32_t>(C[c].id);
    const std::uint32_t info = (C[c].c0 & 1u) | (static_cast<std::uint32_t>(C[c].breaks.size()) << 1);
    std::memcpy(cp + 8 * c, &id, 4);
    std::memcpy(cp + 8 * c + 4, &info, 4);
    for (std::uint32_t e : C[c].edges) mp[c * nw + e / 32] |= 1u << (e % 32);
    for (double b : C[c].breaks) bp[bw++] = b;
  }
  if (es) es->wide++;
  return off;
}

// Bytes of the compact record encode_record would write for this content
// (compact_bytes), or 0 when it would need the wide format.
inline std::uint64_t compact_record_bytes(const std::vector<Edge4>& E, const std::vector<CandIn>& C) {
  if (C.size() > kCompactMaxCands) return 0;
  std::vector<double> ub;
  for (const auto& c : C) {
    for (double b : c.breaks) {
      if (std::find(ub.begin(), ub.end(), b) == ub.end()) ub.push_back(b);
    }
  }
  if (ub.size() > kCompactMaxBreaks) return 0;
  std::vector<double> vx, vy;
  std::uint32_t chain_mask = 0;
  std::vector<std::uint32_t> bit_of;
  if (!detail::chain_edges(E, vx, vy, chain_mask, bit_of, kCompactMaxVerts)) return 0;
  return compact_bytes(static_cast<std::uint32_t>(vx.size()), static_cast<std::uint32_t>(C.size()),
                       static_cast<std::uint32_t>(ub.size()));
}

// Encodes a leaf slot (index_format.h, kind 1) into out[128] if the cell's
// content fits one slot; returns false otherwise.
inline bool encode_slot(const std::vector<Edge4>& E, const std::vector<CandIn>& C,
                        std::uint8_t* out) {
  if (C.size() > kSlotMaxCands) return false;
  std::vector<double> ub;
  for (const auto& c : C) {
    for (double b : c.breaks) {
      if (std::find(ub.begin(), ub.end(), b) == ub.end()) ub.push_back(b);
    }
  }
  if (ub.size() > kSlotMaxBreaks) return false;
  std::sort(ub.begin(), ub.end());
  std::vector<double> vx, vy;
  std::uint32_t chain_mask = 0;
  std::vector<std::uint32_t> bit_of;
  if (!detail::chain_edges(E, vx, vy, chain_mask, bit_of, kSlotMaxVerts)) return false;
  std::memset(out, 0, kSlotBytes);
  out[0] = kSlotLeaf;
  out[1] = static_cast<std::uint8_t>(vx.size());
  out[2] = static_cast<std::uint8_t>(C.size());
  out[3] = static_cast<std::uint8_t>(ub.size());
  if (vx.size() > 3) std::memcpy(out + 64, &chain_mask, 4);  // <= 3 vertices: implied
  for (std::size_t c = 0; c < C.size(); ++c) {
    const std::int32_t id = static_cast<std::int32_t>(C[c].id);
    const std::size_t hi = c < 2 ? 0 : 64, j = c & 1;
    std::memcpy(out + hi + 8 + 4 * j, &id, 4);
    std::uint8_t mask = 0;
    for (std::uint32_t e : C[c].edges) mask |= static_cast<std::uint8_t>(1u << bit_of[e]);
    std::uint8_t info = static_cast<std::uint8_t>((C[c].c0 & 1u) << 7);
    for (double b : C[c].breaks) {
      info |= static_cast<std::uint8_t>(1u << (std::lower_bound(ub.begin(), ub.end(), b) - ub.begin()));
    }
    out[hi + 4 + j] = mask;
    out[hi + 6 + j] = info;
  }
  const bool v3 = vx.size() >= 3;
  for (std::size_t j = 0; j < ub.size(); ++j) {
    const std::size_t o = v3 ? 80 + 8 * j : (j == 0 ? 48 : 80);
    std::memcpy(out + o, &ub[j], 8);
  }
  for (std::size_t k = 0; k < vx.size(); ++k) {
    const std::size_t o = k < 3 ? 16 + 16 * k : 96 + 16 * (k - 3);
    std::memcpy(out + o, &vx[k], 8);
    std::memcpy(out + o + 8, &vy[k], 8);
  }
  return true;
}

// Encodes a double leaf slot (index_format.h, kind 4) into out[256] if the
// cell's content fits one; returns false otherwise.
inline bool encode_double_slot(const std::vector<Edge4>& E, const std::vector<CandIn>& C,
                               std::uint8_t* out) {
  if (C.size() > kDblMaxCands) return false;
  std::vector<double> ub;
  for (const auto& c : C) {
    for (double b : c.breaks) {
      if (std::find(ub.begin(), ub.end(), b) == ub.end()) ub.push_back(b);
    }
  }
  if (ub.size() > kDblMaxBreaks) return false;
  std::sort(ub.begin(), ub.end());
  std::vector<double> vx, vy;
  std::uint32_t chain_mask = 0;
  std::vector<std::uint32_t> bit_of;
  if (!detail::chain_edges(E, vx, vy, chain_mask, bit_of, kDblMaxVerts)) return false;
  std::memset(out, 0, 2 * kSlotBytes);
  out[0] = kSlotDouble;
  out[1] = static_cast<std::uint8_t>(vx.size());
  out[2] = static_cast<std::uint8_t>(C.size());
  out[3] = static_cast<std::uint8_t>(ub.size());
  std::memcpy(out + 4, &chain_mask, 4);
  for (std::size_t c = 0; c < C.size(); ++c) {
    const std::int32_t id = static_cast<std::int32_t>(C[c].id);
    std::memcpy(out + 8 + 4 * c, &id, 4);
    std::uint16_t mask = 0;
    for (std::uint32_t e : C[c].edges) mask |= static_cast<std::uint16_t>(1u << bit_of[e]);
    std::memcpy(out + 40 + 2 * c, &mask, 2);
    std::uint8_t info = static_cast<std::uint8_t>((C[c].c0 & 1u) << 7);
    for (double b : C[c].breaks) {
      info |= static_cast<std::uint8_t>(1u << (std::lower_bound(ub.begin(), ub.end(), b) - ub.begin()));
    }
    out[56 + c] = info;
  }
  for (std::size_t j = 0; j < ub.size(); ++j) std::memcpy(out + 64 + 8 * j, &ub[j], 8);
  for (std::size_t k = 0; k < vx.size(); ++k) {
    std::memcpy(out + 96 + 16 * k, &vx[k], 8);
    std::memcpy(out + 104 + 16 * k, &vy[k], 8);
  }
  return true;
}

// Encodes a split slot (kind 3).
inline void encode_split_slot(double x0, double y0, double inv_hw, double inv_hh,
                              const std::uint32_t child[4], std::uint8_t* out) {
  std::memset(out, 0, kSlotBytes);
  out[0] = kSlotSplit;
  std::memcpy(out + 8, &x0, 8);
  std::memcpy(out + 16, &y0, 8);
  std::memcpy(out + 24, &inv_hw, 8);
  std::memcpy(out + 32, &inv_hh, 8);
  std::memcpy(out + 40, child, 16);
}

// Encodes an overflow slot (kind 2) pointing at byte offset `off`.
inline void encode_overflow_slot(std::uint64_t off, std::uint8_t* out) {
  std::memset(out, 0, kSlotBytes);
  out[0] = kSlotOverflow;
  std::memcpy(out + 8, &off, 8);
}

}  // namespace fm
