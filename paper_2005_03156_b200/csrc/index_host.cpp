// index_host.cpp -- cell-index planning and the host (C++ threads) builder.
//
// Replaces the reference's recursive single-threaded cover build
// (CoverBuilder, cell_index.hpp:279-378, and build_trie, :453-507) with a
// uniform grid whose cells are classified conservatively per (cell, leaf)
// pair.  The classification is purely algebraic, so it is exact for ANY
// input (overlapping, self-intersecting, multi-ring, degenerate); DESIGN.md
// sec. 4 has the argument.  In short, for a point p of cell c and a leaf L
// the reference parity (geometry.hpp:214-225) is the XOR over L's
// non-horizontal edges e of [lo_e.lat < p.lat <= hi_e.lat and cross_e(p) > 0].
// Relative to the cell's latitude slab (expanded by the margin d) every
// edge is one of
//   y-disjoint  never in range for any p of the cell        -> contributes 0
//   left        wholly left of the cell by > d              -> cross <= 0, 0
//   right       wholly right of the cell by > d             -> cross > 0, so it
//               contributes [p.lat > lo] ^ [p.lat > hi]: endpoints below the
//               slab fold into a constant bit c0, endpoints inside the slab
//               become latitude breakpoints (pairs cancel)
//   near        everything else -> evaluated at query time with the
//               reference predicate itself.
// A cell whose leaves all have no near edges and no breakpoints has a
// constant answer (true hit / empty); otherwise it gets a boundary record.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "index_build.h"
#include "record_encode.h"
#include "sweep.h"

namespace fm {
namespace {

struct Contrib {
  std::uint32_t id;
  std::uint32_t c0;
  std::uint32_t force_defer;     // phase-1 capacity rule hit (sweep.h)
  std::uint32_t e_begin, e_end;  // into the row edge pool
  std::uint32_t b_begin, b_end;  // into the row break pool
};

struct RelEdge {
  std::int64_t tlo, thi;
  Edge4 e;
};

void toggle(std::vector<double>& set, double v) {
  auto it = std::lower_bound(set.begin(), set.end(), v);
  if (it != set.end() && *it == v) {
    set.erase(it);
  } else {
    set.insert(it, v);
  }
}

// One leaf's contribution to a rectangle: its near edges, the constant
// parity c0 of the edges wholly right of it, and the breakpoints.
struct PolyC {
  std::uint32_t id = 0, c0 = 0;
  bool force_defer = false;  // phase-1 capacity rule hit (sweep.h)
  std::vector<Edge4> near;
  std::vector<double> breaks;  // ascending, distinct
  bool constant() const { return near.empty() && breaks.empty(); }
};

struct Deferred {
  std::int64_t ix;
  std::vector<PolyC> list;
};

struct RowWorker {
  const Soup& s;
  const GridGeom& g;
  const std::vector<PolySpan>& spans;
  double tol;

  std::vector<std::vector<Contrib>> cols;
  std::vector<std::uint8_t> closed;
  std::vector<std::int64_t> touched;
  std::vector<Edge4> epool;
  std::vector<double> bpool;
  std::vector<RelEdge> rel;
  std::vector<std::uint32_t> order;
  std::vector<double> tog;
  BuildStats st;

  EncodeStats es;
  // per-row outputs (set by run_row)
  std::vector<std::uint8_t> slots;                  // row-local slot arena
  std::vector<std::uint8_t>* ovf = nullptr;         // row-local overflow arena
  std::vector<std::uint64_t>* slot_patches = nullptr;
  std::vector<std::uint64_t>* ovf_patches = nullptr;

  RowWorker(const Soup& s_, const GridGeom& g_, const std::vector<PolySpan>& sp, double t)
      : s(s_), g(g_), spans(sp), tol(t) {
    cols.resize(static_cast<std::size_t>(g.nx));
    closed.assign(static_cast<std::size_t>(g.nx), 0);
  }

  void gather_edges(std::uint32_t pid, double ys0, double ys1) {
    rel.clear();
    for (std::uint64_t r = s.poly_ring[pid]; r < s.poly_ring[pid + 1]; ++r) {
      const std::uint64_t b = s.ring_off[r], e = s.ring_off[r + 1], n = e - b;
      for (std::uint64_t i = 0; i < n; ++i) {
        const std::uint64_t a = b + i, c = (i + 1 < n) ? a + 1 : b;
        SlabEdge se;
        if (!slab_edge(g, tol, ys0, ys1, s.vxy[2 * a], s.vxy[2 * a + 1], s.vxy[2 * c],
                       s.vxy[2 * c + 1], &se)) {
          continue;
        }
        rel.push_back({se.tlo, se.thi, Edge4{se.lx, se.ly, se.hx, se.hy}});
      }
    }
  }

  void add_polygon(std::uint32_t pid, double ys0, double ys1) {
    const PolySpan& sp = spans[pid];
    gather_edges(pid, ys0, ys1);
    order.resize(rel.size());
    for (std::uint32_t k = 0; k < order.size(); ++k) order[k] = k;
    std::sort(order.begin(), order.end(),
              [&](std::uint32_t a, std::uint32_t b) { return rel[a].tlo > rel[b].tlo; });
    tog.clear();
    std::uint32_t c0par = 0;
    std::size_t k = 0;
    std::size_t raw_breaks = 0;  // in-slab endpoints of right edges (sweep.h cap)
    auto add_right = [&](const RelEdge& re) {
      for (const double m : {re.e.ly, re.e.hy}) {
        if (m < ys0) {
          c0par ^= 1u;
        } else if (m < ys1) {
          toggle(tog, m);
          ++raw_breaks;
        }
      }
    };
    const bool rel_over = rel.size() > static_cast<std::size_t>(kRelCap);
    for (std::int64_t ix = sp.c1; ix >= sp.c0; --ix) {
      while (k < order.size() && rel[order[k]].tlo > ix) add_right(rel[order[k++]]);
      if (closed[ix]) continue;
      const std::uint32_t eb = static_cast<std::uint32_t>(epool.size());
      for (const RelEdge& re : rel) {
        if (re.tlo <= ix && ix <= re.thi) epool.push_back(re.e);
      }
      const std::uint32_t ee = static_cast<std::uint32_t>(epool.size());
      const std::uint32_t force = (rel_over || ee - eb > static_cast<std::uint32_t>(kNearCap) ||
                                   tog.size() > static_cast<std::size_t>(kBreakCap) ||
                                   raw_breaks > static_cast<std::size_t>(kBreakRawCap)) ? 1u : 0u;
      if (ee == eb && tog.empty() && !force) {
        if (c0par) {  // constant-true leaf: terminal for this cell
          if (cols[ix].empty()) touched.push_back(ix);
          cols[ix].push_back({pid, 1u, 0u, eb, eb, 0, 0});
          closed[ix] = 1;
        }
        continue;
      }
      const std::uint32_t bb = static_cast<std::uint32_t>(bpool.size());
      bpool.insert(bpool.end(), tog.begin(), tog.end());
      if (cols[ix].empty()) touched.push_back(ix);
      cols[ix].push_back({pid, c0par, force, eb, ee, bb, static_cast<std::uint32_t>(bpool.size())});
    }
  }

  // Re-derive a leaf's contribution for a sub-rectangle of the rectangle
  // `par` was computed for: edges right of the parent
  // stay right of the child, so only the parent's near edges need
  // reclassifying, and the parent's breakpoints fold into the child's c0
  // (below the child slab), stay breakpoints (inside) or vanish (above).
  void reclassify(const PolyC& par, double rx0, double rx1, double ry0, double ry1,
                  PolyC& ch) const {
    const double d = g.margin;
    const double ys0 = ry0 - d, ys1 = ry1 + d, xs0 = rx0 - d, xs1 = rx1 + d;
    ch.id = par.id;
    ch.near.clear();
    ch.breaks.clear();
    std::uint32_t c0 = par.c0;
    for (const double b : par.breaks) {
      if (b < ys0) {
        c0 ^= 1u;
      } else if (b < ys1) {
        ch.breaks.push_back(b);
      }
    }
    for (const Edge4& E : par.near) {
      if (E.hy <= ys0 || E.ly >= ys1) continue;
      const double ya = std::max(E.ly, ys0), yb = std::min(E.hy, ys1);
      const double slope = (E.hx - E.lx) / (E.hy - E.ly);
      const double mnx = std::min(E.lx, E.hx), mxx = std::max(E.lx, E.hx);
      auto x_at = [&](double y) {
        const double x = E.lx + (y - E.ly) * slope;
        return std::min(mxx, std::max(mnx, x));
      };
      const double xa = (ya == E.ly) ? E.lx : x_at(ya);
      const double xb = (yb == E.hy) ? E.hx : x_at(yb);
      const double ex0 = std::min(xa, xb) - tol, ex1 = std::max(xa, xb) + tol;
      if (ex1 < xs0) continue;  // left of the child: never crosses
      if (ex0 > xs1) {          // right of the child: fold into c0 / breakpoints
        for (const double m : {E.ly, E.hy}) {
          if (m < ys0) {
            c0 ^= 1u;
          } else if (m < ys1) {
            toggle(ch.breaks, m);
          }
        }
        continue;
      }
      ch.near.push_back(E);
    }
    ch.c0 = c0;
  }

  // Entry for a rectangle given its leaves' contributions (ascending ids).
  // Appends slots to `slots` (row-local slot numbers; every u32 child entry
  // and u64 overflow offset inside a slot is listed for relocation).
  std::uint32_t finalize(const std::vector<PolyC>& list, double rx0, double ry0, double cw,
                         double chh, int depth, bool* deferred = nullptr) {
    std::vector<Edge4> U;
    std::vector<CandIn> cin;
    std::vector<std::size_t> src;  // index into list per candidate
    for (std::size_t q = 0; q < list.size(); ++q) {
      const PolyC& pc = list[q];
      if (deferred && pc.force_defer) {  // phase-1 capacity rules (sweep.h)
        *deferred = true;
        return kEmpty;
      }
      CandIn cd;
      cd.id = pc.id;
      cd.c0 = pc.c0;
      cd.breaks = pc.breaks;
      for (const Edge4& E : pc.near) {
        std::uint32_t idx = 0;
        while (idx < U.size() && !same_edge(U[idx], E)) ++idx;
        if (idx == U.size()) U.push_back(E);
        auto it = std::find(cd.edges.begin(), cd.edges.end(), idx);
        if (it != cd.edges.end()) {
          cd.edges.erase(it);  // even multiplicity cancels
        } else {
          cd.edges.push_back(idx);
        }
      }
      if (cd.edges.empty() && cd.breaks.empty()) {
        if (cd.c0) {  // constant true: terminal
          cin.push_back(std::move(cd));
          src.push_back(q);
          break;
        }
        continue;  // constant false
      }
      cin.push_back(std::move(cd));
      src.push_back(q);
    }
    if (deferred && (cin.size() > static_cast<std::size_t>(kCellCands) ||
                     U.size() > static_cast<std::size_t>(kCellEdges))) {
      *deferred = true;  // phase-1 per-cell limits (sweep.h)
      return kEmpty;
    }
    if (cin.empty()) return kEmpty;
    if (cin.front().edges.empty() && cin.front().breaks.empty()) return cin.front().id;
    // drop edges no candidate references any more
    std::vector<std::int64_t> remap(U.size(), -1);
    std::vector<Edge4> used;
    for (auto& cd : cin) {
      for (auto& e : cd.edges) {
        if (remap[e] < 0) {
          remap[e] = static_cast<std::int64_t>(used.size());
          used.push_back(U[e]);
        }
        e = static_cast<std::uint32_t>(remap[e]);
      }
    }
    std::uint64_t n_breaks = 0;
    for (const auto& c : cin) n_breaks += c.breaks.size();
    std::uint8_t slot[kSlotBytes];
    if (encode_slot(used, cin, slot)) {
      const std::uint64_t k = slots.size() / kSlotBytes;
      slots.insert(slots.end(), slot, slot + kSlotBytes);
      note_leaf(used.size(), cin.size(), n_breaks);
      es.compact++;
      return slot_entry(k, slot[0], slot[1], slot[2], slot[3]);
    }
    std::uint8_t dbl[2 * kSlotBytes];
    if (encode_double_slot(used, cin, dbl)) {  // e.g. a polygon corner: two slots, one read
      const std::uint64_t k = slots.size() / kSlotBytes;
      slots.insert(slots.end(), dbl, dbl + 2 * kSlotBytes);
      note_leaf(used.size(), cin.size(), n_breaks);
      es.compact++;
      st.slots_double++;
      return slot_entry(k, kSlotDouble, 0, 0, 0);
    }
    if (deferred) {  // phase 1: cells that need a split or overflow wait for phase 2
      *deferred = true;
      return kEmpty;
    }
    // A cell that fits neither a slot nor a double slot but a small compact
    // record takes the record (an overflow slot pointing at it) rather than
    // a split subtree: splitting recurses to kMaxSplitDepth around any
    // vertex where several chains meet (every child holding it is as full),
    // which is how c3's 12.5M corner cells once took 83M split nodes and
    // 270M of its 352M slots.
    const std::uint64_t rec_bytes = compact_record_bytes(used, cin);
    const bool small_record = rec_bytes > 0 && rec_bytes <= kSmallRecordBytes;
    if (!small_record && depth < kMaxSplitDepth && cw > 256.0 * g.margin && chh > 256.0 * g.margin) {
      // split 2x2: child (i, j) covers [rx0 + i*cw/2, rx0 + (i+1)*cw/2] x ...
      const double hw = 0.5 * cw, hh = 0.5 * chh;
      std::uint32_t child[4];
      for (int j = 0; j < 2; ++j) {
        for (int i = 0; i < 2; ++i) {
          const double cx0 = rx0 + i * hw, cy0 = ry0 + j * hh;
          std::vector<PolyC> sub;
          for (const std::size_t q : src) {
            PolyC pc;
            reclassify(list[q], cx0, cx0 + hw, cy0, cy0 + hh, pc);
            if (pc.constant()) {
              if (pc.c0) {
                sub.push_back(std::move(pc));
                break;
              }
              continue;
            }
            sub.push_back(std::move(pc));
          }
          child[2 * j + i] = finalize(sub, cx0, cy0, hw, hh, depth + 1);
        }
      }
      const std::uint64_t k = slots.size() / kSlotBytes;
      encode_split_slot(rx0, ry0, 1.0 / hw, 1.0 / hh, child, slot);
      slots.insert(slots.end(), slot, slot + kSlotBytes);
      for (int c = 0; c < 4; ++c) {
        if (child[c] >= kRecordBit && child[c] != kEmpty) slot_patches->push_back(k * kSlotBytes + 40 + 4 * c);
      }
      st.cells_split++;
      return slot_entry(k, kSlotSplit, 0, 0, 0);
    }
    // past the split depth: variable-size record in the overflow arena
    const std::uint64_t off = ovf->size();
    EncodeStats tmp;
    encode_record(used, cin, *ovf, &tmp);
    es.compact += tmp.compact;
    es.wide += tmp.wide;
    const std::uint64_t k = slots.size() / kSlotBytes;
    encode_overflow_slot(off, slot);
    slots.insert(slots.end(), slot, slot + kSlotBytes);
    ovf_patches->push_back(k * kSlotBytes + 8);
    note_leaf(used.size(), cin.size(), n_breaks);
    st.records_overflow++;
    return slot_entry(k, kSlotOverflow, 0, 0, 0);
  }

  void note_leaf(std::uint64_t ne, std::uint64_t nc, std::uint64_t nb) {
    st.records++;
    st.record_edges += ne;
    st.record_cands += nc;
    st.record_breaks += nb;
    st.max_record_edges = std::max(st.max_record_edges, ne);
    st.max_record_cands = std::max(st.max_record_cands, nc);
  }

  // Phase 1 for one grid row: classify every cell; hits and empties go to
  // the grid, cells that fit one slot get it (row-local numbering), the
  // rest are deferred with their contributions.
  void run_row(std::int64_t iy, const std::uint32_t* ids, std::uint64_t n_ids,
               std::uint32_t* grid_row, std::vector<std::uint8_t>& row_slots,
               std::vector<std::int64_t>& rec_cols, std::vector<Deferred>& deferred) {
    slots.clear();
    const double ys0 = cell_y0(g, iy) - g.margin;
    const double ys1 = cell_y0(g, iy + 1) + g.margin;
    epool.clear();
    bpool.clear();
    touched.clear();
    for (std::uint64_t q = 0; q < n_ids; ++q) add_polygon(ids[q], ys0, ys1);
    std::sort(touched.begin(), touched.end());
    std::vector<PolyC> list;
    for (const std::int64_t ix : touched) {
      list.clear();
      for (const Contrib& c : cols[ix]) {
        PolyC pc;
        pc.id = c.id;
        pc.c0 = c.c0;
        pc.force_defer = c.force_defer != 0;
        pc.near.assign(epool.begin() + c.e_begin, epool.begin() + c.e_end);
        pc.breaks.assign(bpool.begin() + c.b_begin, bpool.begin() + c.b_end);
        list.push_back(std::move(pc));
      }
      bool defer = false;
      const std::uint32_t e = finalize(list, cell_x0(g, ix), cell_y0(g, iy), g.w, g.h, 0, &defer);
      if (defer) {
        deferred.push_back({ix, std::move(list)});
        list = {};
        grid_row[ix] = kEmpty;  // set in phase 2
        st.cells_boundary++;
      } else {
        grid_row[ix] = e;
        if (e == kEmpty) {
          st.cells_empty++;
        } else if (e < kRecordBit) {
          st.cells_hit++;
        } else {
          st.cells_boundary++;
          rec_cols.push_back(ix);
        }
      }
      cols[ix].clear();
      closed[ix] = 0;
    }
    st.cells_empty += static_cast<std::uint64_t>(g.nx) - touched.size();
    row_slots.swap(slots);
  }

  // Phase 2 for one grid row: the deferred cells' split / overflow subtrees
  // (row-local slot numbers and overflow offsets, patch lists for both).
  void run_deferred(std::int64_t iy, const std::vector<Deferred>& deferred,
                    std::vector<std::uint8_t>& row_slots, std::vector<std::uint8_t>& row_ovf,
                    std::vector<std::uint64_t>& spatch, std::vector<std::uint64_t>& opatch,
                    std::vector<std::uint32_t>& entries) {
    slots.clear();
    ovf = &row_ovf;
    slot_patches = &spatch;
    ovf_patches = &opatch;
    entries.clear();
    for (const Deferred& d : deferred) {
      entries.push_back(finalize(d.list, cell_x0(g, d.ix), cell_y0(g, iy), g.w, g.h, 0));
    }
    row_slots.swap(slots);
  }

  // Contributions of the given leaves (ascending ids) to cell (ix, iy),
  // computed directly -- the same arithmetic as the row sweep (used for the
  // cells the GPU builder hands back).
  void cell_contribs(std::int64_t ix, std::int64_t iy, const std::uint32_t* ids, std::uint64_t n,
                     std::vector<PolyC>& list) {
    list.clear();
    const double ys0 = cell_y0(g, iy) - g.margin;
    const double ys1 = cell_y0(g, iy + 1) + g.margin;
    for (std::uint64_t q = 0; q < n; ++q) {
      gather_edges(ids[q], ys0, ys1);
      PolyC pc;
      pc.id = ids[q];
      std::uint32_t c0 = 0;
      for (const RelEdge& re : rel) {
        if (re.tlo > ix) {
          for (const double m : {re.e.ly, re.e.hy}) {
            if (m < ys0) {
              c0 ^= 1u;
            } else if (m < ys1) {
              toggle(pc.breaks, m);
            }
          }
        } else if (re.thi >= ix) {
          pc.near.push_back(re.e);
        }
      }
      pc.c0 = c0;
      if (pc.constant()) {
        if (c0) {
          list.push_back(std::move(pc));
          return;  // terminal: later leaves never matter
        }
        continue;
      }
      list.push_back(std::move(pc));
    }
  }
};

}  // namespace

GridGeom plan_grid(const Soup& s, const BuildOptions& o, BuildStats* st) {
  if (s.n_polys > kMaxLeaves) throw InvalidArgument("too many leaves for int32 ids");
  if (s.n_polys > 0 && (s.poly_ring == nullptr || s.ring_off == nullptr || s.vxy == nullptr)) {
    throw InvalidArgument("null polygon soup arrays");
  }
  if (!(o.cells_per_polygon >= 0.0) || !(o.margin >= 0.0) || o.nx < 0 || o.ny < 0) {
    throw InvalidArgument("invalid index build parameters");
  }
  bool served_exact = false;  // see BuildStats::approx_served_exact
  double ux0 = INFINITY, ux1 = -INFINITY, uy0 = INFINITY, uy1 = -INFINITY;
  double sum_w = 0.0, sum_h = 0.0;
  std::uint64_t active = 0, n_edges = 0;
  for (std::uint64_t p = 0; p < s.n_polys; ++p) {
    const std::uint64_t r0 = s.poly_ring[p], r1 = s.poly_ring[p + 1];
    if (r1 < r0 || r1 > s.n_rings) throw InvalidArgument("bad polygon ring offsets");
    if (r0 == r1) continue;
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (std::uint64_t r = r0; r < r1; ++r) {
      const std::uint64_t b = s.ring_off[r], e = s.ring_off[r + 1];
      if (e < b || e - b < 3) {
        throw InvalidArgument("polygon ring needs at least 3 vertices");  // geometry.hpp:75-77
      }
      n_edges += e - b;
      for (std::uint64_t v = b; v < e; ++v) {
        const double x = s.vxy[2 * v], y = s.vxy[2 * v + 1];
        if (!std::isfinite(x) || !std::isfinite(y)) {
          throw InvalidArgument("non-finite polygon vertex");
        }
        x0 = std::min(x0, x);
        x1 = std::max(x1, x);
        y0 = std::min(y0, y);
        y1 = std::max(y1, y);
      }
    }
    ux0 = std::min(ux0, x0);
    ux1 = std::max(ux1, x1);
    uy0 = std::min(uy0, y0);
    uy1 = std::max(uy1, y1);
    sum_w += x1 - x0;
    sum_h += y1 - y0;
    ++active;
  }
  if (st) st->n_edges = n_edges;
  GridGeom g{};
  if (active == 0) {
    g.gx0 = 0.0;
    g.gx1 = 1.0;
    g.gy0 = 0.0;
    g.gy1 = 1.0;
    g.nx = g.ny = 1;
    g.w = g.h = 1.0;
    g.inv_w = g.inv_h = 1.0;
    g.margin = o.margin > 0 ? o.margin : std::ldexp(1.0, -40);
    return g;
  }
  double M = std::max(std::max(std::fabs(ux0), std::fabs(ux1)),
                      std::max(std::fabs(uy0), std::fabs(uy1)));
  if (!(M >= 1.0)) M = 1.0;
  g.margin = o.margin > 0.0 ? o.margin : std::ldexp(M, -40);
  const double pad = 4.0 * g.margin;
  g.gx0 = ux0 - pad;
  g.gx1 = ux1 + pad;
  g.gy0 = uy0 - pad;
  g.gy1 = uy1 + pad;
  const double GW = g.gx1 - g.gx0, GH = g.gy1 - g.gy0;
  std::int64_t nx = o.nx, ny = o.ny;
  if (nx <= 0 || ny <= 0) {
    double mw = sum_w / static_cast<double>(active), mh = sum_h / static_cast<double>(active);
    const double side = std::sqrt(static_cast<double>(active));
    if (!(mw > 0.0)) mw = GW / side;
    if (!(mh > 0.0)) mh = GH / side;
    double m = o.cells_per_polygon;
    if (!(m > 0.0)) {
      // ~450M cells (c2: 42 cells per polygon side, 9% boundary points;
      // measured optimum 40-48 with 16-byte small sub-blocks), 4..64 per
      // side.  Tilings of more than 4M leaves (c3: 12.5M) get ~800M: their
      // indexes take the binned path on a flat grid, where a finer grid
      // only trades boundary points for arena bytes -- c3 queries 1B points
      // in 22.3 ms at 8 cells per leaf side (474M cells, 25.7 GB arena)
      // against 23.2 at 7 and 24.5 at 6 (profiles/r2ca); 9 per side does
      // not build next to 1B resident points.
      const double budget = active > 4000000 ? 800.0e6 : 450.0e6;
      m = std::sqrt(budget / static_cast<double>(active));
      // (cap 64: c4, 100k concave polygons on the binned path, 4.76 ms per 200M
      // points at 64 per side against 5.13 at 48, 4.82 at 80: profiles/r2cd)
      m = std::min(64.0, std::max(4.0, m));
      // few polygons (>= 64): still at least ~10M cells (a ~40 MB grid, L2-sized),
      // since the 48-per-side cap would leave a needlessly coarse grid
      // (c1, 1,024 polygons: 48 -> 99 per side, 0.70 -> 0.62 ms per 100M
      // points)
      if (active >= 64) m = std::max(m, std::min(1024.0, std::sqrt(10.0e6 / static_cast<double>(active))));
    }
    nx = static_cast<std::int64_t>(std::ceil(GW / (mw / m)));
    ny = static_cast<std::int64_t>(std::ceil(GH / (mh / m)));
    if (!(o.cells_per_polygon > 0.0)) {
      // the budgets above assume the polygons tile their bbox; a sparse
      // layer (polygons covering a fraction f of the bbox) would get 1/f
      // times as many cells, so the total is capped at ~1.5x the intended
      // count (active polygons x m^2)
      const double want = 1.5 * static_cast<double>(active) * m * m;
      const double got = static_cast<double>(nx) * static_cast<double>(ny);
      if (got > want) {
        const double k = std::sqrt(want / got);
        nx = static_cast<std::int64_t>(std::ceil(static_cast<double>(nx) * k));
        ny = static_cast<std::int64_t>(std::ceil(static_cast<double>(ny) * k));
      }
    }
    nx = std::min<std::int64_t>(std::max<std::int64_t>(nx, 1), std::int64_t{1} << 22);
    ny = std::min<std::int64_t>(std::max<std::int64_t>(ny, 1), std::int64_t{1} << 22);
    while (nx * ny > (std::int64_t{1} << 30)) {
      nx = (nx + 1) / 2;
      ny = (ny + 1) / 2;
    }
  }
  if (o.approx_epsilon > 0.0) {
    // fast-approx covers (cell_index.hpp:313-316): every boundary cell's
    // margin-expanded diagonal must be <= epsilon, so raise the resolution
    const double side = o.approx_epsilon / std::sqrt(2.0) * (1.0 - 1e-9) - 2.0 * g.margin;
    if (!(side > 0.0)) throw InvalidArgument("approx epsilon is below the classification margin");
    const double ex = std::ceil(GW / side), ey = std::ceil(GH / side);
    if (ex * ey > static_cast<double>(std::int64_t{1} << 31)) {
      // finer than a uniform grid of 2^31 cells can resolve over this
      // extent: plan the exact grid and serve approximate queries exactly,
      // which meets the reference's bound (answers within epsilon of the
      // exact one, test_cell_index.cpp:381-435) with error 0
      served_exact = true;
      if (st) st->approx_served_exact = true;
    } else {
      // auto resolution: exactly what epsilon needs (the reference's approx
      // cover stops refining there too); explicit resolutions are only raised
      const bool explicit_res = (o.nx > 0 && o.ny > 0) || o.cells_per_polygon > 0.0;
      nx = explicit_res ? std::max(nx, static_cast<std::int64_t>(ex)) : static_cast<std::int64_t>(ex);
      ny = explicit_res ? std::max(ny, static_cast<std::int64_t>(ey)) : static_cast<std::int64_t>(ey);
    }
  }
  if (nx * ny > (std::int64_t{1} << 31)) throw InvalidArgument("grid too large");
  g.nx = nx;
  g.ny = ny;
  g.w = GW / static_cast<double>(nx);
  g.h = GH / static_cast<double>(ny);
  g.inv_w = static_cast<double>(nx) / GW;
  g.inv_h = static_cast<double>(ny) / GH;
  if (o.approx_epsilon > 0.0 && !served_exact &&
      !(std::hypot(g.w + 2.0 * g.margin, g.h + 2.0 * g.margin) <= o.approx_epsilon)) {
    throw InvalidArgument("grid cells exceed the approx epsilon");
  }
  return g;
}

namespace {

std::vector<PolySpan> compute_spans(const Soup& s, const GridGeom& g) {
  std::vector<PolySpan> spans(s.n_polys);
  for (std::uint64_t p = 0; p < s.n_polys; ++p) {
    PolySpan& sp = spans[p];
    sp.active = 0;
    if (s.poly_ring[p + 1] <= s.poly_ring[p]) continue;
    double x0 = INFINITY, x1 = -INFINITY, y0 = INFINITY, y1 = -INFINITY;
    for (std::uint64_t v = s.ring_off[s.poly_ring[p]]; v < s.ring_off[s.poly_ring[p + 1]]; ++v) {
      x0 = std::min(x0, s.vxy[2 * v]);
      x1 = std::max(x1, s.vxy[2 * v]);
      y0 = std::min(y0, s.vxy[2 * v + 1]);
      y1 = std::max(y1, s.vxy[2 * v + 1]);
    }
    polygon_span(g, x0, x1, y0, y1, &sp);
  }
  return spans;
}

// Row -> leaves CSR (ascending ids per row).
void row_lists(const std::vector<PolySpan>& spans, const GridGeom& g,
               std::vector<std::uint64_t>& row_count, std::vector<std::uint32_t>& row_ids) {
  row_count.assign(static_cast<std::size_t>(g.ny) + 1, 0);
  for (const PolySpan& sp : spans) {
    if (!sp.active) continue;
    for (std::int64_t r = sp.r0; r <= sp.r1; ++r) row_count[static_cast<std::size_t>(r) + 1]++;
  }
  for (std::int64_t r = 0; r < g.ny; ++r) row_count[r + 1] += row_count[r];
  row_ids.resize(row_count[static_cast<std::size_t>(g.ny)]);
  std::vector<std::uint64_t> fill(row_count.begin(), row_count.end() - 1);
  for (std::uint64_t p = 0; p < spans.size(); ++p) {
    if (!spans[p].active) continue;
    for (std::int64_t r = spans[p].r0; r <= spans[p].r1; ++r) {
      row_ids[fill[static_cast<std::size_t>(r)]++] = static_cast<std::uint32_t>(p);
    }
  }
}

template <typename Fn>
void parallel_rows(std::int64_t ny, int threads, Fn fn) {
  std::atomic<std::int64_t> next{0};
  std::mutex mu;
  std::exception_ptr failure;
  auto worker = [&](int t) {
    try {
      fn(t, next);
    } catch (...) {
      std::lock_guard<std::mutex> lk(mu);
      if (!failure) failure = std::current_exception();
      next.store(ny);
    }
  };
  std::vector<std::thread> pool;
  for (int t = 1; t < threads; ++t) pool.emplace_back(worker, t);
  worker(0);
  for (auto& th : pool) th.join();
  if (failure) std::rethrow_exception(failure);
}

int thread_count(const BuildOptions& o, std::int64_t ny) {
  int threads = o.threads > 0 ? o.threads : static_cast<int>(std::thread::hardware_concurrency());
  if (threads < 1) threads = 1;
  return static_cast<int>(std::min<std::int64_t>(threads, std::max<std::int64_t>(ny, 1)));
}

void merge_stats(BuildStats& into, const BuildStats& st) {
  into.cells_empty += st.cells_empty;
  into.cells_hit += st.cells_hit;
  into.cells_boundary += st.cells_boundary;
  into.record_edges += st.record_edges;
  into.record_cands += st.record_cands;
  into.record_breaks += st.record_breaks;
  into.max_record_edges = std::max(into.max_record_edges, st.max_record_edges);
  into.max_record_cands = std::max(into.max_record_cands, st.max_record_cands);
  into.records_compact += st.records_compact;
  into.records_wide += st.records_wide;
  into.records += st.records;
  into.records_overflow += st.records_overflow;
  into.cells_split += st.cells_split;
  into.slots_double += st.slots_double;
}

}  // namespace

// Phase 2 (shared by the host and GPU builders): the deferred cells of each
// row, in row-major order, get their split / overflow subtrees appended
// after `slot_base` slots; their grid entries are written into `grid`.
void finish_deferred(const Soup& s, const GridGeom& g, const BuildOptions& o,
                     std::vector<std::vector<Deferred>>& deferred, std::uint64_t slot_base,
                     std::vector<std::uint32_t>& grid, std::vector<std::uint8_t>& slots_out,
                     std::vector<std::uint8_t>& ovf_out, BuildStats& stats) {
  const std::size_t NY = deferred.size();
  const int threads = thread_count(o, static_cast<std::int64_t>(NY));
  std::vector<std::vector<std::uint8_t>> rs(NY), ro(NY);
  std::vector<std::vector<std::uint64_t>> sp(NY), op(NY);
  std::vector<std::vector<std::uint32_t>> ent(NY);
  std::vector<BuildStats> st(static_cast<std::size_t>(threads));
  std::vector<PolySpan> no_spans;
  const double tol = classify_tol(g);
  parallel_rows(static_cast<std::int64_t>(NY), threads, [&](int t, std::atomic<std::int64_t>& next) {
    RowWorker w(s, g, no_spans, tol);
    for (;;) {
      const std::int64_t r = next.fetch_add(1);
      if (r >= static_cast<std::int64_t>(NY)) break;
      if (deferred[r].empty()) continue;
      w.run_deferred(r, deferred[r], rs[r], ro[r], sp[r], op[r], ent[r]);
    }
    st[t] = w.st;
    st[t].records_compact = w.es.compact;
    st[t].records_wide = w.es.wide;
  });
  std::uint64_t n_slots = 0, ovf_bytes = 0;
  std::vector<std::uint64_t> sb(NY), ob(NY);
  for (std::size_t r = 0; r < NY; ++r) {
    sb[r] = slot_base + n_slots;
    ob[r] = ovf_bytes;
    n_slots += rs[r].size() / kSlotBytes;
    ovf_bytes += (ro[r].size() + 15) & ~std::uint64_t{15};
  }
  if (slot_base + n_slots > kMaxSlots) throw RuntimeError("index needs more than 2^29 slots");
  slots_out.assign(n_slots * kSlotBytes, 0);
  ovf_out.assign(ovf_bytes, 0);
  std::uint64_t so = 0;
  for (std::size_t r = 0; r < NY; ++r) {
    if (rs[r].empty() && ent[r].empty()) continue;
    const std::uint32_t base = static_cast<std::uint32_t>(sb[r]);
    std::uint8_t* dst = slots_out.data() + so;
    if (!rs[r].empty()) std::memcpy(dst, rs[r].data(), rs[r].size());
    if (!ro[r].empty()) std::memcpy(ovf_out.data() + ob[r], ro[r].data(), ro[r].size());
    for (const std::uint64_t pos : sp[r]) {
      std::uint32_t v;
      std::memcpy(&v, dst + pos, 4);
      v += base;
      std::memcpy(dst + pos, &v, 4);
    }
    for (const std::uint64_t pos : op[r]) {
      std::uint64_t v;
      std::memcpy(&v, dst + pos, 8);
      v += ob[r];
      std::memcpy(dst + pos, &v, 8);
    }
    for (std::size_t k = 0; k < deferred[r].size(); ++k) {
      std::uint32_t e = ent[r][k];
      if (e >= kRecordBit && e != kEmpty) e += base;
      grid[r * static_cast<std::size_t>(g.nx) + static_cast<std::size_t>(deferred[r][k].ix)] = e;
    }
    so += rs[r].size();
  }
  for (const auto& x : st) merge_stats(stats, x);
}

HostIndex build_index_host(const Soup& s, const BuildOptions& o) {
  HostIndex out;
  out.g = plan_grid(s, o, &out.stats);
  const GridGeom& g = out.g;
  const std::size_t ncell = static_cast<std::size_t>(g.nx * g.ny);
  out.grid.assign(ncell, kEmpty);
  out.slots.assign(kSlotBytes, 0);  // never referenced; keeps device buffers non-empty
  out.overflow.assign(512, 0);
  if (s.n_polys == 0) {
    out.stats.cells_empty = ncell;
    return out;
  }
  const std::vector<PolySpan> spans = compute_spans(s, g);
  std::vector<std::uint64_t> row_count;
  std::vector<std::uint32_t> row_ids;
  row_lists(spans, g, row_count, row_ids);
  const double tol = classify_tol(g);
  const int threads = thread_count(o, g.ny);
  const std::size_t NY = static_cast<std::size_t>(g.ny);

  // phase 1: every row in parallel
  std::vector<std::vector<std::uint8_t>> row_slots(NY);
  std::vector<std::vector<std::int64_t>> row_recs(NY);
  std::vector<std::vector<Deferred>> deferred(NY);
  std::vector<BuildStats> stats(static_cast<std::size_t>(threads));
  parallel_rows(g.ny, threads, [&](int t, std::atomic<std::int64_t>& next) {
    RowWorker w(s, g, spans, tol);
    for (;;) {
      const std::int64_t iy = next.fetch_add(1);
      if (iy >= g.ny) break;
      w.run_row(iy, row_ids.data() + row_count[iy], row_count[iy + 1] - row_count[iy],
                out.grid.data() + iy * g.nx, row_slots[iy], row_recs[iy], deferred[iy]);
    }
    stats[t] = w.st;
    stats[t].records_compact = w.es.compact;
    stats[t].records_wide = w.es.wide;
  });
  for (const auto& st : stats) merge_stats(out.stats, st);
  // phase-1 slots in row-major order
  std::uint64_t n1 = 0;
  std::vector<std::uint64_t> base1(NY);
  for (std::size_t r = 0; r < NY; ++r) {
    base1[r] = n1;
    n1 += row_slots[r].size() / kSlotBytes;
  }
  std::vector<std::uint8_t> slots2, ovf2;
  finish_deferred(s, g, o, deferred, n1, out.grid, slots2, ovf2, out.stats);
  const std::uint64_t n_slots = n1 + slots2.size() / kSlotBytes;
  out.slots.assign((n_slots ? n_slots : 1) * kSlotBytes, 0);
  for (std::size_t r = 0; r < NY; ++r) {
    if (!row_slots[r].empty()) {
      std::memcpy(out.slots.data() + base1[r] * kSlotBytes, row_slots[r].data(), row_slots[r].size());
    }
    const std::uint32_t b = static_cast<std::uint32_t>(base1[r]);
    for (const std::int64_t ix : row_recs[r]) out.grid[r * static_cast<std::size_t>(g.nx) + static_cast<std::size_t>(ix)] += b;
    std::vector<std::uint8_t>().swap(row_slots[r]);
  }
  if (!slots2.empty()) std::memcpy(out.slots.data() + n1 * kSlotBytes, slots2.data(), slots2.size());
  out.overflow = std::move(ovf2);
  out.overflow.resize(out.overflow.size() + 512, 0);  // zero tail
  out.n_slots = n_slots;
  out.n_phase1_slots = n1;
  return out;
}

// For the GPU builder: phase 2 for the cells it deferred.  `cells` are
// linear cell ids in row-major order with their candidate leaves (CSR,
// ascending ids).
void finish_deferred_cells(const Soup& s, const GridGeom& g, const BuildOptions& o,
                           const std::vector<std::int64_t>& cells,
                           const std::vector<std::uint64_t>& cand_off,
                           const std::vector<std::uint32_t>& cand_ids, std::uint64_t slot_base,
                           std::vector<std::uint32_t>& grid, std::vector<std::uint8_t>& slots_out,
                           std::vector<std::uint8_t>& ovf_out, BuildStats& stats) {
  const std::size_t NY = static_cast<std::size_t>(g.ny);
  std::vector<std::vector<Deferred>> deferred(NY);
  std::vector<PolySpan> no_spans;
  const double tol = classify_tol(g);
  // contributions per deferred cell, threads over blocks of cells (the
  // per-row lists stay in row-major, column-ascending order)
  std::vector<std::vector<PolyC>> lists(cells.size());
  const int threads = thread_count(o, static_cast<std::int64_t>(cells.size() / 64 + 1));
  const std::int64_t n_blocks = static_cast<std::int64_t>((cells.size() + 255) / 256);
  parallel_rows(n_blocks, threads, [&](int, std::atomic<std::int64_t>& next) {
    RowWorker w(s, g, no_spans, tol);
    for (;;) {
      const std::int64_t b = next.fetch_add(1);
      if (b >= n_blocks) break;
      const std::size_t k1 = std::min(cells.size(), static_cast<std::size_t>(b + 1) * 256);
      for (std::size_t k = static_cast<std::size_t>(b) * 256; k < k1; ++k) {
        const std::int64_t iy = cells[k] / g.nx, ix = cells[k] % g.nx;
        w.cell_contribs(ix, iy, cand_ids.data() + cand_off[k], cand_off[k + 1] - cand_off[k], lists[k]);
      }
    }
  });
  for (std::size_t k = 0; k < cells.size(); ++k) {
    const std::int64_t iy = cells[k] / g.nx, ix = cells[k] % g.nx;
    deferred[static_cast<std::size_t>(iy)].push_back({ix, std::move(lists[k])});
  }
  finish_deferred(s, g, o, deferred, slot_base, grid, slots_out, ovf_out, stats);
}

}  // namespace fm
