// sweep.h -- cell-classification arithmetic shared by the host builder and
// the GPU builder (__host__ __device__), so both produce bit-identical
// indexes.  DESIGN.md sec. 4.2 states what the classification proves.
#pragma once

#include <cmath>
#include <cstdint>

#include "index_format.h"

namespace fm {

// Phase-1 capacity rules shared by both builders: a cell is deferred to the
// host's phase 2 when, before its first terminal leaf, some leaf's record
// exceeds these (or the cell exceeds the per-cell limits), so the GPU and
// host builders defer exactly the same cells and emit identical arrays.
constexpr int kRelCap = 64;     // slab-relevant edges per (row, leaf)
constexpr int kNearCap = 5;     // near edges per (cell, leaf)
constexpr int kBreakCap = 2;    // breakpoints per (cell, leaf)
constexpr int kBreakRawCap = 64;  // in-slab endpoints of right edges per (cell, leaf)
constexpr int kCellCands = 8;   // non-constant-false leaves per cell
constexpr int kCellEdges = 16;  // distinct edges per cell

// smallest k in [0, n) with g0 + (k+1)*step >= v; n if none
FM_HD std::int64_t first_with_hi_ge(double g0, double step, double inv, std::int64_t n, double v) {
  const double f = floor((v - g0) * inv) - 1.0;
  std::int64_t k = !(f > 0.0) ? 0 : (f > static_cast<double>(n) ? n : static_cast<std::int64_t>(f));
  while (k > 0 && g0 + static_cast<double>(k) * step >= v) --k;  // hi(k-1) = g0 + k*step
  while (k < n && g0 + static_cast<double>(k + 1) * step < v) ++k;
  return k;
}

// largest k in [0, n) with g0 + k*step <= v; -1 if none
FM_HD std::int64_t last_with_lo_le(double g0, double step, double inv, std::int64_t n, double v) {
  const double f = floor((v - g0) * inv) + 1.0;
  std::int64_t k = !(f > -1.0) ? -1 : (f > static_cast<double>(n - 1) ? n - 1 : static_cast<std::int64_t>(f));
  while (k >= 0 && g0 + static_cast<double>(k) * step > v) --k;
  while (k + 1 < n && g0 + static_cast<double>(k + 1) * step <= v) ++k;
  return k;
}

struct PolySpan {
  double x0, x1, y0, y1;      // tight bbox
  std::int64_t c0, c1, r0, r1;  // grid columns / rows whose margin-expanded cells meet it
  std::int32_t active;
  std::int32_t pad;
};

// Cell span of one polygon's bbox (cells whose margin-expanded rectangle
// meets the bbox).
FM_HD void polygon_span(const GridGeom& g, double x0, double x1, double y0, double y1,
                        PolySpan* sp) {
  const double d = g.margin;
  sp->x0 = x0;
  sp->x1 = x1;
  sp->y0 = y0;
  sp->y1 = y1;
  sp->c0 = first_with_hi_ge(g.gx0, g.w, g.inv_w, g.nx, x0 - d);
  sp->c1 = last_with_lo_le(g.gx0, g.w, g.inv_w, g.nx, x1 + d);
  sp->r0 = first_with_hi_ge(g.gy0, g.h, g.inv_h, g.ny, y0 - d);
  sp->r1 = last_with_lo_le(g.gy0, g.h, g.inv_h, g.ny, y1 + d);
  sp->active = (sp->c0 <= sp->c1 && sp->r0 <= sp->r1) ? 1 : 0;
}

// One polygon edge against a row slab [ys0, ys1] (already margin-expanded).
// Orients it like geometry.hpp:219; returns false when it can never be in
// range for a point of the slab (horizontal or y-disjoint).  Otherwise sets
// the oriented coordinates and the column range [tlo, thi] where it is
// "near"; columns < tlo see it wholly to their right, columns > thi wholly
// to their left.
struct SlabEdge {
  double lx, ly, hx, hy;
  std::int64_t tlo, thi;
};

FM_HD bool slab_edge(const GridGeom& g, double tol, double ys0, double ys1, double ax, double ay,
                     double bx, double by, SlabEdge* out) {
  double lx = ax, ly = ay, hx = bx, hy = by;
  if (ly > hy) {  // orient upward exactly like geometry.hpp:219
    lx = bx;
    ly = by;
    hx = ax;
    hy = ay;
  }
  if (ly == hy) return false;               // horizontal: never in range
  if (hy <= ys0 || ly >= ys1) return false;  // y-disjoint with the slab
  const double ya = ly > ys0 ? ly : ys0, yb = hy < ys1 ? hy : ys1;
  const double slope = (hx - lx) / (hy - ly);
  const double mnx = lx < hx ? lx : hx, mxx = lx < hx ? hx : lx;
  double xa, xb;
  if (ya == ly) {
    xa = lx;
  } else {
    const double x = lx + (ya - ly) * slope;
    xa = x < mnx ? mnx : (x > mxx ? mxx : x);
  }
  if (yb == hy) {
    xb = hx;
  } else {
    const double x = lx + (yb - ly) * slope;
    xb = x < mnx ? mnx : (x > mxx ? mxx : x);
  }
  const double ex0 = (xa < xb ? xa : xb) - tol, ex1 = (xa < xb ? xb : xa) + tol;
  out->lx = lx;
  out->ly = ly;
  out->hx = hx;
  out->hy = hy;
  out->tlo = first_with_hi_ge(g.gx0, g.w, g.inv_w, g.nx, ex0 - g.margin);
  out->thi = last_with_lo_le(g.gx0, g.w, g.inv_w, g.nx, ex1 + g.margin);
  return true;
}

// classification rounding guard (well below the margin)
FM_HD double classify_tol(const GridGeom& g) {
  double M = fabs(g.gx0);
  M = fabs(g.gx1) > M ? fabs(g.gx1) : M;
  M = fabs(g.gy0) > M ? fabs(g.gy0) : M;
  M = fabs(g.gy1) > M ? fabs(g.gy1) : M;
  return ldexp(M > 1.0 ? M : 1.0, -46);
}

}  // namespace fm
